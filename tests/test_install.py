"""install() wires the drop-ins into the reference package at its own names
(CPU: only the patching is checked; the functions need the device)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_install_patches_every_route_and_uninstall_restores():
    sys.path.insert(0, REF)
    try:
        import msfm.densify
        import msfm.guided

        from paper_1512_06235_b200 import guided, install
        orig = msfm.guided.guided_match_pair
        done = install.install()
        assert "msfm.guided.guided_match_pair" in done
        assert "msfm.densify.densify_stage" in done
        assert len(done) == len(install._ROUTES)        # every route exists in the reference
        assert msfm.guided.guided_match_pair is guided.guided_match_pair
        assert msfm.densify.guided_match_pair is guided.guided_match_pair
        install.uninstall()
        assert msfm.guided.guided_match_pair is orig
    finally:
        sys.path.remove(REF)
        # later tests resolve the reference's types through `msfm` when importable:
        # leave no trace of it
        for name in [n for n in sys.modules if n == "msfm" or n.startswith("msfm.")]:
            del sys.modules[name]
