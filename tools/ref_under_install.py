"""pytest plugin: the reference's own test modules with the B200 drop-ins installed
(SURVEY.md §4 "run the reference's hot-path suite against the
drop-in").  Loaded with ``-p ref_under_install`` before collection, so every
``from msfm.x import f`` in the reference's tests binds the patched function.

    PYTHONPATH=tools:.:baseline/_ref python -m pytest -p ref_under_install \\
        baseline/_ref/tests/test_guided.py ...

baseline/_ref holds ``pip install --target`` of /root/reference/pkg plus a copy of
its tests/ (git-ignored, shipped to the GPU box with the snapshot).
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (os.path.join(REPO, "baseline", "_ref"), REPO):
    if p not in sys.path:
        sys.path.insert(0, p)

import paper_1512_06235_b200.install as _b200  # noqa: E402

PATCHED = _b200.install()


def pytest_report_header(config):
    return f"B200 drop-ins installed over msfm: {len(PATCHED)} routes ({', '.join(PATCHED)})"
