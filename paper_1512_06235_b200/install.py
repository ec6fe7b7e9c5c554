"""Wire the B200 path into the reference package at its own function names
(SURVEY.md §8b — the reference has no FFI, so its plugin
surface is the set of module attributes the fine stages call).

    import paper_1512_06235_b200.install as b200
    patched = b200.install()        # the reference's msfm must be importable

Every replaced function keeps the reference signature, defaults and errors and
raises DeviceUnavailableError without the library or a device (no CPU
fallback).  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib

# (reference module, attribute) -> (our module, attribute); modules that bind a
# name at import time (``from .x import f``) are listed with the binding module
_ROUTES = [
    # geometry-aware matching (guided.py:393); densify.py binds it at import
    ("msfm.guided", "guided_match_pair", "guided", "guided_match_pair"),
    ("msfm.densify", "guided_match_pair", "guided", "guided_match_pair"),
    # multi-view DLT triangulation (geometry.py:276)
    ("msfm.geometry", "triangulate_track", "triangulation", "triangulate_track"),
    ("msfm.densify", "triangulate_track", "triangulation", "triangulate_track"),
    # PnP-RANSAC (reconstruct.py:168); localize.py binds it
    ("msfm.reconstruct", "pnp_ransac", "pnp", "pnp_ransac"),
    ("msfm.localize", "pnp_ransac", "pnp", "pnp_ransac"),
    # 3D-2D search and the localization stage (localize.py:99-281)
    ("msfm.localize", "direct_3d2d_search", "localize", "direct_3d2d_search"),
    ("msfm.localize", "ranked_2d2d_search", "localize", "ranked_2d2d_search"),
    ("msfm.localize", "localize_image", "localize", "localize_image"),
    ("msfm.localize", "localize_all", "localize", "localize_all"),
    ("msfm.pipeline", "localize_all", "localize", "localize_all"),
    # coarse unguided matching + two-view geometry (matching.py:116-249, geometry.py:153)
    ("msfm.matching", "match_pair", "coarse", "match_pair"),
    ("msfm.matching", "hybrid_match", "coarse", "hybrid_match"),
    ("msfm.matching", "preemptive_pair_filter", "coarse", "preemptive_pair_filter"),
    ("msfm.matching", "build_coarse_matchgraph", "coarse", "build_coarse_matchgraph"),
    ("msfm.pipeline", "build_coarse_matchgraph", "coarse", "build_coarse_matchgraph"),
    ("msfm.geometry", "estimate_fundamental_ransac", "fundamental", "estimate_fundamental_ransac"),
    ("msfm.matching", "estimate_fundamental_ransac", "fundamental", "estimate_fundamental_ransac"),
    # the batched densification stage (densify.py:168-276)
    ("msfm.densify", "densify_stage", "densify", "densify_stage"),
    ("msfm.pipeline", "densify_stage", "densify", "densify_stage"),
    # the 2-NN index (descriptors.py:35-139); matching.py / localize.py bind it
    ("msfm.descriptors", "two_nearest_bruteforce", "descriptors", "two_nearest_bruteforce"),
    ("msfm.descriptors", "DescriptorIndex", "descriptors", "DescriptorIndex"),
    ("msfm.matching", "DescriptorIndex", "descriptors", "DescriptorIndex"),
    ("msfm.localize", "DescriptorIndex", "descriptors", "DescriptorIndex"),
    # .msft staging (features.py:98-130); FeatureStore.load_dir calls it by name
    ("msfm.features", "load_features", "staging", "load_features"),
    # model snapshots (io.py:51-84) read natively into the arrays the stages consume
    ("msfm.io", "read_model", "model_io", "read_model"),
    ("msfm.cli", "read_model", "model_io", "read_model"),
    # reconstruct.py binds triangulate_track (geometry.py:276) at import
    ("msfm.reconstruct", "triangulate_track", "triangulation", "triangulate_track"),
    # the CLI binds the stage entry points at import (cli.py:20-32): its localize,
    # densify and bench-guided commands run the B200 path too
    ("msfm.cli", "guided_match_pair", "guided", "guided_match_pair"),
    ("msfm.cli", "localize_all", "localize", "localize_all"),
    ("msfm.cli", "densify_stage", "densify", "densify_stage"),
    ("msfm.cli", "build_coarse_matchgraph", "coarse", "build_coarse_matchgraph"),
    ("msfm.cli", "load_features", "staging", "load_features"),
]

_SAVED: dict = {}


def install() -> list:
    """Patch the reference modules; returns the "module.attr" names replaced.
    Names a reference version lacks are skipped (and not returned).  The package's
    value types and errors become the reference's own classes first
    (types.adopt_reference_types), so drop-ins raise msfm.errors.* and return
    msfm.matching.Match / msfm.model.FeatureRef objects."""
    from .types import adopt_reference_types

    adopt_reference_types()
    done = []
    for mod, attr, ours, our_attr in _ROUTES:
        m = importlib.import_module(mod)
        if not hasattr(m, attr):
            continue
        impl = getattr(importlib.import_module(f"{__package__}.{ours}"), our_attr)
        _SAVED.setdefault((mod, attr), getattr(m, attr))
        setattr(m, attr, impl)
        done.append(f"{mod}.{attr}")
    return done


def uninstall() -> None:
    """Restore every attribute install() replaced."""
    for (mod, attr), orig in list(_SAVED.items()):
        setattr(importlib.import_module(mod), attr, orig)
    _SAVED.clear()
