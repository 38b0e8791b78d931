"""pytest plugin: run the reference's own test suite against the drop-in.

Loaded with `-p dropin_plugin` before the reference tests are collected, it
applies INTEGRATION.md's Option 2 across the whole reference package: every
public name of w1flow's diagram / condensation / lower_bound / spanner /
network / oracle / pipeline modules that the drop-in provides is rebound to
the drop-in's object -- in the module itself (so the reference's own code,
which looks those names up as module globals, calls the B200 path too), in
the package namespace, and in w1flow.pipeline's imported stage names (the
ones approx_w1 / nn_search bind at import, pipeline.py:17-23).  Test modules
imported afterwards (`from w1flow.spanner import build_wspd`) receive the
drop-in's functions.  What stays the reference's own: the host simplex
(w1flow.simplex), the brute-force matching oracle, PlanarIndex (cKDTree),
the synthetic generator and the CLI's argument handling.
"""

from __future__ import annotations

import importlib
import os

PATCHED = {
    "diagram": ["PersistenceDiagram", "PDPoint", "DiagramFormatError", "SuppliedNodes", "zero_condense",
                "parse_diagram", "serialize_diagram", "load_diagram", "diagonal_distance", "diagonal_projection",
                "diagonal_distances", "diagonal_projections"],
    "condensation": ["CondensationParams", "compute_delta", "delta_condense", "snap_points", "snap_point"],
    "lower_bound": ["rwmd", "wcd"],
    "spanner": ["SplitTree", "WSPairList", "ArcList", "build_split_tree", "build_wspd", "count_pairs",
                "write_pairs", "emit_arcs", "abar_index", "bbar_index", "well_separated"],
    "network": ["NetworkError", "TransshipmentNetwork", "assemble", "build_network"],
    "oracle": ["dense_network", "exact_w1_nodes", "exact_w1_dense"],
    "pipeline": ["ApproxParams", "ApproxDiagnostics", "approx_w1", "nn_search", "PipelineSpec", "PipelineStage",
                 "condensation_epsilon", "total_error_factor", "s_from_error",
                 # stage names pipeline.py imports (pipeline.py:18-23)
                 "CondensationParams", "compute_delta", "delta_condense", "PersistenceDiagram", "zero_condense",
                 "rwmd", "wcd", "assemble", "exact_w1_dense", "build_split_tree", "build_wspd", "emit_arcs"],
}
# modules that import the names above at import time (pkg/src/w1flow/*.py `from .x import y`)
IMPORTERS = ["lower_bound", "spanner", "network", "oracle", "condensation", "simplex", "synth"]

APPLIED: list[str] = []
_SAVED: list[tuple[object, str, object]] = []  # (module, name, original) for undo()


def _rebind(mod, nm, obj):
    _SAVED.append((mod, nm, getattr(mod, nm, None)))
    setattr(mod, nm, obj)


def _dropin_obj(name):
    import paper_2110_14734_b200 as d
    from paper_2110_14734_b200 import exact, spanner

    for mod in (d, spanner, exact):
        if hasattr(mod, name):
            return getattr(mod, name)
    raise AttributeError(name)


def apply():
    import w1flow

    if APPLIED:
        return APPLIED
    for modname, names in PATCHED.items():
        mod = importlib.import_module("w1flow." + modname)
        for nm in names:
            obj = _dropin_obj(nm)
            _rebind(mod, nm, obj)
            if hasattr(w1flow, nm):
                _rebind(w1flow, nm, obj)
            APPLIED.append(f"w1flow.{modname}.{nm}")
    # the same names bound inside the other reference modules (from .diagram import ...)
    every = {nm for names in PATCHED.values() for nm in names}
    for modname in IMPORTERS:
        try:
            mod = importlib.import_module("w1flow." + modname)
        except ImportError:
            continue
        for nm in every:
            if nm in vars(mod) and getattr(mod, nm) is not _dropin_obj(nm):
                _rebind(mod, nm, _dropin_obj(nm))
                APPLIED.append(f"w1flow.{modname}.{nm}")
    return APPLIED


def undo():
    """Restore the reference's own objects (for in-process checks of apply())."""
    while _SAVED:
        mod, nm, orig = _SAVED.pop()
        setattr(mod, nm, orig)
    APPLIED.clear()


def pytest_configure(config):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    apply()


def pytest_report_header(config):
    return f"drop-in: {len(APPLIED)} reference names rebound to paper_2110_14734_b200"
