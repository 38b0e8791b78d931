"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/w1g.h declares, and the host-side logic that
never touches the device (parameter validation, scalar formulas, sharding)
matches the reference."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "w1g.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|void \*|const char \*)\s*\*?\s*(w1g_\w+)\s*\(", txt, re.M)))


def test_header_lists_the_binding():
    from paper_2110_14734_b200 import _lib

    assert header_symbols() == sorted(_lib.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    from paper_2110_14734_b200 import _lib

    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.w1g_version() == 10000


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_2110_14734_b200", "libw1g.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_fused_delta_formula_matches_python():
    # capi.cu computes delta with the same IEEE operation order as
    # condensation.compute_delta; pin the Python side of that equality
    from paper_2110_14734_b200 import condensation, pipeline

    for s in (1.0, 12.0, 40.0, 93.0):
        eps = pipeline.condensation_epsilon(s)
        for L, n in ((949.0501340320344, 200000), (91.27658749087254, 2000), (3.5355, 4)):
            assert condensation.compute_delta(eps, L, n) == 2.0 * eps * L / (math.sqrt(2.0) * n)


def test_params_validation_like_reference():
    from paper_2110_14734_b200 import ApproxParams, CondensationParams

    with pytest.raises(ValueError):
        ApproxParams(s=1.0)
    ApproxParams(s=1.0, best_effort=True)
    with pytest.raises(ValueError):
        ApproxParams(s=0.0, best_effort=True)
    with pytest.raises(ValueError):
        ApproxParams(s=20, delta=-1.0)
    with pytest.raises(ValueError):
        CondensationParams(epsilon=0.5, delta=0.1, k=0.3)
    with pytest.raises(ValueError):
        CondensationParams(epsilon=-1.0, delta=0.1)


def test_error_expression_like_reference():
    from paper_2110_14734_b200 import s_from_error, total_error_factor

    assert total_error_factor(40) == pytest.approx(0.47310, abs=1e-5)
    assert s_from_error(0.5) == 39 and s_from_error(0.2) == 87 and s_from_error(3.4667) == 12


def test_pair_shard_covers_every_pair_once():
    from paper_2110_14734_b200.pipeline import pair_shard

    for n, world in ((64, 8), (7, 3), (2, 4)):
        seen = []
        for r in range(world):
            seen += pair_shard(n, r, world)
        assert sorted(seen) == [(i, j) for i in range(n) for j in range(i + 1, n)]


def test_diagram_validation():
    from paper_2110_14734_b200 import DiagramFormatError, PersistenceDiagram

    with pytest.raises(DiagramFormatError):
        PersistenceDiagram([(1.0, 1.0)])
    with pytest.raises(DiagramFormatError):
        PersistenceDiagram([(0.0, np.inf)])
    assert PersistenceDiagram([(0, 1), (2, 3)]) == PersistenceDiagram([(2, 3), (0, 1)])


# w1flow/__init__.py:10-104 -- every public name of the reference package
REFERENCE_ALL = [
    "ABORTED_STALLING", "ApproxParams", "ArcList", "CondensationParams", "DiagramFormatError", "FlowResult",
    "InfeasibleNetworkError", "NetworkError", "OPTIMAL", "OracleSizeError", "PDPoint", "PersistenceDiagram",
    "PipelineSpec", "PipelineStage", "PlanarIndex", "SplitTree", "SuppliedNodes", "TransshipmentNetwork",
    "WSPairList", "approx_w1", "assemble", "build_network", "build_split_tree", "build_wspd", "compute_delta",
    "count_pairs", "delta_condense", "diagonal_distance", "diagonal_projection", "emit_arcs",
    "exact_w1_bruteforce", "exact_w1_dense", "find_entering_arc", "load_diagram", "nn_search", "parse_diagram",
    "rwmd", "s_from_error", "serialize_diagram", "snap_point", "solve", "total_error_factor", "wcd",
    "well_separated", "write_pairs", "zero_condense",
]


def test_every_reference_name_is_exported():
    import paper_2110_14734_b200 as w

    missing = [n for n in REFERENCE_ALL if not hasattr(w, n)]
    assert not missing, missing


def test_parse_and_serialize_diagram(tmp_path):
    from paper_2110_14734_b200 import DiagramFormatError, load_diagram, parse_diagram, serialize_diagram

    d, dropped = parse_diagram("# comment\n1 2\n\n  3 3 \n1 2\n0.1 0.30000000000000004\n-5e-1 1e2\n")
    assert dropped == 1
    assert d.points.tolist() == [[1.0, 2.0], [1.0, 2.0], [0.1, 0.30000000000000004], [-0.5, 100.0]]
    again, _ = parse_diagram(serialize_diagram(d))
    assert again.points.tobytes() == d.points.tobytes()
    assert serialize_diagram(parse_diagram("")[0]) == ""
    for text, msg in (("1 2 3\n", "line 1: expected two numbers, got 3 tokens"), ("1 x\n", "line 1: non-numeric"),
                      ("\n1 inf\n", "line 2: non-finite"), ("2 1\n", "line 1: death < birth")):
        with pytest.raises(DiagramFormatError, match=msg):
            parse_diagram(text)
    p = tmp_path / "d.txt"
    p.write_text("0 1\n0 1\n")
    d2, n2 = load_diagram(p)
    assert len(d2) == 2 and n2 == 0
    p.write_text("0 1\nbad\n")
    with pytest.raises(DiagramFormatError, match=str(p)):
        load_diagram(p)


def test_pipeline_spec_validation():
    from paper_2110_14734_b200 import PipelineSpec, PipelineStage

    with pytest.raises(ValueError):
        PipelineStage("nope", 1)
    with pytest.raises(ValueError):
        PipelineStage("pdflow", 1)
    with pytest.raises(ValueError):
        PipelineSpec((PipelineStage("wcd", 3), PipelineStage("rwmd", 3), PipelineStage("exact", 1)))
    with pytest.raises(ValueError):
        PipelineSpec((PipelineStage("wcd", 2),))
    PipelineSpec((PipelineStage("wcd", 5), PipelineStage("pdflow", 1, s=4.0)))


def test_reference_suite_plugin_rebinds_the_stage_functions():
    """tools/reference_suite: Option 2 of INTEGRATION.md applied across w1flow."""
    import importlib
    import sys

    from paper_2110_14734_b200 import solver

    try:
        solver.reference_simplex()
    except ImportError:
        pytest.skip("reference package not installed")
    sys.path.insert(0, os.path.join(ROOT, "tools", "reference_suite"))
    try:
        plugin = importlib.import_module("dropin_plugin")
    finally:
        sys.path.pop(0)
    import paper_2110_14734_b200 as d
    import w1flow
    from w1flow import pipeline as rp
    from w1flow import spanner as rs

    original = rs.build_wspd
    try:
        applied = plugin.apply()
        assert rs.build_wspd is d.build_wspd and rp.zero_condense is d.zero_condense
        assert rp.approx_w1 is d.approx_w1 and w1flow.nn_search is d.nn_search
        assert "w1flow.oracle.exact_w1_dense" in applied
    finally:
        plugin.undo()
    assert rs.build_wspd is original
