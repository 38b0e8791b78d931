"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the C oracle (w1oracle.c).

The oracle is a scalar CPU restatement of the reference sparsify front-end
(/root/reference/pkg/src/w1flow, pipeline.py:105-130).  It is the checker
for the CUDA path and the CPU baseline bench.py reports; only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import it.  The product package (paper_2110_14734_b200) never does.

Parity of this restatement against the live reference is pinned by
tests/test_oracle_golden.py (committed fixtures from tests/golden/make_golden.py)
and tests/test_oracle_vs_reference.py (live import, this container only).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "w1oracle.c")
LIB = os.path.join(HERE, "libw1oracle.so")

_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_f64 = ctypes.c_double

SQRT2 = math.sqrt(2.0)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FP contraction, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = [
            "gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
            "-fno-fast-math", "-o", LIB, SRC, "-lm",
        ]
        subprocess.check_call(cmd)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.orc_pairwise_sum.restype = _f64
        L.orc_pairwise_sum.argtypes = [_F64P, _i64]
        L.orc_zero_condense.restype = _i64
        L.orc_zero_condense.argtypes = [_F64P, _i64, _F64P, _i64, _F64P, _I64P, _I64P]
        L.orc_rwmd.restype = _f64
        L.orc_rwmd.argtypes = [_F64P, _I64P, _I64P, _i64, _F64P, _F64P]
        L.orc_rwmd_best.restype = _i64
        L.orc_rwmd_best.argtypes = [_F64P, _I64P, _I64P, _i64, _F64P]
        L.orc_snap_cells.restype = ctypes.c_int
        L.orc_snap_cells.argtypes = [_F64P, _i64, _f64, _I64P]
        L.orc_delta_condense.restype = _i64
        L.orc_delta_condense.argtypes = [_F64P, _I64P, _I64P, _i64, _f64, _f64, ctypes.c_uint64,
                                         _F64P, _I64P, _I64P]
        L.orc_split_tree.restype = ctypes.c_int
        L.orc_split_tree.argtypes = [_F64P, _i64, _I64P, _I64P, _F64P, _I64P, _I64P]
        L.orc_wspd_count.restype = _i64
        L.orc_wspd_count.argtypes = [_I64P, _I64P, _F64P, _i64, _f64, _I64P]
        L.orc_wspd_write.restype = ctypes.c_int
        L.orc_wspd_write.argtypes = [_I64P, _I64P, _F64P, _i64, _f64, _I64P, _I64P, _I64P]
        L.orc_hypot_port.restype = _f64
        L.orc_hypot_port.argtypes = [_f64, _f64]
        L.orc_hypot_libm.restype = _f64
        L.orc_hypot_libm.argtypes = [_f64, _f64]
        L.orc_emit_arcs.restype = _i64
        L.orc_emit_arcs.argtypes = [_I64P, _i64, _F64P, _I64P, _I64P, _i64, _I64P, _I64P, _F64P]
        L.orc_build_network.restype = _i64
        L.orc_build_network.argtypes = [_i64, _I64P, _I64P, _I64P, _F64P, _i64, _I64P, _I64P,
                                        _F64P, _I64P]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------- stages


@dataclass
class Nodes:
    points: np.ndarray
    a_mass: np.ndarray
    b_mass: np.ndarray
    abar_supply: int
    bbar_supply: int

    def n_points(self) -> int:
        return int(self.a_mass.sum() + self.b_mass.sum())


def pairwise_sum(v) -> float:
    v = _f(v)
    return float(lib().orc_pairwise_sum(_p(v, _F64P), v.shape[0]))


def zero_condense(a_pts, b_pts) -> Nodes:
    """diagram.py:190-208"""
    a = _f(a_pts).reshape(-1, 2)
    b = _f(b_pts).reshape(-1, 2)
    n = a.shape[0] + b.shape[0]
    pts = np.empty((max(n, 0), 2))
    am = np.empty(n, np.int64)
    bm = np.empty(n, np.int64)
    k = lib().orc_zero_condense(_p(a, _F64P), a.shape[0], _p(b, _F64P), b.shape[0],
                                _p(pts, _F64P), _p(am, _I64P), _p(bm, _I64P))
    if k < 0:
        raise MemoryError("oracle zero_condense failed")
    return Nodes(pts[:k].copy(), am[:k].copy(), bm[:k].copy(), -a.shape[0], b.shape[0])


def rwmd(nodes: Nodes) -> tuple[float, float, float]:
    """lower_bound.py:61-75 -> (L, L_A, L_B)"""
    pts = _f(nodes.points).reshape(-1, 2)
    am, bm = _i(nodes.a_mass), _i(nodes.b_mass)
    la, lb = _f64(), _f64()
    L = lib().orc_rwmd(_p(pts, _F64P), _p(am, _I64P), _p(bm, _I64P), pts.shape[0],
                       ctypes.byref(la), ctypes.byref(lb))
    return float(L), la.value, lb.value


def rwmd_best(nodes: Nodes, side: str) -> np.ndarray:
    """per-source min(nn distance, diagonal distance), sources in node order"""
    pts = _f(nodes.points).reshape(-1, 2)
    am, bm = _i(nodes.a_mass), _i(nodes.b_mass)
    src, dst = (am, bm) if side == "a" else (bm, am)
    out = np.empty(int((src > 0).sum()))
    lib().orc_rwmd_best(_p(pts, _F64P), _p(src, _I64P), _p(dst, _I64P), pts.shape[0], _p(out, _F64P))
    return out


def snap_cells(points, pitch: float) -> np.ndarray:
    pts = _f(points).reshape(-1, 2)
    cells = np.empty_like(pts, dtype=np.int64)
    rc = lib().orc_snap_cells(_p(pts, _F64P), pts.shape[0], pitch, _p(cells, _I64P))
    if rc != 0:
        raise ValueError("lattice pitch too small for the coordinate range")
    return cells


def delta_condense(nodes: Nodes, delta: float, k: float = 0.99, seed: int = 0) -> Nodes:
    """condensation.py:105-124 (pitch and half_width computed as the reference does)"""
    if delta == 0.0 or nodes.points.shape[0] == 0:
        return nodes
    pitch = k * delta
    half_width = (1.0 - k) * delta / 2.0
    pts = _f(nodes.points).reshape(-1, 2)
    am, bm = _i(nodes.a_mass), _i(nodes.b_mass)
    K = pts.shape[0]
    opts = np.empty((K, 2))
    oam = np.empty(K, np.int64)
    obm = np.empty(K, np.int64)
    kk = lib().orc_delta_condense(_p(pts, _F64P), _p(am, _I64P), _p(bm, _I64P), K, pitch,
                                  half_width, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
                                  _p(opts, _F64P), _p(oam, _I64P), _p(obm, _I64P))
    if kk == -3:
        raise ValueError("lattice pitch too small for the coordinate range")
    if kk < 0:
        raise MemoryError("oracle delta_condense failed")
    return Nodes(opts[:kk].copy(), oam[:kk].copy(), obm[:kk].copy(), nodes.abar_supply,
                 nodes.bbar_supply)


@dataclass
class Tree:
    points: np.ndarray
    left: np.ndarray
    right: np.ndarray
    bbox: np.ndarray
    rep: np.ndarray
    size: np.ndarray
    root: int

    @property
    def n_nodes(self) -> int:
        return self.left.shape[0]


def split_tree(points) -> Tree:
    """spanner.py:96-159"""
    pts = _f(points).reshape(-1, 2)
    n = pts.shape[0]
    nn = max(2 * n - 1, 0)
    left = np.empty(nn, np.int64)
    right = np.empty(nn, np.int64)
    bbox = np.empty((nn, 4))
    rep = np.empty(nn, np.int64)
    size = np.empty(nn, np.int64)
    rc = lib().orc_split_tree(_p(pts, _F64P), n, _p(left, _I64P), _p(right, _I64P),
                              _p(bbox, _F64P), _p(rep, _I64P), _p(size, _I64P))
    if rc == -2:
        raise ValueError("split tree input contains duplicate points")
    if rc != 0:
        raise MemoryError("oracle split tree failed")
    return Tree(pts, left, right, bbox, rep, size, 0 if n else -1)


def wspd(tree: Tree, s: float) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """spanner.py:263-307 -> (counts per internal node, node_pairs (P,2), indices (P,2))"""
    if s <= 0:
        raise ValueError("s must be positive")
    nn = tree.n_nodes
    counts = np.zeros(nn, np.int64)
    if nn == 0:
        e = np.empty((0, 2), np.int64)
        return counts[:0], e, e.copy()
    L = lib()
    total = L.orc_wspd_count(_p(tree.left, _I64P), _p(tree.right, _I64P), _p(tree.bbox, _F64P),
                             nn, float(s), _p(counts, _I64P))
    internal = np.flatnonzero(tree.left >= 0)
    offsets = np.zeros(nn, np.int64)
    ci = counts[internal]
    offsets[internal] = np.concatenate([[0], np.cumsum(ci)])[:-1]
    pairs = np.empty((total, 2), np.int64)
    rc = L.orc_wspd_write(_p(tree.left, _I64P), _p(tree.right, _I64P), _p(tree.bbox, _F64P), nn,
                          float(s), _p(counts, _I64P), _p(offsets, _I64P), _p(pairs, _I64P))
    if rc != 0:
        raise AssertionError("WSPD write pass disagrees with counted offsets")
    indices = tree.rep[pairs] if total else np.empty((0, 2), np.int64)
    return ci, pairs, indices


def hypot_port(x: float, y: float) -> float:
    return float(lib().orc_hypot_port(x, y))


def hypot_libm(x: float, y: float) -> float:
    return float(lib().orc_hypot_libm(x, y))


def emit_arcs(indices, nodes: Nodes):
    """spanner.py:310-337 -> (tails, heads, costs) in reference arc order"""
    idx = _i(indices).reshape(-1, 2)
    pts = _f(nodes.points).reshape(-1, 2)
    am, bm = _i(nodes.a_mass), _i(nodes.b_mass)
    P, K = idx.shape[0], pts.shape[0]
    M = 2 * P + int((am > 0).sum()) + int((bm > 0).sum()) + 1
    t = np.empty(M, np.int64)
    h = np.empty(M, np.int64)
    c = np.empty(M)
    m = lib().orc_emit_arcs(_p(idx, _I64P), P, _p(pts, _F64P), _p(am, _I64P), _p(bm, _I64P), K,
                            _p(t, _I64P), _p(h, _I64P), _p(c, _F64P))
    assert m == M
    return t, h, c


_NET_ERRORS = {
    -10: "unbalanced supplies",
    -11: "arc endpoint out of range",
    -12: "self-loop arc",
    -13: "non-finite arc cost",
    -14: "negative arc cost",
}


@dataclass
class Network:
    node_count: int
    supplies: np.ndarray
    tails: np.ndarray
    heads: np.ndarray
    costs: np.ndarray
    row_offsets: np.ndarray

    @property
    def arc_count(self) -> int:
        return self.tails.shape[0]


def build_network(supplies, tails, heads, costs) -> Network:
    """network.py:44-85"""
    sup = _i(supplies)
    t, h, c = _i(tails), _i(heads), _f(costs)
    n, m = sup.shape[0], t.shape[0]
    ot = np.empty(m, np.int64)
    oh = np.empty(m, np.int64)
    oc = np.empty(m)
    ro = np.empty(n + 1, np.int64)
    mm = lib().orc_build_network(n, _p(sup, _I64P), _p(t, _I64P), _p(h, _I64P), _p(c, _F64P), m,
                                 _p(ot, _I64P), _p(oh, _I64P), _p(oc, _F64P), _p(ro, _I64P))
    if mm < 0:
        raise ValueError(_NET_ERRORS.get(int(mm), "oracle build_network failed"))
    return Network(n, sup, ot[:mm].copy(), oh[:mm].copy(), oc[:mm].copy(), ro)


def assemble(nodes: Nodes, t, h, c) -> Network:
    """network.py:88-93"""
    sup = np.concatenate([nodes.a_mass - nodes.b_mass, [nodes.abar_supply, nodes.bbar_supply]])
    return build_network(sup.astype(np.int64), t, h, c)


# ------------------------------------------------------------ the chain


def condensation_epsilon(s: float) -> float:
    """pipeline.py:67-69"""
    return 8.0 / (s - 4.0) if s >= 12 else 1.0


def compute_delta(epsilon: float, lower_bound: float, n_points: int) -> float:
    """condensation.py:47-59"""
    return 2.0 * epsilon * lower_bound / (SQRT2 * n_points)


@dataclass
class FrontEnd:
    nodes0: Nodes
    lower_bound: float
    delta: float
    nodes: Nodes
    tree: Tree | None
    node_pairs: np.ndarray | None
    network: Network | None
    short_circuit: bool


def front_end(a_pts, b_pts, s: float, delta: float | None = None, k: float = 0.99,
              seed: int = 0, use_condensation: bool = True) -> FrontEnd:
    """pipeline.py:105-130 (approx_w1 up to the solve).  delta=None derives it
    from the RWMD bound as the reference does (pipeline.py:116-122); a float
    fixes it (the chain of tests/test_acceptance.py:224-237 with a given delta)."""
    nodes0 = zero_condense(a_pts, b_pts)
    if nodes0.points.shape[0] == 0 or np.array_equal(nodes0.a_mass, nodes0.b_mass):
        return FrontEnd(nodes0, 0.0, 0.0, nodes0, None, None, None, True)
    L, _, _ = rwmd(nodes0)
    nodes = nodes0
    d = 0.0
    if use_condensation and L > 0.0:
        d = compute_delta(condensation_epsilon(s), L, nodes0.n_points()) if delta is None else delta
        if d > 0.0:
            nodes = delta_condense(nodes0, d, k, seed)
    tree = split_tree(nodes.points)
    _, node_pairs, indices = wspd(tree, s)
    t, h, c = emit_arcs(indices, nodes)
    net = assemble(nodes, t, h, c)
    return FrontEnd(nodes0, L, d, nodes, tree, node_pairs, net, False)
