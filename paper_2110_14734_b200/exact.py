"""Exact W1 for validation (reference: w1flow/oracle.py).

The dense network -- every A-member x B-member arc over the 0-condensed nodes
plus the diagonal arcs, oracle.py:66-93 -- is built on the B200 straight into
CSR order (corpus.cu, w1g_dense_network) and solved by the reference's own
host network simplex, like the sparsified networks.  The brute-force matching
enumeration (oracle.py:33-63, <= 12 points) and the size-guard exception are
the reference's own (re-exported through `solver`).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, solver
from .diagram import SuppliedNodes, load_nodes, zero_condense
from .network import TransshipmentNetwork, fetch_network

BRUTE_FORCE_LIMIT = 12
DENSE_ARC_LIMIT = 10_000_000


def dense_network(nodes: SuppliedNodes, device: int | None = None) -> TransshipmentNetwork:
    """Complete bipartite transshipment network over condensed nodes (oracle.py:66-93)."""
    na = int(np.count_nonzero(np.asarray(nodes.a_mass) > 0))
    nb = int(np.count_nonzero(np.asarray(nodes.b_mass) > 0))
    if na * nb > DENSE_ARC_LIMIT:
        raise solver.reference_attr("OracleSizeError")("dense oracle arc guard exceeded")
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES0, nodes)
    n, m = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("w1g_dense_network", ctypes.byref(n), ctypes.byref(m))
    return fetch_network(ctx, int(n.value), int(m.value))


def exact_w1_nodes(nodes: SuppliedNodes, device: int | None = None) -> float:
    """Exact W1 of the diagrams a condensed node set represents (oracle.py:96-102)."""
    if nodes.points.shape[0] == 0:
        return 0.0
    result = solver.solve(dense_network(nodes, device))
    if result.status != solver.OPTIMAL:
        raise RuntimeError("dense oracle solve did not reach optimality")
    return result.objective


def exact_w1_dense(a, b, device: int | None = None) -> float:
    """Exact W1 via 0-condensation and a dense min-cost flow solve (oracle.py:105-108)."""
    return exact_w1_nodes(zero_condense(a, b, device), device)
