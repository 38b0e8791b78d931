"""Access to the reference's own host min-cost-flow solver.

The network simplex (w1flow/simplex.py) is outside the accelerated path by
design (BASELINE.json north star): approx_w1 hands the device-built network
to the reference's `simplex.solve` unchanged.  It is looked up from an
installed `w1flow` package, or from the repo-local install under
baseline/_ref (python -m pip install --target baseline/_ref <reference>).
"""

from __future__ import annotations

import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_LOCAL = os.path.join(_ROOT, "baseline", "_ref")

_simplex = None


def reference_simplex():
    """The reference's `w1flow.simplex` module (raises ImportError if absent)."""
    global _simplex
    if _simplex is None:
        os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(_ROOT, "build", "numba_cache"))
        try:
            from w1flow import simplex  # type: ignore
        except ImportError:
            if os.path.isdir(_LOCAL) and _LOCAL not in sys.path:
                sys.path.append(_LOCAL)
            try:
                from w1flow import simplex  # type: ignore
            except ImportError as exc:
                raise ImportError(
                    "approx_w1 needs the reference's host solver (w1flow.simplex); install the "
                    "reference package or populate baseline/_ref"
                ) from exc
        _simplex = simplex
    return _simplex


# names of the reference package that are outside the accelerated path and are
# re-exported unchanged (host solver types, the brute-force oracle, cKDTree index)
REFERENCE_EXPORTS = {
    "FlowResult": "simplex",
    "InfeasibleNetworkError": "simplex",
    "find_entering_arc": "simplex",
    "OracleSizeError": "oracle",
    "exact_w1_bruteforce": "oracle",
    "PlanarIndex": "lower_bound",
}


def reference_attr(name: str):
    """`name` from the reference module REFERENCE_EXPORTS assigns it to."""
    import importlib

    reference_simplex()  # puts the reference on sys.path if it comes from baseline/_ref
    return getattr(importlib.import_module("w1flow." + REFERENCE_EXPORTS[name]), name)


def solve(network, *args, **kwargs):
    """simplex.solve(network, ...) of the reference (simplex.py:339-395), every argument forwarded."""
    return reference_simplex().solve(network, *args, **kwargs)


OPTIMAL = "optimal"
ABORTED_STALLING = "aborted_stalling"
