"""Shared fixtures-by-function for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle.oracle import RefInput, RefSession, Restated, have_ref, ref_init_factors  # noqa: F401
from paper_1904_07935_b200 import plnmf as P

# The 20News / TDT2 shapes of BASELINE.json.
NEWS20 = dict(rows=26214, cols=11314, density=1018191 / (26214 * 11314))
TDT2 = dict(rows=36771, cols=10212, density=1323869 / (36771 * 10212))


def instance(rows, cols, density, seed=20):
    m = P.synth_csr(rows, cols, density, seed)
    return m


def bits_equal(a, b) -> bool:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and bool((a.view(np.uint64) == b.view(np.uint64)).all())


def rel_max(ref, other) -> float:
    """factor_deviation (proj/src/metrics.cpp:129-143)."""
    ref, other = np.asarray(ref), np.asarray(other)
    mr = np.abs(ref).max() if ref.size else 0.0
    md = np.abs(ref - other).max() if ref.size else 0.0
    if mr == 0.0:
        return 0.0 if md == 0.0 else np.inf
    return float(md / mr)


def elem_rel(ref, other) -> float:
    """max_i |ref_i - other_i| / |ref_i| over nonzero ref entries."""
    ref, other = np.asarray(ref), np.asarray(other)
    nz = ref != 0
    if not nz.any():
        return float(np.abs(other).max()) if other.size else 0.0
    return float((np.abs(ref - other)[nz] / np.abs(ref[nz])).max())
