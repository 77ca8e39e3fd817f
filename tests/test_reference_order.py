"""Whole-trajectory parity: Math.reference_order against the compiled reference.

The fast path reproduces the reference's per-element order everywhere but
forms two reductions as fixed trees (the W column norms and the error dots).
Math.reference_order forms those in the reference's own order too — serial
for fast-hals (proj/src/hals.cpp:97-100), per-OpenMP-thread chunk partials
for pl-nmf (proj/src/tiled.cpp:103-142) with the reference's team size, and
serial <P,W>, <S,Q> (proj/src/metrics.cpp:104-115) — so a 10-iteration
iterate() is compared BIT FOR BIT with the unmodified reference
(oracle/_ref, run with the same thread count): every trace rel_error, W and
Ht.  That meets BASELINE.json's literal gate (per-iteration error within
1e-5, W/H within 1e-3 after 10 iterations) with zero deviation.
"""
import numpy as np
import pytest

from _helpers import NEWS20, bits_equal, instance
from oracle.oracle import RefInput, have_ref, ref, ref_iterate
from paper_1904_07935_b200 import plnmf as P

A = P.Algorithm
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_ref(), reason="oracle/_ref (the compiled reference) not built")]


def _run_both(m, k, iters, tile, threads, rel_tol=0.0):
    cfg = P.SolverConfig(rank=k, max_iters=iters, rel_tol=rel_tol, tile_size=tile)
    f = P.init_factors(m.rows, m.cols, cfg)
    w0, h0 = f.w.copy(order="F"), f.ht.copy(order="F")
    a = P.InputMatrix(m)
    eng = P.Engine(a, k)
    eng.set_math(P.Math.reference_order)
    eng.set_reference_threads(threads)
    eng.set_factors(f)
    tr = eng.iterate(cfg, A.tiled if tile else A.reference)
    got = eng.get_factors()
    eng.close()

    ra = RefInput(m.rows, m.cols, m.row_ptr, m.col_idx, m.values)
    prev = ref().ref_max_threads()
    ref().ref_set_threads(threads)
    try:
        w, ht, rtr = ref_iterate(ra, w0, h0, k, max_iters=iters, rel_tol=rel_tol, tile=tile, tiled=bool(tile))
    finally:
        ref().ref_set_threads(prev)
    return tr, got, (w, ht, rtr)


def _assert_bitwise(tr, got, refout):
    w, ht, rtr = refout
    assert bits_equal([tr.initial_error], [rtr["initial_error"]]), (tr.initial_error, rtr["initial_error"])
    ref_errs = rtr["records"][:, 1]
    got_errs = np.array([r.rel_error for r in tr.records])
    assert len(got_errs) == len(ref_errs)
    assert [r.iteration for r in tr.records] == [int(x) for x in rtr["records"][:, 0]]
    assert bits_equal(got_errs, ref_errs), np.abs(got_errs - ref_errs).max()
    assert bits_equal(got.ht, ht), np.abs(got.ht - ht).max()
    assert bits_equal(got.w, w), np.abs(got.w - w).max()
    assert tr.update_macs == rtr["update_macs"]


@pytest.mark.parametrize("tile,threads", [(0, 1), (5, 1), (5, 3), (5, 8), (16, 7)])
def test_small_trajectory_bitwise(gpu, tile, threads):
    m = instance(1500, 900, 0.02)
    _assert_bitwise(*_run_both(m, 16, 10, tile, threads))


def test_small_trajectory_stop_rule_bitwise(gpu):
    """Default rel_tol: the stop decision is taken on bit-identical errors, so
    both runs stop at the same iteration."""
    m = instance(800, 500, 0.03)
    tr, got, refout = _run_both(m, 6, 200, 2, 4, rel_tol=1e-4)
    assert len(tr.records) < 200
    _assert_bitwise(tr, got, refout)


@pytest.mark.parametrize("tile", [0, 9])
def test_c1_ten_iterations_bitwise(gpu, tile):
    """BASELINE configs[0] (C1: 20News shape, K=80, 10 iterations), fast-hals
    and pl-nmf at T_auto = 9, the reference on all host cores."""
    m = instance(**NEWS20)
    _assert_bitwise(*_run_both(m, 80, 10, tile, ref().ref_max_threads()))


def test_c2_pl_nmf_ten_iterations_bitwise(gpu):
    """C2 (K=240) pl-nmf at the bench tile T=16: 10 iterations bit for bit."""
    m = instance(**NEWS20)
    _assert_bitwise(*_run_both(m, 240, 10, 16, ref().ref_max_threads()))


def test_c2_fast_hals_ten_iterations_bitwise(gpu):
    """C2 fast-hals (the reference's serial W update: ~5 s/iteration on the CPU)."""
    m = instance(**NEWS20)
    _assert_bitwise(*_run_both(m, 240, 10, 0, 1))
