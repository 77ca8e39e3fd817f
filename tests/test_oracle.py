"""The oracle itself (CPU): the C restatement is pinned bit for bit to the
compiled reference (oracle/_ref) on randomized inputs, and the reference's own
known-answer tests (proj/tests/test_engine_*.cpp) hold for the restatement.
"""
import numpy as np
import pytest

from _helpers import Restated as R, bits_equal
from oracle import oracle as O
from paper_1904_07935_b200 import plnmf as P

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("rows,cols,density,k", [(1, 1, 1.0, 1), (50, 40, 0.3, 7), (700, 300, 0.02, 33),
                                                 (2049, 100, 0.05, 16)])
def test_restatement_matches_reference_bitwise(rows, cols, density, k):
    m = P.synth_csr(rows, cols, density, 11)
    rp, ci, val = m.row_ptr, m.col_idx, m.values
    for x, y in zip(O.ref_transpose(rows, cols, rp, ci, val), R.transpose(rows, cols, rp, ci, val)):
        assert (x == y).all()
    w, ht = O.ref_init_factors(rows, cols, k, seed=5)
    assert bits_equal(w, R.init_factors(rows, cols, k, seed=5)[0])
    assert bits_equal(O.ref_spmm(rows, cols, rp, ci, val, ht), R.spmm(rows, cols, rp, ci, val, ht))
    assert bits_equal(O.ref_gram(w), R.gram(w))
    a = O.RefInput(rows, cols, rp, ci, val)
    assert a.norm_sq == R.norm_sq(val)
    nth = O.ref().ref_max_threads()
    for tile in (0, 1, max(1, k // 3), k):
        s = O.RefSession(a, k)
        s.precompute_h(w)
        r_, s_ = s.get("r"), s.get("s")
        ht1 = s.update_h(ht, tile=tile)
        want_h = R.update_tiled(ht, s_, r_, tile, is_w=False)[0] if tile else R.update_h_reference(ht, r_, s_)
        assert bits_equal(ht1, want_h)
        s.precompute_w(ht1)
        p_, q_ = s.get("p"), s.get("q")
        w1 = s.update_w(w, tile=tile)
        want_w, norms = (R.update_tiled(w, q_, p_, tile, is_w=True, nthreads=nth) if tile
                         else R.update_w_reference(w, p_, q_))
        assert bits_equal(w1, want_w)
        assert bits_equal(s.get("column_norms"), norms)


@needs_ref
def test_restatement_error_and_deviation_match_reference():
    m = P.synth_csr(120, 90, 0.1, 3)
    k = 5
    w, ht = R.init_factors(120, 90, k, seed=1)
    a = O.RefInput(120, 90, m.row_ptr, m.col_idx, m.values)
    p = R.spmm(120, 90, m.row_ptr, m.col_idx, m.values, ht)
    q, s = R.gram(ht), R.gram(w)
    out = np.zeros(3)
    O.ref().ref_relative_error_gram(a.norm_sq, O.f64p(O.F(w)), 120, O.f64p(O.F(ht)), 90, k, O.f64p(O.F(p)),
                                    O.f64p(O.F(q)), O.f64p(O.F(s)), O.f64p(out))
    assert bits_equal(out, R.relative_error_gram(a.norm_sq, w, p, q, s))
    d = np.zeros(2)
    O.ref().ref_relative_error_direct(a.h, O.f64p(O.F(w)), O.f64p(O.F(ht)), k, O.f64p(d))
    assert bits_equal(d, R.relative_error_direct_csr(120, 90, m.row_ptr, m.col_idx, m.values, a.norm_sq, w, ht))
    x = np.asfortranarray(np.random.default_rng(0).random((7, 3)))
    y = x + 1e-9
    assert O.ref().ref_factor_deviation(O.f64p(x), O.f64p(y), 7, 3) == R.factor_deviation(x, y)


@needs_ref
@pytest.mark.parametrize("k,t", [(16, 16), (16, 4), (160, 15), (8, 1), (7, 3)])
def test_plan_tiles_matches_reference(k, t):
    plan = P.plan_tiles(k, t)
    assert [(x.begin, x.end) for x in plan.tiles] == O.ref_plan_tiles(k, t)


# ---- the reference's known-answer tests, restated (proj/tests/test_engine_reference.cpp, _tiled.cpp)
def test_kat_update_h_k1_clamp_r():
    """test_engine_reference.cpp:117-129"""
    ht = np.array([[2.0], [3.0], [4.0]], order="F")
    r = np.array([[5.0], [10.0], [15.0]], order="F")
    got = R.update_h_reference(ht, r, np.ones((1, 1), order="F"))
    assert (got == r).all()


def test_kat_negative_r_clamps_to_epsilon():
    """test_engine_reference.cpp:131-144"""
    rng = np.random.default_rng(2)
    ht = np.asfortranarray(rng.uniform(0.1, 1.0, (4, 2)))
    r = np.asfortranarray(-1.0 - (np.arange(4)[:, None] + np.arange(2)[None, :]).astype(float))
    got = R.update_h_reference(ht, r, np.eye(2, order="F"), eps=1e-12)
    assert (got == 1e-12).all()


def test_kat_q_identity_normalises_p():
    """test_engine_reference.cpp:170-190"""
    v, k = 4, 3
    w = np.asfortranarray(1.0 + np.arange(v)[:, None] + np.arange(k)[None, :])
    p = np.asfortranarray(3.0 + 2 * np.arange(v)[:, None] + np.arange(k)[None, :])
    got, _ = R.update_w_reference(w, p, np.eye(k, order="F"))
    want = p / np.sqrt((p ** 2).sum(axis=0))
    assert np.allclose(got, want, rtol=1e-15, atol=0)


def test_kat_dyadic_w_all_tiles_equal_reference():
    """test_engine_tiled.cpp:213-239 (passes in the reference)"""
    v = k = 4
    q = np.ones((k, k), order="F")
    p = np.asfortranarray(np.tile(5.0 - 0.5 * np.arange(k), (v, 1)))
    w0 = np.ones((v, k), order="F")
    ref_w, _ = R.update_w_reference(w0, p, q)
    assert (ref_w == 0.5).all()
    for t in range(1, k + 1):
        assert bits_equal(R.update_tiled(w0, q, p, t, is_w=True)[0], ref_w)


def test_kat_macs_parity_formula():
    """test_engine_tiled.cpp:341-363: tiled and reference MAC counts agree."""
    for n, k in [(7, 5), (30, 12)]:
        ref = n * k * k + n * k * (k + 3)  # update_h + update_w (hals.cpp:70,105)
        for t in range(1, k + 1):
            tiled = 0
            for is_w in (False, True):
                m = n * k if is_w else 0
                for b in range(0, k, t):
                    e = min(k, b + t)
                    wdt = e - b
                    m += n * wdt * b + n * wdt * wdt + (2 * n * wdt if is_w else 0) + n * wdt * (k - e)
                tiled += m
            assert tiled == ref


@pytest.mark.parametrize("rows,cols,density,seed", [(0, 5, 0.5, 1), (1, 1, 1.0, 2), (300, 200, 0.05, 20),
                                                    (5000, 3000, 0.003, 7), (64, 50, 1.0, 3)])
def test_oracle_generator_matches_engine_generator(rows, cols, density, seed):
    """oracle/synth.c (used by bench.py's reference arm so that it never loads
    the engine) produces exactly the engine's plnmf_synth_csr stream."""
    rp, ci, val = O.synth_csr(rows, cols, density, seed)
    m = P.synth_csr(rows, cols, density, seed)
    assert (rp == m.row_ptr).all() and (ci == m.col_idx).all() and bits_equal(val, m.values)
