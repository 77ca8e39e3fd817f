"""Parity at every BASELINE.json config, on the GPU.

C1/C2 are covered bit for bit by test_reference_order.py (10-iteration
trajectories) and test_gpu_parity.py (one-step from a reference state).  Here:

  C3  TDT2 shape, K = 480.  A 10-iteration pl-nmf trajectory at T_auto = 22 in
      Math.reference_order, bit-identical to the compiled reference; then, from
      that well-conditioned shared state, one production (Math.exact)
      iteration at T = 22 and at the GPU tile selector's T = 16 against the
      reference's own one iteration: products and Ht bitwise, W within 1e-10
      (only the column-norm summation order differs).  T = 22 at 249 rows per
      SM runs the persistent W kernel with nothing staged (plan 2), the
      instantiation the planner picks for this shape.
  C4  dense 20K x 20K, K = 160 (bench_updates' dense U(0, 1) shape,
      proj/bench/bench_updates.cpp:31-38; numpy-seeded values): one full
      iterate() step bit-identical to the reference in Math.reference_order,
      and the production path's products / Ht bitwise, W within 1e-10.
  C5  2M x 1M, ~1e9 nonzeros, K = 256 on one GPU, generated on the device:
      one iteration, checked on sampled rows against the oracle — R, P and
      the H update bitwise — plus the unit-norm / floor invariants of W
      (proj/tests/acceptance.cpp:105-156) and a finite error.
"""
import time

import numpy as np
import pytest

from _helpers import TDT2, bits_equal, instance, rel_max
from oracle.oracle import RefInput, RefSession, Restated as R, have_ref, ref, ref_iterate
from paper_1904_07935_b200 import plnmf as P

A = P.Algorithm
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_ref(), reason="oracle/_ref (the compiled reference) not built")]


def _ref_threads(n):
    prev = ref().ref_max_threads()
    ref().ref_set_threads(n)
    return prev


# ------------------------------------------------------------------------------ generator
@pytest.mark.parametrize("rows,cols,density,seed", [(1, 1, 1.0, 2), (300, 200, 0.05, 20), (64, 50, 1.0, 3),
                                                    (5000, 3000, 0.003, 7), (26214, 11314, 1018191 / (26214 * 11314), 20)])
def test_device_generator_matches_host_generator(gpu, rows, cols, density, seed):
    eng = P.Engine.synthetic(rows, cols, density, seed, rank=2)
    got = eng.get_csr()
    m = P.synth_csr(rows, cols, density, seed)
    assert (got.row_ptr == m.row_ptr).all() and (got.col_idx == m.col_idx).all()
    assert bits_equal(got.values, m.values)
    assert eng.norm_sq == R.norm_sq(m.values)  # serial, input_matrix.cpp:15-20


# ------------------------------------------------------------------------------ C3
def test_c3_tdt2_k480(gpu):
    k = 480
    m = instance(**TDT2)
    a = P.InputMatrix(m)
    nth = ref().ref_max_threads()
    cfg = P.SolverConfig(rank=k, max_iters=10, rel_tol=0.0, tile_size=22)
    f = P.init_factors(m.rows, m.cols, cfg)
    eng = P.Engine(a, k)
    eng.set_math(P.Math.reference_order)
    eng.set_reference_threads(nth)
    eng.set_factors(f)
    tr = eng.iterate(cfg, A.tiled)
    state = eng.get_factors()
    ra = RefInput(m.rows, m.cols, m.row_ptr, m.col_idx, m.values)
    w, ht, rtr = ref_iterate(ra, f.w, f.ht, k, max_iters=10, rel_tol=0.0, tile=22, tiled=True)
    assert bits_equal(state.w, w) and bits_equal(state.ht, ht)
    assert bits_equal([r.rel_error for r in tr.records], rtr["records"][:, 1])

    # one production iteration from the shared iteration-10 state
    eng.set_math(P.Math.exact)
    ses = RefSession(ra, k)
    for tile in (22, 16):
        eng.set_factors(P.FactorPair(w, ht))
        c = P.SolverConfig(rank=k, tile_size=tile)
        eng.precompute_h_products()
        assert bits_equal(eng.get_product("r"), R.spmm(*_at(m), w))
        eng.update_h(c, A.tiled)
        eng.precompute_w_products()
        eng.update_w(c, A.tiled)
        if tile == 22:  # K=480, 249 rows per SM: the panel does not fit, the streaming W kernel
            assert eng.stats()["w_plan"] == 3
        rep = eng.evaluate_error()
        got = eng.get_factors()
        w1, ht1 = ses.one_iteration(w, ht, tile=tile)
        assert bits_equal(got.ht, ht1)
        assert bits_equal(eng.get_product("p"), ses.get("p"))
        assert rel_max(w1, got.w) <= 1e-10
        e1 = R.relative_error_gram(R.norm_sq(m.values), w1, ses.get("p"), ses.get("q"), R.gram(w1))[1]
        assert abs(rep.relative - e1) <= 1e-12 * e1


def _at(m):
    trp, tci, tval = R.transpose(m.rows, m.cols, m.row_ptr, m.col_idx, m.values)
    return m.cols, m.rows, trp, tci, tval


# ------------------------------------------------------------------------------ C4
def test_c4_dense_20k_k160(gpu):
    v = d = 20000
    k, tile = 160, 13
    rng = np.random.default_rng(4242)
    dense = np.asfortranarray(rng.uniform(0.0, 1.0, (v, d)))
    a = P.InputMatrix(dense)
    cfg = P.SolverConfig(rank=k, max_iters=1, rel_tol=0.0, tile_size=tile)
    f = P.init_factors(v, d, cfg)
    nth = ref().ref_max_threads()
    ra = RefInput(v, d, dense=dense)
    w, ht, rtr = ref_iterate(ra, f.w, f.ht, k, max_iters=1, rel_tol=0.0, tile=tile, tiled=True)

    eng = P.Engine(a, k)
    eng.set_math(P.Math.reference_order)
    eng.set_reference_threads(nth)
    eng.set_factors(f)
    tr = eng.iterate(cfg, A.tiled)
    got = eng.get_factors()
    assert bits_equal(got.ht, ht) and bits_equal(got.w, w)
    assert bits_equal([tr.initial_error, tr.records[0].rel_error], [rtr["initial_error"], rtr["records"][0, 1]])

    eng.set_math(P.Math.exact)
    eng.set_factors(f)
    tr2 = eng.iterate(cfg, A.tiled)
    got2 = eng.get_factors()
    assert bits_equal(got2.ht, ht)
    assert rel_max(w, got2.w) <= 1e-10
    assert abs(tr2.records[0].rel_error - rtr["records"][0, 1]) <= 1e-12 * rtr["records"][0, 1]

    # the tensor-core products (Ozaki u8 tcgen05, Math.tensor) against the exact ones
    # (bit-identical to the reference's gemm) on the reference's iteration-1 state
    exact = {}
    for math in (P.Math.exact, P.Math.tensor):
        eng.set_math(math)
        eng.set_factors(P.FactorPair(w, ht))
        eng.precompute_h_products()
        eng.precompute_w_products()
        exact[math] = (eng.get_product("r"), eng.get_product("p"))
    # the Ozaki bound (csrc/ozaki.cu): |err(i,j)| <= n 2^-46 sa(i) sb(j), sa/sb the row
    # maxima of the left operand and the column maxima of the right one, n = 20,000; the
    # exact products carry their own sequential-sum rounding (1e-13 relative covers it)
    bounds = (np.outer(dense.max(axis=0), w.max(axis=0)), np.outer(dense.max(axis=1), ht.max(axis=0)))
    for a0, a1, bnd in zip(exact[P.Math.exact], exact[P.Math.tensor], bounds):
        assert np.all(np.abs(a1 - a0) <= v * 2.0 ** -46 * bnd + 1e-13 * np.abs(a0))


# ------------------------------------------------------------------------------ C5
def _compact(csr, fetch):
    """(rows, cols, rp, ci, val) of csr with its columns renumbered onto the
    distinct columns it touches, and those operand rows fetched (col-major)."""
    uniq = np.unique(csr.col_idx)
    ci = np.searchsorted(uniq, csr.col_idx).astype(np.int64)
    x = np.asfortranarray(fetch(uniq))
    return (csr.rows, len(uniq), csr.row_ptr, ci, csr.values), x


def test_c5_large_one_gpu(gpu):
    V, D, k, tile = 2_000_000, 1_000_000, 256, 16
    t0 = time.perf_counter()
    eng = P.Engine.synthetic(V, D, 5e-4, 20, rank=k)
    t_gen = time.perf_counter() - t0
    assert 0.99e9 < eng.nnz < 1.01e9
    cfg = P.SolverConfig(rank=k, tile_size=tile)
    eng.init_factors(cfg)
    rng = np.random.default_rng(0)
    hs = np.sort(rng.choice(D, 48, replace=False))
    vs = np.sort(rng.choice(V, 48, replace=False))
    ht0 = eng.get_rows("ht", hs)

    eng.precompute_h_products()
    at_rows = eng.get_csr_rows(hs, transposed=True)
    (args, wx) = _compact(at_rows, lambda u: eng.get_rows("w", u))
    assert bits_equal(eng.get_rows("r", hs), R.spmm(*args, wx))
    s = eng.get_product("s")
    assert bits_equal(s, s.T)

    eng.update_h(cfg, A.tiled)
    ht1_ref, _ = R.update_tiled(np.asfortranarray(ht0), s, np.asfortranarray(eng.get_rows("r", hs)), tile,
                                is_w=False)
    assert bits_equal(eng.get_rows("ht", hs), ht1_ref)

    eng.precompute_w_products()
    a_rows = eng.get_csr_rows(vs)
    (args, hx) = _compact(a_rows, lambda u: eng.get_rows("ht", u))
    assert bits_equal(eng.get_rows("p", vs), R.spmm(*args, hx))

    eng.update_w(cfg, A.tiled)
    assert eng.stats()["w_plan"] == 3  # V/SM rows exceed the persistent kernel: streaming
    norms = eng.get_product("column_norms")
    assert np.isfinite(norms).all() and (norms > 0).all()
    w1 = eng.get_rows("w", vs)
    assert w1.min() >= cfg.epsilon
    rep = eng.evaluate_error()  # leaves S = gram(W): its diagonal holds the squared column norms
    assert np.isfinite(rep.relative) and 0.0 < rep.relative < 2.0  # iteration 1 from the seed: ~1
    assert np.abs(np.diag(eng.get_product("s")) - 1.0).max() <= 1e-12  # unit columns (acceptance.cpp:105-156)
    ms = eng.run_iterations(P.SolverConfig(rank=k, tile_size=tile), A.tiled, 1)
    print(f"C5 on one GPU: nnz {eng.nnz}, device generation {t_gen:.1f} s, {ms:.1f} ms per FAST-HALS iteration, "
          f"phases {eng.phase_ms()}")
