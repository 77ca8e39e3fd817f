"""GPU parity tests (P0-P3 of SURVEY.md 8(c)) — the CUDA engine through its C-ABI
against the oracle (the C restatement, itself pinned bit-for-bit to the
compiled reference in test_oracle.py).

Bit-exactness is asserted wherever the engine and the reference share an
operation order (Math.exact): SpMM, Gram, both H updates, phase A.  The W
updates differ only in how the per-column sum of squares is reduced (the
reference: serial or per-OpenMP-thread partials; the engine: a fixed
grid-wide tree), so W is held to 1e-12 relative (measured: ~1e-15).
"""
import numpy as np
import pytest

from _helpers import NEWS20, Restated as R, bits_equal, elem_rel, instance, rel_max
from paper_1904_07935_b200 import plnmf as P

pytestmark = pytest.mark.gpu

A = P.Algorithm


def make(rows, cols, density, k, seed=20, fseed=0):
    m = instance(rows, cols, density, seed)
    a = P.InputMatrix(m)
    eng = P.Engine(a, k)
    cfg = P.SolverConfig(rank=k, seed=fseed)
    f = P.init_factors(rows, cols, cfg)
    eng.set_factors(f)
    return m, eng, f


def ref_at(m):
    trp, tci, tval = R.transpose(m.rows, m.cols, m.row_ptr, m.col_idx, m.values)
    return trp, tci, tval


@pytest.mark.parametrize("k", [1, 7, 37, 80, 240, 300])
def test_spmm_both_directions_bitwise(gpu, k):
    m, eng, f = make(3000, 1500, 0.01, k)
    eng.precompute_w_products()
    eng.precompute_h_products()
    p_ref = R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, f.ht)
    trp, tci, tval = ref_at(m)
    r_ref = R.spmm(m.cols, m.rows, trp, tci, tval, f.w)
    assert bits_equal(eng.get_product("p"), p_ref)
    assert bits_equal(eng.get_product("r"), r_ref)


@pytest.mark.parametrize("k,block", [(2, 1), (24, 37), (240, 100), (256, 977), (64, 1499), (30, 3000)])
def test_spmm_column_blocked_bitwise(gpu, k, block):
    """The column-blocked SpMM (operands beyond L2, spmm.cu) carries each output's
    running sum through y from block to block: bit-identical to the oracle for
    any block size, including blocks a row has no entries in and empty rows."""
    m, eng, f = make(3000, 1500, 0.01, k)
    rp = m.row_ptr.copy()
    eng.force_spmm_blocks(block)
    eng.precompute_w_products()
    eng.precompute_h_products()
    trp, tci, tval = ref_at(m)
    assert bits_equal(eng.get_product("p"), R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, f.ht))
    assert bits_equal(eng.get_product("r"), R.spmm(m.cols, m.rows, trp, tci, tval, f.w))
    assert np.array_equal(rp, m.row_ptr)


@pytest.mark.parametrize("n", [1, 2, 3, 2047, 2048, 2049, 5001])
@pytest.mark.parametrize("k", [1, 5, 33, 64])
def test_gram_bitwise(gpu, n, k):
    m, eng, f = make(n, 40, 0.2, k)
    eng.precompute_h_products()  # S = W^T W
    eng.precompute_w_products()  # Q = Ht^T Ht
    assert bits_equal(eng.get_product("s"), R.gram(f.w))
    assert bits_equal(eng.get_product("q"), R.gram(f.ht))


def test_gram_and_spmm_20news_shape_bitwise(gpu):
    k = 240
    m, eng, f = make(**NEWS20, k=k)
    eng.precompute_h_products()
    eng.precompute_w_products()
    assert bits_equal(eng.get_product("s"), R.gram(f.w))
    assert bits_equal(eng.get_product("q"), R.gram(f.ht))
    assert bits_equal(eng.get_product("p"), R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, f.ht))
    trp, tci, tval = ref_at(m)
    assert bits_equal(eng.get_product("r"), R.spmm(m.cols, m.rows, trp, tci, tval, f.w))


@pytest.mark.parametrize("tile,w_plan", [(16, 0), (20, 1), (24, 2)])
def test_tiled_updates_20news_scale(gpu, tile, w_plan):
    """The bench shape (C2, K=240): 77 H rows / 178 W rows per SM, so the
    staged look-ahead GEMM (lookahead_gemm_private) and the latency-ordered W
    chain run exactly as in bench.py.  H bitwise; W (norm reduction order
    only) to 1e-12 from the oracle's own H-updated state.  The tile sizes
    reach the three look-ahead W plans (operands + panel staged, panel only,
    neither)."""
    k = 240
    m, eng, f = make(**NEWS20, k=k)
    eng.precompute_h_products()
    r, s = eng.get_product("r"), eng.get_product("s")
    cfg = P.SolverConfig(rank=k, tile_size=tile)
    eng.update_h(cfg, A.tiled)
    ht1, _ = R.update_tiled(f.ht, s, r, tile, is_w=False)
    assert bits_equal(eng.get_factors().ht, ht1)
    eng.precompute_w_products()
    p, q = eng.get_product("p"), eng.get_product("q")
    eng.update_w(cfg, A.tiled)
    assert eng.stats()["w_plan"] == w_plan
    w1, norms = R.update_tiled(f.w, q, p, tile, is_w=True)
    w_eng = eng.get_factors().w
    assert rel_max(w1, w_eng) <= 1e-12
    assert elem_rel(norms, eng.get_product("column_norms")) <= 1e-12
    # the next iteration's R = A^T W from the engine's new W
    eng.precompute_h_products()
    trp, tci, tval = ref_at(m)
    assert bits_equal(eng.get_product("r"), R.spmm(m.cols, m.rows, trp, tci, tval, w_eng))


@pytest.mark.parametrize("k,tile", [(50, 7), (33, 32), (8, 8), (1, 1)])
def test_step_api_r_after_w_update_bitwise(gpu, k, tile):
    """Through the step API, R = A^T W_new after each tiled W update (ragged
    last tile, a single tile, K=1) equals spmm_into of the engine's own new W
    bit for bit, over two whole iterations."""
    m, eng, f = make(3000, 1700, 0.01, k)
    cfg = P.SolverConfig(rank=k, tile_size=tile)
    trp, tci, tval = ref_at(m)
    for _ in range(2):
        eng.precompute_h_products()
        eng.update_h(cfg, A.tiled)
        eng.precompute_w_products()
        eng.update_w(cfg, A.tiled)
        eng.precompute_h_products()
        w = eng.get_factors().w
        assert bits_equal(eng.get_product("r"), R.spmm(m.cols, m.rows, trp, tci, tval, w))


@pytest.mark.parametrize("k,tile", [(24, 5), (40, 16), (9, 9)])
def test_streaming_fallback_updates(gpu, k, tile, monkeypatch):
    """The streaming tiled update (stream.cu: phase A + one persistent
    streaming launch; the planner's choice when one SM's rows do not fit the
    persistent kernel, e.g. C5), forced on a small instance: H bitwise, W to
    1e-12 (norm reduction order only)."""
    m, eng, f = make(2500, 1300, 0.01, k)
    eng.force_streaming(True)
    eng.precompute_h_products()
    r, s = eng.get_product("r"), eng.get_product("s")
    cfg = P.SolverConfig(rank=k, tile_size=tile)
    eng.update_h(cfg, A.tiled)
    ht1, _ = R.update_tiled(f.ht, s, r, tile, is_w=False)
    assert bits_equal(eng.get_factors().ht, ht1)
    eng.precompute_w_products()
    p, q = eng.get_product("p"), eng.get_product("q")
    eng.update_w(cfg, A.tiled)
    w1, norms = R.update_tiled(f.w, q, p, tile, is_w=True)
    assert rel_max(w1, eng.get_factors().w) <= 1e-12
    assert elem_rel(norms, eng.get_product("column_norms")) <= 1e-12


def test_streaming_chosen_for_tall_w(gpu):
    """More W rows than 256 per SM: the planner streams the W update on its
    own (no override); still within 1e-12 of the oracle."""
    k, tile = 8, 3
    m, eng, f = make(40000, 300, 0.02, k)
    cfg = P.SolverConfig(rank=k, tile_size=tile)
    eng.precompute_w_products()
    p, q = eng.get_product("p"), eng.get_product("q")
    eng.update_w(cfg, A.tiled)
    w1, norms = R.update_tiled(f.w, q, p, tile, is_w=True)
    assert rel_max(w1, eng.get_factors().w) <= 1e-12
    assert elem_rel(norms, eng.get_product("column_norms")) <= 1e-12


def test_best_integer_tile_measures_and_restores(gpu):
    """The GPU tile selector (f3) returns one of the candidates, times each,
    and leaves the factors exactly as they were."""
    k = 40
    m, eng, f = make(3000, 1700, 0.01, k)
    before = eng.get_factors()
    cfg = P.SolverConfig(rank=k)
    best, times = eng.best_integer_tile(cfg, [4, 8, 16, 40])
    assert best in (4, 8, 16, 40) and set(times) == {4, 8, 16, 40}
    assert all(t > 0 for t in times.values()) and times[best] == min(times.values())
    after = eng.get_factors()
    assert bits_equal(after.w, before.w) and bits_equal(after.ht, before.ht)
    best_default, times_default = eng.best_integer_tile(cfg)
    assert best_default in times_default and max(times_default) <= k
    with pytest.raises(ValueError):
        eng.best_integer_tile(cfg, [0])


def _well_conditioned_state(m, k, iters=3, tile=0):
    """Oracle fast-hals trajectory from the seed, to move past the collapse
    of iteration 1 (Finding 1)."""
    w, ht = R.init_factors(m.rows, m.cols, k, seed=0)
    trp, tci, tval = ref_at(m)
    for _ in range(iters):
        r = R.spmm(m.cols, m.rows, trp, tci, tval, w)
        s = R.gram(w)
        ht = R.update_h_reference(ht, r, s)
        p = R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, ht)
        q = R.gram(ht)
        w, _ = R.update_w_reference(w, p, q)
    return w, ht


@pytest.mark.parametrize("k", [1, 16, 80])
def test_update_h_reference_bitwise(gpu, k):
    m, eng, f = make(2500, 1200, 0.02, k)
    eng.precompute_h_products()
    r, s = eng.get_product("r"), eng.get_product("s")
    eng.update_h(P.SolverConfig(rank=k), A.reference)
    want = R.update_h_reference(f.ht, r, s)
    assert bits_equal(eng.get_factors().ht, want)


@pytest.mark.parametrize("k,tile", [(1, 1), (16, 1), (16, 5), (16, 16), (80, 9), (240, 16), (64, 24), (37, 37), (70, 33)])
def test_update_h_tiled_bitwise(gpu, k, tile):
    m, eng, f = make(2500, 1200, 0.02, k)
    eng.precompute_h_products()
    r, s = eng.get_product("r"), eng.get_product("s")
    eng.update_h(P.SolverConfig(rank=k, tile_size=tile), A.tiled)
    want, _ = R.update_tiled(f.ht, s, r, tile, is_w=False)
    assert bits_equal(eng.get_factors().ht, want)


@pytest.mark.parametrize("k,tile", [(16, 0), (80, 0), (16, 1), (16, 4), (80, 9), (240, 16), (64, 24), (37, 37), (70, 33)])
def test_update_w_from_conditioned_state(gpu, k, tile):
    """One W update from a well-conditioned state: everything but the norm
    reduction order is shared, so W matches to ~1 ulp."""
    m = instance(2500, 1200, 0.02)
    w, ht = _well_conditioned_state(m, k)
    eng = P.Engine(P.InputMatrix(m), k)
    eng.set_factors(P.FactorPair(w, ht))
    eng.precompute_w_products()
    p, q = eng.get_product("p"), eng.get_product("q")
    alg = A.tiled if tile else A.reference
    eng.update_w(P.SolverConfig(rank=k, tile_size=tile), alg)
    if tile:
        want, norms = R.update_tiled(w, q, p, tile, is_w=True)
    else:
        want, norms = R.update_w_reference(w, p, q)
    got = eng.get_factors().w
    assert rel_max(want, got) <= 1e-12
    assert elem_rel(norms, eng.get_product("column_norms")) <= 1e-12
    assert got.min() >= 1e-16
    assert np.abs(np.sqrt((got ** 2).sum(axis=0)) - 1.0).max() <= 1e-12


def test_phase_a_exact_on_dyadic_inputs(gpu):
    """test_engine_tiled.cpp:213-239 analogue: dyadic W update, every path exact."""
    v, k = 4, 4
    m = instance(v, 4, 1.0)
    eng = P.Engine(P.InputMatrix(m), k)
    q = np.ones((k, k), order="F")
    p = np.asfortranarray(np.tile(5.0 - 0.5 * np.arange(k), (v, 1)))
    w0 = np.ones((v, k), order="F")
    for t in range(1, k + 1):
        eng.set_factors(P.FactorPair(w0, np.ones((4, k), order="F")))
        eng.set_product("q", q)
        eng.set_product("p", p)
        eng.update_w(P.SolverConfig(rank=k, tile_size=t), A.tiled)
        assert (eng.get_factors().w == 0.5).all()
    eng.set_factors(P.FactorPair(w0, np.ones((4, k), order="F")))
    eng.set_product("q", q)
    eng.set_product("p", p)
    eng.update_w(P.SolverConfig(rank=k), A.reference)
    assert (eng.get_factors().w == 0.5).all()


def test_error_gram_and_direct(gpu):
    k = 24
    m, eng, f = make(3000, 1400, 0.01, k)
    eng.precompute_w_products()
    rep = eng.evaluate_error()
    a2 = R.norm_sq(m.values)
    assert eng.norm_sq == a2  # serial order, bit-identical (input_matrix.cpp:15-20)
    want = R.relative_error_gram(a2, f.w, eng.get_product("p"), eng.get_product("q"), R.gram(f.w))
    assert abs(rep.relative - want[1]) <= 1e-13 * want[1]
    assert rep.cancellation == bool(want[2])
    d = eng.relative_error_direct()
    want_d = R.relative_error_direct_csr(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, a2, f.w, f.ht)
    assert abs(d.relative - want_d[1]) <= 1e-12 * want_d[1]
    assert abs(d.relative - rep.relative) <= 1e-9 * rep.relative  # Gram identity == direct


@pytest.mark.parametrize("tile", [0, 9])
def test_iterate_trace_matches_oracle(gpu, tile):
    """P2/P3: iterate() from the seed; the initial error and iteration-1 error
    match to ~1e-15, later iterations stay inside the fp64 chaos envelope."""
    k, iters = 16, 6
    m = instance(1500, 900, 0.02)
    cfg = P.SolverConfig(rank=k, max_iters=iters, rel_tol=0.0, tile_size=tile)
    f = P.init_factors(m.rows, m.cols, cfg)
    a = P.InputMatrix(m)
    tr = P.iterate(a, f, cfg, A.tiled if tile else A.reference)
    # oracle trajectory
    w, ht = R.init_factors(m.rows, m.cols, k, seed=0)
    trp, tci, tval = ref_at(m)
    a2 = R.norm_sq(m.values)
    p = R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, ht)
    e0 = R.relative_error_gram(a2, w, p, R.gram(ht), R.gram(w))[1]
    assert abs(tr.initial_error - e0) <= 1e-14 * e0
    errs = []
    for _ in range(iters):
        r = R.spmm(m.cols, m.rows, trp, tci, tval, w)
        s = R.gram(w)
        ht = R.update_tiled(ht, s, r, tile, is_w=False)[0] if tile else R.update_h_reference(ht, r, s)
        p = R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, ht)
        q = R.gram(ht)
        w = R.update_tiled(w, q, p, tile, is_w=True)[0] if tile else R.update_w_reference(w, p, q)[0]
        errs.append(R.relative_error_gram(a2, w, p, q, R.gram(w))[1])
    got = [rec.rel_error for rec in tr.records]
    assert [rec.iteration for rec in tr.records] == list(range(1, iters + 1))
    assert abs(got[0] - errs[0]) <= 1e-12 * errs[0]
    for g, e in zip(got, errs):
        assert abs(g - e) <= 5e-3 * e  # chaotic after iteration 1
    assert f.w.min() >= 1e-16 and f.ht.min() >= 1e-16


def test_one_step_parity_from_reference_snapshot(gpu):
    """P1 (primary gate): from the oracle's fast-hals state at iteration 10 of
    a 20News-shaped K=80 run, one GPU iteration vs one oracle iteration."""
    k = 80
    m = instance(**NEWS20)
    w, ht = _well_conditioned_state(m, k, iters=10)
    trp, tci, tval = ref_at(m)
    a2 = R.norm_sq(m.values)
    eng = P.Engine(P.InputMatrix(m), k)
    for tile, alg in [(0, A.reference), (9, A.tiled)]:
        eng.set_factors(P.FactorPair(w, ht))
        cfg = P.SolverConfig(rank=k, tile_size=tile)
        eng.precompute_h_products()
        eng.update_h(cfg, alg)
        eng.precompute_w_products()
        eng.update_w(cfg, alg)
        rep = eng.evaluate_error()
        got = eng.get_factors()
        r = R.spmm(m.cols, m.rows, trp, tci, tval, w)
        s = R.gram(w)
        ht1 = R.update_tiled(ht, s, r, tile, is_w=False)[0] if tile else R.update_h_reference(ht, r, s)
        p = R.spmm(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, ht1)
        q = R.gram(ht1)
        w1 = R.update_tiled(w, q, p, tile, is_w=True)[0] if tile else R.update_w_reference(w, p, q)[0]
        e1 = R.relative_error_gram(a2, w1, p, q, R.gram(w1))[1]
        assert bits_equal(got.ht, ht1)  # H update from identical inputs: bitwise
        assert rel_max(w1, got.w) <= 1e-10  # north-star gate is 1e-3
        assert abs(rep.relative - e1) <= 1e-12 * e1  # north-star gate is 1e-5


def test_dense_input_products_and_update(gpu):
    rng = np.random.default_rng(4242)
    v, d, k = 300, 200, 12
    ad = np.asfortranarray(rng.random((v, d)))
    a = P.InputMatrix(ad)
    eng = P.Engine(a, k)
    cfg = P.SolverConfig(rank=k, tile_size=5)
    f = P.init_factors(v, d, cfg)
    eng.set_factors(f)
    eng.precompute_w_products()
    eng.precompute_h_products()
    # accumulate_nn: sequential k; accumulate_tn: 2 lanes over V (linalg.cpp:45-79)
    p_want = np.zeros((v, k), order="F")
    for kk in range(d):
        p_want = p_want + f.ht[kk][None, :] * ad[:, kk][:, None]
    assert bits_equal(eng.get_product("p"), p_want)
    even = np.zeros((d, k))
    odd = np.zeros((d, k))
    for vv in range(0, v - 1, 2):
        even = even + ad[vv][:, None] * f.w[vv][None, :]
        odd = odd + ad[vv + 1][:, None] * f.w[vv + 1][None, :]
    if v % 2:
        even = even + ad[v - 1][:, None] * f.w[v - 1][None, :]
    assert bits_equal(eng.get_product("r"), (even + 0.0) + odd)
    rep = eng.evaluate_error()
    direct = eng.relative_error_direct()
    assert abs(rep.relative - direct.relative) <= 1e-9 * direct.relative


def test_errors_map_to_reference_exceptions(gpu):
    m = instance(50, 40, 0.1)
    a = P.InputMatrix(m)
    f = P.init_factors(50, 40, P.SolverConfig(rank=4))
    with pytest.raises(P.InvalidArgument, match="tile_size"):
        P.iterate(a, f, P.SolverConfig(rank=4, tile_size=0), A.tiled)
    with pytest.raises(P.InvalidArgument):
        P.iterate(a, f, P.SolverConfig(rank=5), A.reference)
    with pytest.raises(P.InvalidArgument, match="epsilon"):
        P.iterate(a, f, P.SolverConfig(rank=4, epsilon=0.0), A.reference)
    z = P.CsrMatrix(3, 3, np.zeros(4, np.int64), np.zeros(0, np.int64), np.zeros(0))
    fz = P.init_factors(3, 3, P.SolverConfig(rank=2))
    with pytest.raises(P.DomainError):
        P.iterate(P.InputMatrix(z), fz, P.SolverConfig(rank=2), A.reference)
    bad = P.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 1]), np.array([1.0, -1.0]))
    with pytest.raises(P.InvalidArgument, match="non-negative"):
        P.Engine(P.InputMatrix(bad), 2)
