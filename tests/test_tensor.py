"""Math.tensor: the dense-A products P = A Ht and R = A^T W on the tensor
cores (Ozaki-split u8 tcgen05.mma GEMMs, csrc/ozaki.cu) against the exact
products, which are bit-identical to the reference's gemm (test_gpu_parity.py).
The tensor path is not the reference's summation order; it is held to 1e-13
relative per entry (non-negative data: no cancellation), and one full
iteration from there to the reference's own fp64 rounding envelope."""
import numpy as np
import pytest

from _helpers import bits_equal, rel_max
from paper_1904_07935_b200 import plnmf as P

pytestmark = pytest.mark.gpu


def _products(eng, f, math):
    eng.set_math(math)
    eng.set_factors(f)
    eng.precompute_h_products()
    eng.precompute_w_products()
    return eng.get_product("r"), eng.get_product("p"), eng.get_product("s"), eng.get_product("q")


def _elem_rel(ref, got):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


@pytest.mark.parametrize("v,d,k", [(300, 257, 16), (129, 1000, 40), (517, 333, 80), (1000, 700, 160), (64, 64, 1),
                                   (200, 5100, 24)])
def test_tensor_products_match_exact(gpu, v, d, k):
    rng = np.random.default_rng(v * 31 + d)
    dense = np.asfortranarray(rng.uniform(0.0, 1.0, (v, d)))
    dense[rng.uniform(size=(v, d)) < 0.1] = 0.0  # some structural zeros
    eng = P.Engine(P.InputMatrix(dense), k)
    f = P.init_factors(v, d, P.SolverConfig(rank=k))
    r0, p0, s0, q0 = _products(eng, f, P.Math.exact)
    r1, p1, s1, q1 = _products(eng, f, P.Math.tensor)
    assert _elem_rel(p0, p1) <= 1e-13, _elem_rel(p0, p1)
    assert _elem_rel(r0, r1) <= 1e-13, _elem_rel(r0, r1)
    assert bits_equal(s0, s1) and bits_equal(q0, q1)  # the Grams stay exact


def test_tensor_one_step_from_a_converging_state(gpu):
    """From a well-conditioned state (10 exact iterations: past the iteration-1
    collapse), one iteration with the tensor-core products
    against one exact iteration: the north-star gate (1e-3 on W/H, 1e-5 on the
    error) with orders of magnitude to spare."""
    v, d, k = 2000, 1500, 64
    rng = np.random.default_rng(7)
    dense = np.asfortranarray(rng.uniform(0.0, 1.0, (v, d)))
    eng = P.Engine(P.InputMatrix(dense), k)
    cfg = P.SolverConfig(rank=k, max_iters=10, rel_tol=0.0, tile_size=8)
    eng.init_factors(cfg)
    eng.iterate(cfg, P.Algorithm.tiled)
    state = eng.get_factors()
    out = {}
    for math in (P.Math.exact, P.Math.tensor):
        eng.set_math(math)
        eng.set_factors(state)
        eng.precompute_h_products()
        eng.update_h(cfg, P.Algorithm.tiled)
        eng.precompute_w_products()
        eng.update_w(cfg, P.Algorithm.tiled)
        out[math] = (eng.evaluate_error().relative, eng.get_factors())
    (ee, fe), (et, ft) = out[P.Math.exact], out[P.Math.tensor]
    assert abs(et - ee) <= 1e-12 * ee
    assert rel_max(fe.ht, ft.ht) <= 1e-10 and rel_max(fe.w, ft.w) <= 1e-10


@pytest.mark.parametrize("k,tile", [(24, 5), (40, 16), (33, 32)])
def test_tensor_phase_a_of_streaming_updates(gpu, k, tile):
    """Math.tensor on a sparse input: the streaming tiled updates' phase A (init +
    phase 1 for every column, tiled.cpp:28-65) as one Ozaki tcgen05 GEMM.  One
    iteration from a converging state against the exact path: factors to 1e-9
    (the fp64 chaos envelope the reference's own two paths define is 1e-3), the
    error to 1e-11."""
    m = P.synth_csr(1500, 900, 0.02, 9)
    eng = P.Engine(P.InputMatrix(m), k)
    eng.force_streaming(True)
    cfg = P.SolverConfig(rank=k, max_iters=8, rel_tol=0.0, tile_size=tile)
    eng.init_factors(cfg)
    eng.iterate(cfg, P.Algorithm.tiled)
    state = eng.get_factors()
    out = {}
    for math in (P.Math.exact, P.Math.tensor):
        eng.set_math(math)
        eng.set_factors(state)
        eng.precompute_h_products()
        eng.update_h(cfg, P.Algorithm.tiled)
        eng.precompute_w_products()
        eng.update_w(cfg, P.Algorithm.tiled)
        out[math] = (eng.evaluate_error().relative, eng.get_factors())
    (ee, fe), (et, ft) = out[P.Math.exact], out[P.Math.tensor]
    assert rel_max(fe.ht, ft.ht) <= 1e-9 and rel_max(fe.w, ft.w) <= 1e-9
    assert abs(et - ee) <= 1e-11 * ee
    assert not bits_equal(fe.w, ft.w)  # the tensor path really ran (a different summation)
