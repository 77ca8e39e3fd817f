"""Golden fixtures produced by the compiled reference (tests/golden/make_golden.py).

CPU: the C restatement reproduces every fixture bit for bit (this pins the
oracle the GPU tests use).  GPU: the engine reproduces the products and the H
updates bit for bit and W to 1e-12 (its norm reduction order is its own).
"""
from pathlib import Path

import numpy as np
import pytest

from _helpers import Restated as R, bits_equal, rel_max
from paper_1904_07935_b200 import plnmf as P

GOLDEN = Path(__file__).resolve().parent / "golden"
NAMES = ["tiny_mtx", "synth_small", "dense_small"]


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def restated_iteration(g, tile):
    """One iteration with the restatement, in the reference's step order."""
    w, ht = g["w0"], g["ht0"]
    if "dense" in g:
        a = g["dense"]
        r = np.zeros((a.shape[1], w.shape[1]), order="F")
        # accumulate_tn: (lane0 + 0.0) + lane1 over rows, then 0 + 1.0*acc
        ev = np.zeros_like(r)
        od = np.zeros_like(r)
        n = a.shape[0]
        for v in range(0, n - 1, 2):
            ev = ev + a[v][:, None] * w[v][None, :]
            od = od + a[v + 1][:, None] * w[v + 1][None, :]
        if n % 2:
            ev = ev + a[n - 1][:, None] * w[n - 1][None, :]
        r = 0.0 + 1.0 * ((ev + 0.0) + od)
    else:
        r = R.spmm(int(g["cols"]), int(g["rows"]), g["trp"], g["tci"], g["tval"], w)
    s = R.gram(w)
    ht1 = R.update_tiled(ht, s, r, tile, is_w=False)[0] if tile else R.update_h_reference(ht, r, s)
    if "dense" in g:
        a = g["dense"]
        p = np.zeros((a.shape[0], w.shape[1]), order="F")
        for kk in range(a.shape[1]):
            p = p + ht1[kk][None, :] * a[:, kk][:, None]
    else:
        p = R.spmm(int(g["rows"]), int(g["cols"]), g["rp"], g["ci"], g["val"], ht1)
    q = R.gram(ht1)
    if tile:
        w1, norms = R.update_tiled(w, q, p, tile, is_w=True, nthreads=1)
    else:
        w1, norms = R.update_w_reference(w, p, q)
    return dict(r=r, s=s, ht1=ht1, p=p, q=q, w1=w1, norms=norms)


@pytest.mark.parametrize("name", NAMES)
def test_golden_init_factors_bitwise(name):
    g = load(name)
    k, seed = int(g["k"]), int(g["seed"])
    w, ht = R.init_factors(int(g["rows"]), int(g["cols"]), k, seed=seed)
    assert bits_equal(w, g["w0"]) and bits_equal(ht, g["ht0"])
    f = P.init_factors(int(g["rows"]), int(g["cols"]), P.SolverConfig(rank=k, seed=seed))  # product host code
    assert bits_equal(f.w, g["w0"]) and bits_equal(f.ht, g["ht0"])


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("alg", ["ref", "tiled"])
def test_golden_restatement_bitwise(name, alg):
    g = load(name)
    tile = int(g["tile"]) if alg == "tiled" else 0
    got = restated_iteration(g, tile)
    for key in ("r", "s", "ht1", "p", "q", "w1", "norms"):
        assert bits_equal(got[key], g[f"{alg}_{key}"]), key
    if "val" in g:
        assert R.norm_sq(g["val"]) == g["a_norm_sq"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("alg", ["ref", "tiled"])
def test_golden_engine(gpu, name, alg):
    g = load(name)
    k = int(g["k"])
    tile = int(g["tile"]) if alg == "tiled" else 0
    if "dense" in g:
        a = P.InputMatrix(g["dense"])
    else:
        a = P.InputMatrix(P.CsrMatrix(int(g["rows"]), int(g["cols"]), g["rp"], g["ci"], g["val"]))
    eng = P.Engine(a, k)
    assert eng.norm_sq == g["a_norm_sq"]
    eng.set_factors(P.FactorPair(g["w0"], g["ht0"]))
    cfg = P.SolverConfig(rank=k, tile_size=tile)
    algorithm = P.Algorithm.tiled if tile else P.Algorithm.reference
    eng.precompute_h_products()
    assert bits_equal(eng.get_product("r"), g[f"{alg}_r"])
    assert bits_equal(eng.get_product("s"), g[f"{alg}_s"])
    eng.update_h(cfg, algorithm)
    assert bits_equal(eng.get_factors().ht, g[f"{alg}_ht1"])
    eng.precompute_w_products()
    assert bits_equal(eng.get_product("p"), g[f"{alg}_p"])
    assert bits_equal(eng.get_product("q"), g[f"{alg}_q"])
    eng.update_w(cfg, algorithm)
    assert rel_max(g[f"{alg}_w1"], eng.get_factors().w) <= 1e-12
    assert rel_max(g[f"{alg}_norms"], eng.get_product("column_norms")) <= 1e-12
    # iterate(): initial error to ~1 ulp; first iteration to 1e-12
    f = P.FactorPair(g["w0"].copy(order="F"), g["ht0"].copy(order="F"))
    tr = P.iterate(a, f, P.SolverConfig(rank=k, tile_size=tile, max_iters=5, rel_tol=0.0), algorithm)
    assert abs(tr.initial_error - g[f"{alg}_trace_initial"]) <= 1e-14 * g[f"{alg}_trace_initial"]
    want = g[f"{alg}_trace_rel"]
    got = np.array([r.rel_error for r in tr.records])
    assert abs(got[0] - want[0]) <= 1e-12 * want[0]
    assert abs(got[1] - want[1]) <= 1e-9 * want[1]
    # From iteration 3 on, the ~1-ulp norm difference is amplified by the
    # collapse of iteration 1 (Finding 1): the reference's own
    # fast-hals and pl-nmf paths drift apart the same way; hold the trajectory
    # to the fp64 chaos envelope and to the reference's monotonicity check
    # (acceptance.cpp criterion 7).
    assert np.all(np.abs(got - want) <= 2e-2 * want)
    assert np.all(np.diff(np.concatenate([[tr.initial_error], got])) <= 1e-8)
    assert tr.update_macs == int(g[f"{alg}_trace_macs"])  # acceptance.cpp criterion 6 bookkeeping
