"""Generates the golden fixtures in this directory from the REFERENCE ITSELF
(oracle/_ref/libplnmf_ref.so: libplnmf compiled from /root/reference/proj/src
by oracle/Makefile, unmodified, driven through its public API by
oracle/ref_shim.cpp).  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures are small .npz files; tests/test_golden.py checks the C
restatement (CPU) and the GPU engine (gpu marker) against them.  Contents:

  tiny_mtx.npz   proj/tests/data/tiny.mtx parsed by read_matrix_market; init
                 factors (K=3, seed 7); one fast-hals and one pl-nmf (T=2)
                 iteration step by step (R, S, Ht, P, Q, W, column norms);
                 iterate() traces for both algorithms (5 iterations).
  synth_small.npz  a 300x200 synthetic CSR (density 0.05, generator seed 20),
                 K=12: the same quantities, pl-nmf with T=5, plus the
                 relative_error_gram / _direct reports.
  dense_small.npz  a dense 60x40 U(0,1) matrix (mt19937_64 seed 4242, like
                 proj/bench/bench_updates.cpp:31-38), K=6, T=4.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import (RefInput, RefSession, ref, ref_init_factors, ref_iterate,  # noqa: E402
                           ref_read_mm, ref_transpose)

OUT = Path(__file__).resolve().parent
TINY = Path("/root/reference/proj/tests/data/tiny.mtx")


def one_iteration(sess, w, ht, tile):
    sess.precompute_h(w)
    r, s = sess.get("r"), sess.get("s")
    ht1 = sess.update_h(ht, tile=tile)
    sess.precompute_w(ht1)
    p, q = sess.get("p"), sess.get("q")
    w1 = sess.update_w(w, tile=tile)
    return dict(r=r, s=s, ht1=ht1, p=p, q=q, w1=w1, norms=sess.get("column_norms"), macs=sess.macs())


def dump(name, a: RefInput, k, tile, seed, extra):
    w, ht = ref_init_factors(a.rows, a.cols, k, seed=seed)
    out = dict(k=k, tile=tile, seed=seed, w0=w, ht0=ht, a_norm_sq=a.norm_sq, **extra)
    for alg, t in (("ref", 0), ("tiled", tile)):
        sess = RefSession(a, k)
        it = one_iteration(sess, w, ht, t)
        for key, v in it.items():
            out[f"{alg}_{key}"] = v
        # error of the updated factors: gram + direct
        sess.precompute_w(it["ht1"])
        wf, htf, tr = ref_iterate(a, w, ht, k, max_iters=5, rel_tol=0.0, seed=seed, tile=t, tiled=bool(t))
        out[f"{alg}_trace_initial"] = tr["initial_error"]
        out[f"{alg}_trace_rel"] = tr["records"][:, 1].copy()
        out[f"{alg}_trace_macs"] = tr["update_macs"]
        out[f"{alg}_w5"] = wf
        out[f"{alg}_ht5"] = htf
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, {k2: getattr(v, "shape", v) for k2, v in out.items() if k2.endswith(("w1", "trace_rel"))})


def main():
    ref().ref_set_threads(1)  # the pl-nmf norm partials depend on the OpenMP team size (tiled.cpp:97-99)
    m = ref_read_mm(TINY)
    a = RefInput(m["rows"], m["cols"], m["rp"], m["ci"], m["val"])
    trp, tci, tval = ref_transpose(m["rows"], m["cols"], m["rp"], m["ci"], m["val"])
    dump("tiny_mtx", a, 3, 2, 7, dict(rows=m["rows"], cols=m["cols"], rp=m["rp"], ci=m["ci"], val=m["val"],
                                      trp=trp, tci=tci, tval=tval))

    from paper_1904_07935_b200 import plnmf as P  # the generator is host code (no GPU needed)
    s = P.synth_csr(300, 200, 0.05, 20)
    a = RefInput(s.rows, s.cols, s.row_ptr, s.col_idx, s.values)
    trp, tci, tval = ref_transpose(s.rows, s.cols, s.row_ptr, s.col_idx, s.values)
    dump("synth_small", a, 12, 5, 0, dict(rows=s.rows, cols=s.cols, rp=s.row_ptr, ci=s.col_idx, val=s.values,
                                          trp=trp, tci=tci, tval=tval))

    rng = np.random.Generator(np.random.MT19937(4242))
    dense = np.asfortranarray(rng.random((60, 40)))
    a = RefInput(60, 40, dense=dense)
    dump("dense_small", a, 6, 4, 3, dict(rows=60, cols=40, dense=dense))


if __name__ == "__main__":
    main()
