"""C5 SpMM column-block sweep: P = A Ht and R = A^T W on one GPU (sharded engine,
world 1) for several block sizes; host-timed step calls (each ends in a sync).
   python tools/c5_spmm_sweep.py [block_rows ...]   (0 = automatic, -1 = unblocked)"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402
from paper_1904_07935_b200.sharded import ShardEngine  # noqa: E402

blocks = [int(x) for x in sys.argv[1:]] or [-1, 0, 8192, 16384, 32768, 65536]
eng = ShardEngine.generate(bench.V5, bench.D5, bench.DENS5, bench.GEN_SEED, bench.K5, 1, 0)
eng.set_norm_sq(1.0)
rng = np.random.default_rng(1000)
eng.set_factors(P.FactorPair(np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.v, bench.K5))),
                             np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.d, bench.K5)))))
ref = None
for b in blocks:
    eng.force_spmm_blocks(10**12 if b < 0 else b)
    eng.precompute_w_products()  # warm
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        eng.precompute_w_products()
        t1 = time.perf_counter()
        eng.precompute_h_products()
        t.append((t1 - t0, time.perf_counter() - t1))
    rows = np.arange(0, bench.V5, 9973)
    p = eng.get_rows("p", rows)
    same = "" if ref is None else ("bitwise" if (p.view(np.uint64) == ref.view(np.uint64)).all() else "DIFFERS")
    ref = p if ref is None else ref
    print(f"block {b:>8d}: precompute_w (P + Q) {1e3 * min(x[0] for x in t):7.1f} ms, "
          f"precompute_h (R + S) {1e3 * min(x[1] for x in t):7.1f} ms  {same}", flush=True)
