"""The bench's e2e leg alone: plnmf_gpu_iterate_host (100 iterations, error every
iteration, rel_tol 0) on pinned host factors at C2; iterations/s on the host clock."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

m = bench.make_input()
eng = P.Engine(P.InputMatrix(m), bench.K)
cfg = P.SolverConfig(rank=bench.K, tile_size=bench.TILE, max_iters=100, rel_tol=0.0, error_every=1)
f = P.init_factors(m.rows, m.cols, cfg)
for rep in range(4):
    w = np.asfortranarray(f.w.copy())
    ht = np.asfortranarray(f.ht.copy())
    eng.set_factors(P.FactorPair(w, ht))
    t0 = time.perf_counter()
    tr = eng.iterate(cfg, P.Algorithm.tiled)
    dt = time.perf_counter() - t0
    print(f"iterate(100, error_every=1): {100 / dt:.1f} it/s ({1e3 * dt / 100:.3f} ms/iteration); "
          f"error_eval {1e6 * tr.totals.error_eval / 100:.1f} us/it; final rel {tr.records[-1].rel_error:.6f}")
