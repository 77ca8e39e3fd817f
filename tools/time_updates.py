"""CUDA-event times of the engine's kernel families.
   python tools/time_updates.py [V D NNZ K TILE [dense]]   (default: the bench workload C2)"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

if len(sys.argv) >= 6:
    v, d, nnz, k, tile = (int(x) for x in sys.argv[1:6])
    if len(sys.argv) > 6 and sys.argv[6] == "dense":
        rng = np.random.Generator(np.random.MT19937(4242))
        a = P.InputMatrix(np.asfortranarray(rng.random((v, d))))
    else:
        a = P.InputMatrix(P.synth_csr(v, d, nnz / (v * d), 20))
else:
    v, d, k, tile = bench.V, bench.D, bench.K, bench.TILE
    a = P.InputMatrix(bench.make_input())
eng = P.Engine(a, k)
cfg = P.SolverConfig(rank=k, tile_size=tile, max_iters=1, rel_tol=0.0)
eng.init_factors(cfg)
eng.run_iterations(cfg, P.Algorithm.tiled, 2)
names = ["A*Ht", "At*W", "gram W", "update W", "update H", "gram Ht", "precompute_w", "phase A (H)", "precompute_h"]
print(f"V={v} D={d} K={k} T={tile} nnz={eng.nnz}")
for i, n in enumerate(names):
    print(f"{n:12s} {eng.time_kernel(cfg, i, 3) * 1e3:10.1f} us")
print(f"iteration    {eng.run_iterations(cfg, P.Algorithm.tiled, 5) * 2e2:10.1f} us")
