"""C5 (2M x 1M, ~1e9 nonzeros, K=256) iterations on one GPU through the sharded
engine (world 1), for profilers:  ncu ... python tools/c5_step.py [iters]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402
from paper_1904_07935_b200.sharded import ShardEngine  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
eng = ShardEngine.generate(bench.V5, bench.D5, bench.DENS5, bench.GEN_SEED, bench.K5, 1, 0)
eng.set_norm_sq(1.0)
rng = np.random.default_rng(1000)
eng.set_factors(P.FactorPair(np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.v, bench.K5))),
                             np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.d, bench.K5)))))
cfg = P.SolverConfig(rank=bench.K5, tile_size=bench.TILE5)
ms = eng.run_iterations(cfg, P.Algorithm.tiled, iters)
print(f"C5 {iters} iterations: {ms / iters:.1f} ms/iteration; phases {eng.phase_ms()}")
