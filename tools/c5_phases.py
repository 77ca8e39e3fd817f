"""C5 one-GPU per-iteration phase times through the sharded engine (world 1)."""
import sys; sys.path.insert(0, '.')
import numpy as np, bench
from paper_1904_07935_b200 import plnmf as P
from paper_1904_07935_b200.sharded import ShardEngine
eng = ShardEngine.generate(bench.V5, bench.D5, bench.DENS5, bench.GEN_SEED, bench.K5, 1, 0)
eng.set_norm_sq(1.0)
rng = np.random.default_rng(1000)
eng.set_factors(P.FactorPair(np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.v, bench.K5))),
                             np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.d, bench.K5)))))
cfg = P.SolverConfig(rank=bench.K5, tile_size=bench.TILE5)
for i in range(6):
    ms = eng.run_iterations(cfg, P.Algorithm.tiled, 1)
    print(f"{ms:.1f}", {a: round(b, 1) for a, b in eng.phase_ms().items()}, flush=True)
print("stats", eng.stats())
