"""Math.tensor against Math.exact for the streaming tiled updates (phase A on the
tensor cores): C3 (TDT2, K=480, T=22 — W on the streaming plan) and C5 on one GPU."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402
from paper_1904_07935_b200.sharded import ShardEngine  # noqa: E402

m = P.synth_csr(36771, 10212, 1323869 / (36771 * 10212), 20)
eng = P.Engine(P.InputMatrix(m), 480)
cfg = P.SolverConfig(rank=480, tile_size=22)
for math in (P.Math.exact, P.Math.tensor):
    eng.set_math(math)
    eng.init_factors(cfg)
    eng.run_iterations(cfg, P.Algorithm.tiled, 2)
    ms = eng.run_iterations(cfg, P.Algorithm.tiled, 3) / 3
    ph = {a: round(b / 3, 3) for a, b in eng.phase_ms().items()}
    print(f"C3 T=22 {math.name}: {ms:.2f} ms/iter {ph}", flush=True)
eng.close()

# C5 on one GPU: the single engine on the device-generated matrix (the shard engine refuses Math.tensor)
e5 = P.Engine.synthetic(bench.V5, bench.D5, bench.DENS5, bench.GEN_SEED, bench.K5)
rng = np.random.default_rng(1000)
e5.set_factors(P.FactorPair(np.asfortranarray(rng.uniform(1e-3, 1.0, (bench.V5, bench.K5))),
                            np.asfortranarray(rng.uniform(1e-3, 1.0, (bench.D5, bench.K5)))))
c5 = P.SolverConfig(rank=bench.K5, tile_size=bench.TILE5)
for math in (P.Math.exact, P.Math.tensor):
    e5.set_math(math)
    e5.run_iterations(c5, P.Algorithm.tiled, 1)
    ms = e5.run_iterations(c5, P.Algorithm.tiled, 2) / 2
    ph = {a: round(b / 2, 1) for a, b in e5.phase_ms().items()}
    print(f"C5 {math.name}: {ms:.1f} ms/iter {ph}", flush=True)
