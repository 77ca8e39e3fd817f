"""C5 tiled H and W update times on one GPU (single engine on the device-generated matrix),
CUDA events over repeated launches (time_kernel), for A/B comparisons of the streaming kernels."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

e = P.Engine.synthetic(bench.V5, bench.D5, bench.DENS5, bench.GEN_SEED, bench.K5)
rng = np.random.default_rng(1000)
e.set_factors(P.FactorPair(np.asfortranarray(rng.uniform(1e-3, 1.0, (bench.V5, bench.K5))),
                           np.asfortranarray(rng.uniform(1e-3, 1.0, (bench.D5, bench.K5)))))
cfg = P.SolverConfig(rank=bench.K5, tile_size=bench.TILE5)
e.precompute_h_products()
e.precompute_w_products()
for rep in range(3):
    h = e.time_kernel(cfg, 4, 3)
    w = e.time_kernel(cfg, 3, 3)
    print(f"C5 update H {h:.2f} ms, update W {w:.2f} ms", flush=True)
