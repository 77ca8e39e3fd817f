"""A C4-shaped dense iteration with the Math::tensor products (Ozaki u8
tcgen05.mma GEMMs), smaller than C4 so ncu replays stay short:
   ncu ... python tools/tensor_step.py [n] [k]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else 160
dense = np.asfortranarray(np.random.default_rng(4242).uniform(0.0, 1.0, (n, n)))
eng = P.Engine(P.InputMatrix(dense), k)
eng.set_math(P.Math.tensor)
cfg = P.SolverConfig(rank=k, tile_size=13)
eng.init_factors(cfg)
ms = eng.run_iterations(cfg, P.Algorithm.tiled, 2)
print(f"{n}x{n} K={k} tensor: {ms / 2:.3f} ms/iteration")
