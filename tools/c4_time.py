"""C4 (dense 20K x 20K, K = 160, T = 13) per-iteration device time, exact SIMT
products vs the tensor-core (Ozaki u8 tcgen05) products; per-phase split and the
two dense products alone (CUDA events on the engine stream)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

v = d = 20000
k, tile = 160, 13
dense = np.asfortranarray(np.random.default_rng(4242).uniform(0.0, 1.0, (v, d)))
eng = P.Engine(P.InputMatrix(dense), k)
cfg = P.SolverConfig(rank=k, tile_size=tile)
for math in (P.Math.exact, P.Math.tensor):
    eng.set_math(math)
    eng.init_factors(cfg)
    eng.run_iterations(cfg, P.Algorithm.tiled, 1)
    ms = eng.run_iterations(cfg, P.Algorithm.tiled, 3) / 3
    ph = {k2: v2 / 3 for k2, v2 in eng.phase_ms().items()}
    pa = eng.time_kernel(cfg, 0, 3)
    ra = eng.time_kernel(cfg, 1, 3)
    print(f"C4 {math.name}: {ms:.2f} ms/iteration ({1e3 / ms:.1f} it/s); A*Ht {pa:.2f} ms, A^T*W {ra:.2f} ms; "
          f"phases " + " ".join(f"{a} {b:.2f}" for a, b in ph.items()), flush=True)
