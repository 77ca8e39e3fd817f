"""Runs a few C2 FAST-HALS iterations (the bench workload) for profilers:
   ncu --metrics gpu__time_duration.sum ... python tools/profile_step.py [iters] [tile] [math]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tile = int(sys.argv[2]) if len(sys.argv) > 2 else bench.TILE
math = sys.argv[3] if len(sys.argv) > 3 else "exact"
m = bench.make_input()
eng = P.Engine(P.InputMatrix(m), bench.K)
eng.set_math(P.Math.exact if math == "exact" else P.Math.fused)
cfg = P.SolverConfig(rank=bench.K, tile_size=tile, max_iters=1, rel_tol=0.0)
eng.init_factors(cfg)
ms = eng.run_iterations(cfg, P.Algorithm.tiled, iters)
print(f"{iters} iterations: {ms:.3f} ms ({ms / iters:.3f} ms/iter)")
