"""CUDA-event times of the engine's kernel families on the bench workload (C2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

tile = int(sys.argv[1]) if len(sys.argv) > 1 else bench.TILE
m = bench.make_input()
eng = P.Engine(P.InputMatrix(m), bench.K)
cfg = P.SolverConfig(rank=bench.K, tile_size=tile, max_iters=1, rel_tol=0.0)
eng.init_factors(cfg)
eng.run_iterations(cfg, P.Algorithm.tiled, 3)
names = ["spmm A*Ht", "spmm At*W", "gram W", "update W", "update H"]
for i, n in enumerate(names):
    print(f"{n:12s} {eng.time_kernel(cfg, i, 5) * 1e3:9.1f} us")
print(f"iteration    {eng.run_iterations(cfg, P.Algorithm.tiled, 10) * 1e2:9.1f} us")
