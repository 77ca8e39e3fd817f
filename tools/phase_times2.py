"""Per-phase device times of iterate() on the bench workload (CUDA events in the engine)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

m = bench.make_input()
eng = P.Engine(P.InputMatrix(m), bench.K)
cfg = P.SolverConfig(rank=bench.K, tile_size=bench.TILE, max_iters=20, rel_tol=0.0)
eng.init_factors(cfg)
eng.run_iterations(cfg, P.Algorithm.tiled, 3)
tr = eng.iterate(cfg, P.Algorithm.tiled)
t = tr.totals
n = len(tr.records)
for k in ("precompute_h", "update_h", "precompute_w", "update_w", "phase2", "error_eval"):
    print(f"{k:14s} {getattr(t, k) / n * 1e6:9.1f} us/iter")
print(f"total          {tr.total_seconds / n * 1e6:9.1f} us/iter (incl. error evaluation)")
