"""Per-phase CUDA-event times of iterate() on the bench workload."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

m = bench.make_input()
eng = P.Engine(P.InputMatrix(m), bench.K)
alg = P.Algorithm.tiled if len(sys.argv) < 2 else P.Algorithm(int(sys.argv[1]))
cfg = P.SolverConfig(rank=bench.K, tile_size=bench.TILE, max_iters=6, rel_tol=0.0)
eng.init_factors(cfg)
tr = eng.iterate(cfg, alg)
for r in tr.records[2:]:
    ph = r.phases
    print(f"it {r.iteration}: pre_h {ph.precompute_h*1e6:7.1f} upd_h {ph.update_h*1e6:7.1f} pre_w {ph.precompute_w*1e6:7.1f} "
          f"upd_w {ph.update_w*1e6:7.1f} phase2 {ph.phase2*1e6:7.1f} err {ph.error_eval*1e6:7.1f} us  rel={r.rel_error:.6f}")
