"""W update time of the look-ahead plans against the streaming plan, per tile size, on the C2
(20News, K=240) and C3 (TDT2, K=480) shapes: which plan the planner should take when the
coefficient panel does not fit shared memory (plan 2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

for name, (v, d, nnz, k) in {"C2": (26214, 11314, 1018191, 240), "C3": (36771, 10212, 1323869, 480)}.items():
    m = P.synth_csr(v, d, nnz / (v * d), 20)
    eng = P.Engine(P.InputMatrix(m), k)
    for T in (12, 16, 20, 24, 32):
        row = []
        for streaming in (False, True):
            eng.force_streaming(streaming)
            cfg = P.SolverConfig(rank=k, tile_size=T)
            eng.init_factors(cfg)
            eng.run_iterations(cfg, P.Algorithm.tiled, 1)
            eng.run_iterations(cfg, P.Algorithm.tiled, 2)
            ph = eng.phase_ms()
            row.append((ph["update_w"] / 2, eng.stats()["w_plan"]))
        print(f"{name} T={T:2d}: look-ahead W {row[0][0]:7.3f} ms (plan {row[0][1]}), streaming W {row[1][0]:7.3f} ms",
              flush=True)
