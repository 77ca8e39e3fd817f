"""C3 (TDT2 shape, K=480) per-iteration time and update plans for several tile sizes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_07935_b200 import plnmf as P  # noqa: E402

# TDT2 shape
m = P.synth_csr(36771, 10212, 1323869 / (36771 * 10212), 20)
k = 480
eng = P.Engine(P.InputMatrix(m), k)
for T in (16, 22, 24, 32):
    cfg = P.SolverConfig(rank=k, tile_size=T)
    eng.init_factors(cfg)
    eng.run_iterations(cfg, P.Algorithm.tiled, 2)
    ms = eng.run_iterations(cfg, P.Algorithm.tiled, 3) / 3
    ph = {a: round(b / 3, 3) for a, b in eng.phase_ms().items()}
    st = eng.stats()
    print(f"C3 T={T}: {ms:.2f} ms/iter {ph} w_plan {st['w_plan']} h_plan {st['h_plan']}", flush=True)
# the streaming plan (column-major stream_w_kernel) for the same tiles, for comparison
eng.force_streaming(True)
for T in (16, 22, 24, 32):
    cfg = P.SolverConfig(rank=k, tile_size=T)
    eng.init_factors(cfg)
    eng.run_iterations(cfg, P.Algorithm.tiled, 2)
    ms = eng.run_iterations(cfg, P.Algorithm.tiled, 3) / 3
    ph = {a: round(b / 3, 3) for a, b in eng.phase_ms().items()}
    print(f"C3 T={T} streaming: {ms:.2f} ms/iter {ph}", flush=True)
