# Round-2 second profile set: the C5 streaming W kernel (column-major), the C3 W update on the
# streaming plan, and the Math::tensor phase-A GEMM at C3 (tensor pipe utilisation)
mkdir -p gpurun_out
N="ncu --set full --clock-control none -f"
timeout 1500 $N -k regex:stream_w_kernel -c 1 -o gpurun_out/r2_c5_wupdate python tools/c5_step.py 1 > gpurun_out/r2_c5_wupdate.log 2>&1
cat > /tmp/c3t.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1904_07935_b200 import plnmf as P
m = P.synth_csr(36771, 10212, 1323869 / (36771 * 10212), 20)
eng = P.Engine(P.InputMatrix(m), 480)
cfg = P.SolverConfig(rank=480, tile_size=22)
eng.set_math(P.Math.tensor)
eng.init_factors(cfg)
eng.run_iterations(cfg, P.Algorithm.tiled, 1)
PY
timeout 900 $N -k regex:"ozaki_gemm|stream_w_kernel" -c 2 -o gpurun_out/r2_c3_tensor python /tmp/c3t.py > gpurun_out/r2_c3_tensor.log 2>&1
for r in c5_wupdate c3_tensor; do ncu -i gpurun_out/r2_$r.ncu-rep --page raw --csv > gpurun_out/r2_raw_$r.csv 2>/dev/null; done
tail -2 gpurun_out/r2_c3_tensor.log
