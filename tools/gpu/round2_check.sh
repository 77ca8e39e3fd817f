# Round-2 check: full GPU suite, smoke, C2 bench + reference arm, C5 bench (1 GPU), SpMM ncu captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
N="ncu --set full --import-source on --clock-control none -f"
timeout 600 $N -k regex:spmm_csr_v2 --launch-skip 3 -c 1 -o gpurun_out/r2_spmm python tools/profile_step.py 2 > gpurun_out/r2_spmm.log 2>&1
timeout 1200 $N -k regex:spmm_blocked -c 2 -o gpurun_out/r2_c5_spmm python tools/c5_step.py 1 > gpurun_out/r2_c5_spmm.log 2>&1
for r in spmm c5_spmm; do ncu -i gpurun_out/r2_$r.ncu-rep --page raw --csv > gpurun_out/r2_raw_$r.csv 2>/dev/null; done
tail -3 gpurun_out/r2_pytest_gpu.log; cat gpurun_out/r2_smoke.log; cat gpurun_out/r2_bench.json | head -c 600; echo; cat gpurun_out/r2_bench_c5.json | head -c 400
