# Round-2 final set (after the one-row Gram step and the W panel staged from coeff): full GPU suite, smoke,
# bench line + reference arm, the launch list, ncu --set full of the H update and the Gram.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r2f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_bench_reference.json 2> gpurun_out/r2f_bench_reference.err
timeout 300 python tools/time_updates.py > gpurun_out/r2f_times.txt 2>&1
N="ncu --set full --import-source on --clock-control none -f"
P="python tools/profile_step.py 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_b_ncu.log 2>&1
tail -3 gpurun_out/r2f_pytest_gpu.log; cat gpurun_out/r2f_smoke.log; cat gpurun_out/r2f_times.txt
head -c 400 gpurun_out/r2f_bench.json; echo; head -c 300 gpurun_out/r2f_bench_reference.json; echo
ls -la gpurun_out | grep r2f_
