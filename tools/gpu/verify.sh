mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -20 > gpurun_out/v1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1_smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/v1_bench.json 2> gpurun_out/v1_bench.err
timeout 300 python tools/time_updates.py > gpurun_out/v1_times.txt 2>&1
tail -3 gpurun_out/v1_pytest.log; cat gpurun_out/v1_smoke.log; cat gpurun_out/v1_times.txt; head -c 300 gpurun_out/v1_bench.json
