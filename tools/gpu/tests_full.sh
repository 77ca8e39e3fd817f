# Full GPU test suite (no -x: every failure is listed), then smoke.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40 > gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -12 gpurun_out/pytest_gpu_full.log; cat gpurun_out/smoke.log
