# A/B of the update kernels: HEAD (built in _ab/) vs the working tree, then the WT parity tests for the updates
mkdir -p gpurun_out
for i in 1 2 3; do
echo "HEAD $(cd _ab && python tools/time_updates.py 2>&1 | grep -E "update W|update H|gram|iteration" | tr -s " " | tr "\n" " ")"
echo "WT   $(python tools/time_updates.py 2>&1 | grep -E "update W|update H|gram|iteration" | tr -s " " | tr "\n" " ")"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_configs.py -m gpu -x -q 2>&1 | tail -3
