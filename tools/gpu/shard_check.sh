# Sharded engine on the B200: the test file, then the C5 workload on one GPU via bench.py.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_gpu.py -q -rf 2>&1 | tail -30 > gpurun_out/sharded.log
tail -5 gpurun_out/sharded.log
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -3 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
