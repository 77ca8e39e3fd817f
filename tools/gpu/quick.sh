# quick GPU check: parity tests, bench (no CPU baseline), L2 ceilings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value']); print(d['kernels_ms'])"
tail -3 gpurun_out/bench.err
[ -x tools/l2bw_bench.bin ] && timeout 60 ./tools/l2bw_bench.bin | tee gpurun_out/l2_peak.json
