# Round-2 closing set (after the Gram ragged-tile and H full-tile changes): full GPU suite, smoke,
# bench line + reference arm, the launch list, ncu --set full of the H update and the Gram.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r2d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2d_bench_reference.json 2> gpurun_out/r2d_bench_reference.err
timeout 300 python tools/time_updates.py > gpurun_out/r2d_times.txt 2>&1
N="ncu --set full --import-source on --clock-control none -f"
P="python tools/profile_step.py 2"
timeout 900 $N -k regex:pl_update_kernel --launch-skip 2 -c 1 -o gpurun_out/r2d_hupdate $P > gpurun_out/r2d_hupdate.log 2>&1
timeout 600 $N -k regex:gram_block_kernel --launch-skip 2 -c 1 -o gpurun_out/r2d_gram $P > gpurun_out/r2d_gram.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2d_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_b_ncu.log 2>&1
for r in hupdate gram; do ncu -i gpurun_out/r2d_$r.ncu-rep --page raw --csv > gpurun_out/r2d_raw_$r.csv 2>/dev/null; done
tail -3 gpurun_out/r2d_pytest_gpu.log; cat gpurun_out/r2d_smoke.log; cat gpurun_out/r2d_times.txt
head -c 400 gpurun_out/r2d_bench.json; echo; head -c 300 gpurun_out/r2d_bench_reference.json; echo
ls -la gpurun_out | grep r2d_
