# Round profile set: one `ncu --set full` capture per hot kernel family on the
# bench workload (C2), the launch list of a short bench run, and the bench line.
mkdir -p gpurun_out
P="python tools/profile_step.py 2"
N="ncu --set full --import-source on --clock-control none -f"
timeout 600 $N -k regex:spmm_csr_kernel --launch-skip 3 -c 1 -o gpurun_out/prof_spmm $P > gpurun_out/prof_spmm.log 2>&1
timeout 600 $N -k regex:gram_block_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_gram $P > gpurun_out/prof_gram.log 2>&1
timeout 900 $N -k regex:pl_update_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_hupdate $P > gpurun_out/prof_hupdate.log 2>&1
timeout 900 $N -k regex:pl_update_kernel --launch-skip 3 -c 1 -o gpurun_out/prof_wupdate $P > gpurun_out/prof_wupdate.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ls -la gpurun_out; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
