# Round-2 closing profile set (C2 bench workload): the H and W update kernels, the Gram, the
# co-run SpMM, the launch list of a short bench run, and the bench line.
mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none -f"
P="python tools/profile_step.py 2"
timeout 900 $N -k regex:pl_update_kernel --launch-skip 2 -c 1 -o gpurun_out/r2c_hupdate $P > gpurun_out/r2c_hupdate.log 2>&1
timeout 900 $N -k regex:pl_update_kernel --launch-skip 3 -c 1 -o gpurun_out/r2c_wupdate $P > gpurun_out/r2c_wupdate.log 2>&1
timeout 600 $N -k regex:gram_block_kernel --launch-skip 2 -c 1 -o gpurun_out/r2c_gram $P > gpurun_out/r2c_gram.log 2>&1
timeout 600 $N -k regex:spmm_csr_v2 --launch-skip 3 -c 1 -o gpurun_out/r2c_spmm $P > gpurun_out/r2c_spmm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_b_ncu.log 2>&1
for r in hupdate wupdate gram spmm; do
  ncu -i gpurun_out/r2c_$r.ncu-rep --page raw --csv > gpurun_out/r2c_raw_$r.csv 2>/dev/null
done
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
ls -la gpurun_out | grep r2c_
