# Round-2 profile set: ncu --set full of each hot kernel family (C2 bench workload, the C4
# tensor-core GEMM, the C5 SpMM and sharded W update), the bench launch list, bench lines.
mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none -f"
P="python tools/profile_step.py 2"
timeout 600 $N -k regex:spmm_csr_kernel --launch-skip 3 -c 1 -o gpurun_out/r2_spmm $P > gpurun_out/r2_spmm.log 2>&1
timeout 600 $N -k regex:gram_block_kernel --launch-skip 2 -c 1 -o gpurun_out/r2_gram $P > gpurun_out/r2_gram.log 2>&1
timeout 900 $N -k regex:pl_update_kernel --launch-skip 2 -c 1 -o gpurun_out/r2_hupdate $P > gpurun_out/r2_hupdate.log 2>&1
timeout 900 $N -k regex:pl_update_kernel --launch-skip 3 -c 1 -o gpurun_out/r2_wupdate $P > gpurun_out/r2_wupdate.log 2>&1
timeout 900 $N -k regex:ozaki -c 2 -o gpurun_out/r2_ozaki python tools/tensor_step.py > gpurun_out/r2_ozaki.log 2>&1
timeout 1200 ncu --set full --clock-control none -f -k regex:spmm_csr_kernel -c 1 -o gpurun_out/r2_c5_spmm python tools/c5_step.py 1 > gpurun_out/r2_c5_spmm.log 2>&1
timeout 1200 ncu --set full --clock-control none -f -k regex:stream_update_kernel -c 2 -o gpurun_out/r2_c5_update python tools/c5_step.py 1 > gpurun_out/r2_c5_update.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b_ncu.log 2>&1
for r in spmm gram hupdate wupdate ozaki c5_spmm c5_update; do
  ncu -i gpurun_out/r2_$r.ncu-rep --page raw --csv > gpurun_out/r2_raw_$r.csv 2>/dev/null
done
ls -la gpurun_out | tail -30
