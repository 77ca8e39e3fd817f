# ncu --set full of the Gram and SpMM kernels on the bench workload; raw pages as CSV
mkdir -p gpurun_out
P="python tools/profile_step.py 2"
N="ncu --set full --import-source on --clock-control none -f"
timeout 600 $N -k regex:gram_block_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_gram $P > gpurun_out/prof_gram.log 2>&1
timeout 600 $N -k regex:spmm_csr --launch-skip 3 -c 1 -o gpurun_out/prof_spmm $P > gpurun_out/prof_spmm.log 2>&1
for r in gram spmm; do ncu -i gpurun_out/prof_$r.ncu-rep --page raw --csv > gpurun_out/raw_$r.csv 2>/dev/null; done
ls -la gpurun_out
