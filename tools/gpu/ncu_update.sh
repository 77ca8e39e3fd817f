# ncu --set full of the W (NORMALIZE=1) and H tiled update kernels on the bench workload
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pl_update_kernel -c 2 \
  -o gpurun_out/prof_update -f python tools/profile_step.py 1 > gpurun_out/ncu_update.log 2>&1
tail -5 gpurun_out/ncu_update.log
