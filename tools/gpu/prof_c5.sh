# ncu --set full of one kernel (regex $1) in a C5 iteration on one GPU; raw + source pages
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none -f -k regex:$1 -c 1 -o gpurun_out/one python tools/c5_step.py 1 > gpurun_out/one.log 2>&1
ncu -i gpurun_out/one.ncu-rep --page raw --csv > gpurun_out/one_raw.csv 2>/dev/null
ncu -i gpurun_out/one.ncu-rep --page source --csv > gpurun_out/one_source.csv 2>/dev/null
ncu -i gpurun_out/one.ncu-rep --page details --csv > gpurun_out/one_details.csv 2>/dev/null
tail -2 gpurun_out/one.log
