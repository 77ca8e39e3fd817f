mkdir -p gpurun_out
./tools/xb.bin > gpurun_out/xb.txt 2>&1
PLNMF_PROFILE=1 timeout 300 python tools/profile_step.py 2 > gpurun_out/prof_sections.txt 2>&1
cat gpurun_out/xb.txt gpurun_out/prof_sections.txt
