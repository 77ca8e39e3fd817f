# All microbenchmarks behind DESIGN.md's W-chain / GEMM analysis; output -> gpurun_out/microbench.txt
mkdir -p gpurun_out
o=gpurun_out/microbench.txt
: > $o
for b in latency_bench l2lat_bench pingpong_bench smem_bench exchange_bench2 chain_bench cluster_probe; do
  echo "==== tools/$b.cu" >> $o; timeout 120 ./tools/$b.bin >> $o 2>&1
done
echo "==== tools/gemm_bench.cu (H shape: 416 threads, V=11314)" >> $o; timeout 120 ./tools/gemm_bench.bin 416 11314 >> $o 2>&1
echo "==== tools/gemm_bench.cu (W shape: 288 threads, V=26214)" >> $o; timeout 120 ./tools/gemm_bench.bin 288 26214 >> $o 2>&1
echo "==== tools/div_check.cu" >> $o; timeout 300 ./tools/div_check.bin >> $o 2>&1
wc -l $o
