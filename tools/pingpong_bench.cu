// One-way cross-SM signalling latency: CTA 0 and CTA b ping-pong a counter
// through global memory (st.relaxed / ld.relaxed.gpu polling).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pingpong_bench.bin tools/pingpong_bench.cu
#include <cstdio>
__global__ void pp(unsigned* f, long long* cyc, int iters, int partner) {
    if (threadIdx.x != 0) return;
    if (blockIdx.x != 0 && (int)blockIdx.x != partner) return;
    unsigned* mine = f + (blockIdx.x == 0 ? 0 : 64);
    unsigned* theirs = f + (blockIdx.x == 0 ? 64 : 0);
    const long long t0 = clock64();
    for (unsigned i = 1; i <= (unsigned)iters; ++i) {
        if (blockIdx.x == 0) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(i) : "memory");
            unsigned v;
            do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(theirs) : "memory"); } while (v != i);
        } else {
            unsigned v;
            do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(theirs) : "memory"); } while (v != i);
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(i) : "memory");
        }
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    unsigned* f; long long* cyc;
    cudaMalloc(&f, 4096); cudaMalloc(&cyc, 64);
    for (int partner : {1, 2, 37, 74, 100, 147}) {
        cudaMemset(f, 0, 4096);
        pp<<<148, 32>>>(f, cyc, 1000, partner);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("CTA 0 <-> CTA %3d: %.0f cycles per round trip (one-way ~%.0f) (%s)\n", partner, c / 1000.0, c / 2000.0,
               cudaGetErrorString(cudaGetLastError()));
    }
}
