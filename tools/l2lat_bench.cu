// Round-trip latency of the load/atomic flavours usable for cross-SM polling
// (dependent chain on one L2-resident word).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2lat_bench.bin tools/l2lat_bench.cu
#include <cstdio>

template <int OP>
__global__ void lat(unsigned* p, long long* cyc, int iters) {
    unsigned idx = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned v;
        unsigned* a = p + (idx & 1) * 64;  // 0 in practice (words hold 0): a dependent chain
        if (OP == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
        if (OP == 1) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
        if (OP == 2) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
        if (OP == 3) asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 0;" : "=r"(v) : "l"(a) : "memory");
        if (OP == 4) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
        if (OP == 5) asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
        if (OP == 6) asm volatile("ld.relaxed.cluster.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
        idx += v;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (idx == 12345) p[1000] = idx;
}

int main() {
    unsigned* p;
    long long* cyc;
    cudaMalloc(&p, 1 << 20);
    cudaMemset(p, 0, 1 << 20);
    cudaMalloc(&cyc, 8 * 256);
    const char* names[] = {"ld.relaxed.gpu", "ld.volatile", "ld.global.cg", "atom.add 0 (relaxed.gpu)", "ld.acquire.gpu",
                           "ld.global.cv", "ld.relaxed.cluster"};
    void (*fns[])(unsigned*, long long*, int) = {lat<0>, lat<1>, lat<2>, lat<3>, lat<4>, lat<5>, lat<6>};
    for (int i = 0; i < 7; ++i) {
        for (int blocks : {1, 148}) {
            fns[i]<<<blocks, 32>>>(p, cyc, 2000);
            cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
            double m = 0, mx = 0;
            for (int b = 0; b < blocks; ++b) { m += h[b]; mx = h[b] > mx ? h[b] : mx; }
            printf("%-26s %3d CTAs: %.0f cycles mean (max %.0f) per dependent access (%s)\n", names[i], blocks,
                   m / blocks / 2000, mx / 2000, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
