// Shared-memory load cost probe on sm_100a: SM cycles per warp-level load
// instruction for broadcast / few-address / conflict-free patterns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smem_bench.bin tools/smem_bench.cu
#include <cstdio>

template <int MODE>
__global__ void probe(double* out, int iters, long long* cyc) {
    __shared__ __align__(16) double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // MODE 0: LDS.128 all lanes same address; 1: LDS.128 two addresses (half-warps);
    // 2: LDS.128 32 distinct conflict-free; 3: LDS.64 all same; 4: LDS.64 16 distinct (half-warps equal);
    // 5: LDS.64 32 distinct conflict-free; 6: LDS.128 4 addresses (quarter-warps)
    int off;
    if (MODE == 0 || MODE == 3) off = warp * 2;
    else if (MODE == 1) off = (lane >> 4) * 40 + warp * 2;
    else if (MODE == 6) off = (lane >> 3) * 40 + warp * 2;
    else if (MODE == 2) off = lane * 2;
    else if (MODE == 4) off = (lane & 15);
    else off = lane;
    unsigned acc = 0;
    const unsigned base = (unsigned)__cvta_generic_to_shared(s + off);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const unsigned a = base + ((u * 64 * 8) & 16383);
            if (MODE <= 2 || MODE == 6) {
                unsigned x, y, z, w;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
                acc ^= x ^ w;
            } else {
                unsigned x, y;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
                acc ^= x;
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 12345u) out[0] = acc;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 8 * 1024);
    const char* names[] = {"LDS.128 same addr", "LDS.128 2 addrs (half-warps)", "LDS.128 32 distinct",
                           "LDS.64 same addr", "LDS.64 16 distinct", "LDS.64 32 distinct", "LDS.128 4 addrs (quarters)"};
    void (*fns[])(double*, int, long long*) = {probe<0>, probe<1>, probe<2>, probe<3>, probe<4>, probe<5>, probe<6>};
    const int iters = 2000, warps = 16;
    for (int m = 0; m < 7; ++m) {
        fns[m]<<<148, warps * 32>>>(out, iters, cyc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double per = (double)c / ((double)iters * 16 * warps);
        printf("%-30s: %.2f SM cycles per warp instruction (%s)\n", names[m], per,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
