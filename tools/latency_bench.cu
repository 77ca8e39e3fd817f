// Dependent-chain latency of the chain's critical-path operations on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency_bench.bin tools/latency_bench.cu
#include <cstdio>

template <int OP>
__global__ void lat(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x * 1e-12;
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        if (OP == 0) x = __dadd_rn(x, b);
        if (OP == 1) x = __dmul_rn(x, b);
        if (OP == 2) x = __fma_rn(x, b, a);
        if (OP == 3) x = __ddiv_rn(b, x);
        if (OP == 4) x = __dsqrt_rn(x + 1.5);
        if (OP == 5) x = __shfl_down_sync(~0u, x, 1) + 0.0;
        if (OP == 6) x = __dadd_rn(x, __shfl_down_sync(~0u, x, 16));
        if (OP == 7) x = (x > b) ? x : b;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (x == 1234.5) out[0] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 64);
    const char* names[] = {"DADD", "DMUL", "DFMA", "DDIV (__ddiv_rn)", "DSQRT (__dsqrt_rn)", "SHFL.f64 (+0)",
                           "DADD(SHFL)", "max (DSETP+SEL)"};
    void (*fns[])(double*, long long*, double, double) = {lat<0>, lat<1>, lat<2>, lat<3>, lat<4>, lat<5>, lat<6>, lat<7>};
    for (int i = 0; i < 8; ++i) {
        fns[i]<<<1, 32>>>(out, cyc, 1.000001, 0.9999999);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-20s: %.1f cycles per dependent op\n", names[i], c / 1024.0);
    }
    return 0;
}
