// FP64 SIMT GEMM-loop probe: one thread = one row x CG columns, operands in
// shared memory (no staging, no barriers), exact DMUL+DADD per term.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_loop_bench.bin tools/fp64_loop_bench.cu
#include <cstdio>

template <int CG, int PF>
__global__ void __launch_bounds__(512, 1) loop(int kdim, int reps, double* out) {
    extern __shared__ __align__(16) double sm[];
    double* q = sm;                      // kdim x 16
    double* x = sm + kdim * 16;          // rows x (kdim + 2)
    const int ld = kdim + 2;
    for (int i = threadIdx.x; i < kdim * 16 + blockDim.x * ld; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
    __syncthreads();
    const int ncg = 16 / CG;
    const int r = threadIdx.x / ncg, c0 = (threadIdx.x % ncg) * CG;
    double a[CG];
#pragma unroll
    for (int u = 0; u < CG; ++u) a[u] = 0;
    const double* xr = x + r * ld;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
        for (int kk = 0; kk < kdim; kk += 2) {
            const double2 xx = *reinterpret_cast<const double2*>(xr + kk);
            const double* q0 = q + kk * 16 + c0;
#pragma unroll
            for (int u = 0; u < CG; u += 2) {
                const double2 qa = *reinterpret_cast<const double2*>(q0 + u);
                const double2 qb = *reinterpret_cast<const double2*>(q0 + 16 + u);
                a[u] = __dadd_rn(a[u], __dmul_rn(-qa.x, xx.x));
                a[u + 1] = __dadd_rn(a[u + 1], __dmul_rn(-qa.y, xx.x));
                a[u] = __dadd_rn(a[u], __dmul_rn(-qb.x, xx.y));
                a[u + 1] = __dadd_rn(a[u + 1], __dmul_rn(-qb.y, xx.y));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int u = 0; u < CG; ++u) s += a[u];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int kdim = 96, reps = 200;
    auto run = [&](auto fn, int cg, int threads) {
        const size_t smem = 8 * ((size_t)kdim * 16 + (size_t)threads * (kdim + 2));
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int i = 0; i < 2; ++i) {
            cudaEventRecord(e0);
            fn<<<sms, threads, smem>>>(kdim, reps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double lane_ops = (double)sms * threads * reps * kdim * cg * 2;
        printf("CG%2d %3d threads (%2d warps): %.1f%% of fp64 peak (%s)\n", cg, threads, threads / 32,
               100.0 * lane_ops / (ms * 1e-3) / sms / 64 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    };
    for (int t : {128, 192, 256, 384}) {
        run(loop<16, 0>, 16, t);
        run(loop<8, 0>, 8, t);
        run(loop<4, 0>, 4, t);
    }
    return 0;
}
