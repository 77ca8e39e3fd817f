// Isolated timing of the staged look-ahead GEMM (csrc/lookahead.cuh) at the
// C2 W-update shape, plus fp64 pipe peak probes.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1904_07935_b200/csrc \
//        -o tools/gemm_bench.bin tools/gemm_bench.cu && tools/gemm_bench.bin
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lookahead.cuh"
#include "gemm_variants.cuh"

using namespace plnmf;

// fp64 pipe probe: 8 independent DMUL+DADD (exact) or DFMA chains per thread
template <bool FUSED>
__global__ void fp64_peak(double* out, int iters) {
    double a[8], b = 1.0000001 + threadIdx.x * 1e-9, c = 0.999999;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = FUSED ? __fma_rn(a[i], b, c) : __dadd_rn(__dmul_rn(a[i], b), c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

template <class M, int MODE, int CG = 0, int NI = 1, int KC = 8, int ST = 3>
__global__ void __launch_bounds__(512, 1) gemm_kernel(int nrows_per, int64_t n, int k, int tile, const double* old_m,
                                                      const double* out, const double* qpanel, int nthreads,
                                                      double* sink) {
    extern __shared__ double smem[];
    const int tq = (tile + 7) & ~7, ldt = tile + 1;
    double* q = smem;                       // k x tq
    double* dst = q + k * tq;               // rows x ldt
    double* xbuf = dst + ((nrows_per * ldt + 1) & ~1);
    const int bufd = nrows_per * (KC + 2);
    const int64_t r0 = (int64_t)blockIdx.x * nrows_per;
    const int nrows = (int)max((int64_t)0, min((int64_t)nrows_per, n - r0));
    if ((int)threadIdx.x >= nthreads) return;
    for (int i = threadIdx.x; i < k * tq; i += nthreads) q[i] = qpanel[i];
    named_sync(2, nthreads);
    for (int b = 0; b + tile < k; b += tile) {
        const int bn = b + tile, en = min(bn + tile, k);
        const int wn = en - bn;
        int rg = (nrows * wn + nthreads - 1) / nthreads;
        rg = rg <= 2 ? 2 : rg <= 4 ? 4 : rg <= 6 ? 6 : rg <= 8 ? 8 : rg <= 10 ? 10 : 12;
        GemmArgs ga{dst, ldt, q, tq, bn, en, b, 1, old_m, out, r0, nrows, k, xbuf,
                    bufd, nthreads, (int)threadIdx.x, 2};
        if (CG > 0) {
            lookahead_gemm_rows<M, (CG > 0 ? CG : 2), NI, MODE, KC, ST>(ga);
        } else switch (rg) {
            case 2: lookahead_gemm<M, 2, MODE>(ga); break;
            case 4: lookahead_gemm<M, 4, MODE>(ga); break;
            case 6: lookahead_gemm<M, 6, MODE>(ga); break;
            case 8: lookahead_gemm<M, 8, MODE>(ga); break;
            case 10: lookahead_gemm<M, 10, MODE>(ga); break;
            default: lookahead_gemm<M, 12, MODE>(ga); break;
        }
        named_sync(2, nthreads);
    }
    if (threadIdx.x == 0) sink[blockIdx.x] = dst[0];
}


template <class M, int CG>
__global__ void __launch_bounds__(512, 1) bulk_kernel(int nrows_per, int64_t n, int k, int tile, const double* old_m,
                                                      const double* out, const double* qpanel, int nthreads,
                                                      double* sink) {
    extern __shared__ double smem[];
    const int tq = (tile + 7) & ~7, ldt = tile + 1;
    double* q = smem;                       // k x tq
    double* dst = q + k * tq;               // rows x ldt
    double* bufs = dst + ((nrows_per * ldt + 1) & ~1);
    const int bufd = nrows_per * kBulkKCP;
    __shared__ __align__(8) unsigned long long bars[2 * kBulkStages];
    const int64_t r0 = (int64_t)blockIdx.x * nrows_per;
    const int nrows = (int)max((int64_t)0, min((int64_t)nrows_per, n - r0));
    if ((int)threadIdx.x >= nthreads) return;
    BulkPipe pp{smem_u32(bars), smem_u32(bars + kBulkStages), smem_u32(bufs), bufd, 0};
    if (threadIdx.x == 0) {
        for (int s = 0; s < kBulkStages; ++s) {
            mbar_init(pp.full + 8 * s, 32);
            mbar_init(pp.empty + 8 * s, nthreads / 32 - 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < k * tq; i += nthreads) q[i] = qpanel[i];
    named_sync(2, nthreads);
    for (int b = 0; b + tile < k; b += tile) {
        const int bn = b + tile, en = min(bn + tile, k);
        GemmArgs ga{dst, ldt, q, tq, bn, en, b, 1, old_m, out, r0, nrows, k, bufs, bufd, nthreads,
                    (int)threadIdx.x, 2};
        lookahead_gemm_bulk<M, CG>(ga, pp);
    }
    named_sync(2, nthreads);
    if (threadIdx.x == 0) sink[blockIdx.x] = dst[0];
}

template <class M, int KC, int ST, int TQC = 0, int CG = 16>
__global__ void __launch_bounds__(512, 1) priv_kernel(int nrows_per, int64_t n, int k, int tile, const double* old_m,
                                                      const double* out, const double* qpanel, int nthreads,
                                                      double* sink) {
    extern __shared__ double smem[];
    const int tq = (tile + 7) & ~7, ldt = tile + 1;
    double* q = smem;
    double* dst = q + k * tq;
    double* bufs = dst + ((nrows_per * ldt + 1) & ~1);
    const int bufd = nrows_per * (KC + 2);
    const int64_t r0 = (int64_t)blockIdx.x * nrows_per;
    const int nrows = (int)max((int64_t)0, min((int64_t)nrows_per, n - r0));
    if ((int)threadIdx.x >= nthreads) return;
    for (int i = threadIdx.x; i < k * tq; i += nthreads) q[i] = qpanel[i];
    named_sync(2, nthreads);
    for (int b = 0; b + tile < k; b += tile) {
        const int bn = b + tile, en = min(bn + tile, k);
        GemmArgs ga{dst, ldt, q, tq, bn, en, b, 1, old_m, out, r0, nrows, k, bufs, bufd, nthreads,
                    (int)threadIdx.x, 2};
        lookahead_gemm_private<M, CG, KC, ST, TQC>(ga);
    }
    named_sync(2, nthreads);
    if (threadIdx.x == 0) sink[blockIdx.x] = dst[0];
}

int main(int argc, char** argv) {
    const int only_nt = argc > 1 ? atoi(argv[1]) : 0;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    {
        const int iters = 20000;
        for (int fused = 0; fused < 2; ++fused) {
            for (int warps : {4, 8, 16}) {
                cudaEventRecord(a);
                if (fused) fp64_peak<true><<<sms, warps * 32>>>(sink, iters);
                else fp64_peak<false><<<sms, warps * 32>>>(sink, iters);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                const double ops = (double)sms * warps * 32 * iters * 8 * (fused ? 1 : 2);
                printf("fp64 %s, %2d warps/SM: %.2f Tinstr/s = %.1f lane-ops/clk/SM @1.965GHz\n",
                       fused ? "DFMA     " : "DMUL+DADD", warps, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
            }
        }
    }
    const int V = argc > 2 ? atoi(argv[2]) : 26214, K = 240, T = 16;
    const int rows = (V + sms - 1) / sms;
    std::vector<double> h((size_t)V * K);
    for (size_t i = 0; i < h.size(); ++i) h[i] = 0.5 + (double)((i * 2654435761u) % 1000) / 1000.0;
    double *old_m, *out, *qp;
    cudaMalloc(&old_m, h.size() * 8);
    cudaMalloc(&out, h.size() * 8);
    cudaMalloc(&qp, (size_t)K * 16 * 8);
    cudaMemcpy(old_m, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(out, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(qp, h.data(), (size_t)K * 16 * 8, cudaMemcpyHostToDevice);
    const size_t smem = 8 * ((size_t)K * 16 + ((rows * (T + 1) + 1) & ~1) + 6 * rows * 18);
    auto run = [&](auto kern, const char* what, int nt, bool fused) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            kern<<<(V + rows - 1) / rows, 512, smem>>>(rows, V, K, T, old_m, out, qp, nt, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        double macs = 0;
        for (int bb = 0; bb + T < K; bb += T) macs += (double)V * T * (K - (bb + 2 * T) + bb);
        const double lane_ops = macs * (fused ? 1 : 2);
        printf("lookahead gemm %-22s %3d threads: %7.1f us (%5.1f us/tile), fp64 %.1f%% of peak (%s)\n", what, nt,
               ms * 1e3, ms * 1e3 / (K / T - 1), 100.0 * lane_ops / (ms * 1e-3) / sms / 64 / 1.965e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int nt : {288, 416}) {
        if (only_nt && nt != only_nt) continue;
        run(priv_kernel<MathExact, 16, 2, 16, 16>, "private CG16", nt, false);
        run(priv_kernel<MathExact, 16, 2, 16, 8>, "private CG8", nt, false);
        run(priv_kernel<MathExact, 16, 2, 16, 4>, "private CG4", nt, false);
    }
    return 0;
}
