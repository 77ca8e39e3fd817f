// The engine's exact W-chain column loop (update_kern.cuh), ported verbatim
// into a standalone cooperative kernel (no look-ahead): 16 warps per CTA (6
// row warps + 1 exchange warp + 9 idle), 178 rows per CTA, smem layout as the
// engine's, 15 tiles of 16 columns.  Used to bisect the in-kernel cost of
// the chain against tools/chain_bench.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1904_07935_b200/csrc -I include \
//        -o tools/chain_bench2.bin tools/chain_bench2.cu
#include <cstdio>
#include <cstdlib>

#include "exchange.cuh"
#include "lookahead.cuh"

using namespace plnmf;

struct Args {
    int64_t n;
    int k, T, R;
    double eps;
    const double* add;
    double* out;
    double* norms;
    double* partials;
    unsigned* counters;
    int xch, flags;
};

template <int TM>
__global__ void __launch_bounds__(512, 1) chain2(Args p) {
    extern __shared__ double smem[];
    const int T = p.T, k = p.k, R = p.R, ldt = T + 1;
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int nrows = (int)((r0 + R < p.n) ? R : (p.n > r0 ? p.n - r0 : 0));
    const int tid = threadIdx.x;
    const int row_warps = min(8, max(1, (R + 31) / 32));
    const int nrowt = row_warps * 32, nchain = (row_warps + 1) * 32, nupd = 512 - nchain;
    const bool is_chain = tid >= nupd;
    const int ctid = tid - nupd;
    const bool is_xwarp = ctid >= nrowt;
    double* A = smem;
    double* oldB = A + (int64_t)R * ldt;
    double* sqc = oldB + (int64_t)R * ldt;
    double* red = sqc + T * T;
    double* prodS = red + 48;
    for (int i = tid; i < R * ldt * 2 + T * T; i += 512) smem[i] = 1.0 + 1e-6 * (i % 97);
    __syncthreads();
    double add_carry = 0.0;
    for (int b = 0; b < k; b += T) {
        const int e = min(b + T, k), w = e - b;
        const bool has_next = e < k;
        if (is_chain) {
            const int r = ctid;
            const bool own = !is_xwarp && r < nrows;
            double* prod = prodS + r;
            double* arow = A + r * ldt;
            const double* addr = p.add + (r0 + r) * k + b;
            const double* orow = oldB + r * ldt;
            double val = 0.0;
            {
                const double add0 = b == 0 ? (own ? addr[0] : 0.0) : add_carry;
                if (own) {
                    double s = 0.0;
#pragma unroll
                    for (int j = 0; j < TM; ++j)
                        if (j < w) s = plnmf::dadd(s, plnmf::dmul(orow[j], sqc[j * T]));
                    val = clamp_floor(p.eps, plnmf::dsub(plnmf::dadd(arow[0], add0), s));
                }
            }
#pragma unroll 1
            for (int tt = 0; tt < w; ++tt) {
                const bool more = tt + 1 < w;
                if (!is_xwarp) {
                    const double ss = (p.flags & 128) ? val : warp_sum_lane0(plnmf::dmul(val, val));
                    if (lane_id() == 0) red[ctid >> 5] = ss;
                }
                named_sync(1, nchain);
                double pre = 0.0, c1 = 0.0, u1 = 0.0;
                if (is_xwarp) {
                    double blk = 0.0;
                    if (lane_id() == 0) {
                        blk = red[0];
                        if (p.flags & 4) {
#pragma unroll
                            for (int i = 1; i < 6; ++i) blk = plnmf::dadd(blk, red[i]);
                        } else {
                            for (int i = 1; i < row_warps; ++i) blk = plnmf::dadd(blk, red[i]);
                        }
                    }
                    blk = __shfl_sync(0xffffffffu, blk, 0);
                    const double norm = p.xch ? grid_exchange(blk, b + tt, gridDim.x, p.partials, p.counters)
                                              : __dsqrt_rn(blk);
                    if (lane_id() == 0) {
                        red[40] = norm;
                        if (p.flags & 256) red[41] = __drcp_rn(norm);
                        if (blockIdx.x == 0) p.norms[b + tt] = norm;
                    }
                } else if (own && !more && has_next) {
                    add_carry = addr[w];
                } else if (own && more && !(p.flags & 1)) {
#pragma unroll
                    for (int j = 0; j < TM; ++j)
                        if (j < tt) pre = plnmf::dadd(pre, plnmf::dmul(arow[j], sqc[j * T + tt + 1]));
#pragma unroll
                    for (int j = 0; j < TM; ++j)
                        if (j > tt && j < w) prod[j * R] = plnmf::dmul(orow[j], sqc[j * T + tt + 1]);
                    c1 = sqc[tt * T + tt + 1];
                    u1 = plnmf::dadd(arow[tt + 1], addr[tt + 1]);
                }
                named_sync(1, nchain);
                double nv;
                if (p.flags & 64) {
                    nv = clamp_floor(p.eps, plnmf::dmul(val, red[40]));
                } else if (p.flags & 256) {  // reciprocal + one fma correction (Markstein)
                    const double bn = red[40], y = red[41];
                    const double q0 = __dmul_rn(val, y);
                    const double rr = __fma_rn(-q0, bn, val);
                    nv = clamp_floor(p.eps, __fma_rn(rr, y, q0));
                } else {
                    nv = clamp_floor(p.eps, __ddiv_rn(val, red[40]));
                }
                if (own) {
                    if (!(p.flags & 8)) arow[tt] = nv;
                    if (more) {
                        double s2 = plnmf::dadd(pre, plnmf::dmul(nv, c1));
                        if (p.flags & 16) {
                            for (int j = tt + 1; j < w; ++j) s2 = plnmf::dadd(s2, prod[j * R]);
                        } else if (!(p.flags & 32)) {
#pragma unroll
                            for (int j = 0; j < TM; ++j)
                                if (j > tt && j < w) s2 = plnmf::dadd(s2, prod[j * R]);
                        }
                        val = clamp_floor(p.eps, plnmf::dsub(u1, s2));
                    }
                }
            }
            named_sync(1, nchain);
            if (!(p.flags & 2))
                for (int idx = ctid; idx < nrows * w; idx += nchain) {
                    const int rr = idx / w, j = idx % w;
                    p.out[(r0 + rr) * k + b + j] = A[rr * ldt + j];
                }
        }
        __syncthreads();
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int V = 26214, K = 240, T = 16, R = (V + sms - 1) / sms;
    double *add, *out, *norms, *partials;
    unsigned* counters;
    cudaMalloc(&add, sizeof(double) * V * K);
    cudaMalloc(&out, sizeof(double) * V * K);
    cudaMalloc(&norms, sizeof(double) * K);
    cudaMalloc(&partials, sizeof(double) * xch_partials(K, sms));
    cudaMalloc(&counters, sizeof(unsigned) * xch_counters(K));
    cudaMemset(add, 0, sizeof(double) * V * K);
    const size_t smem = sizeof(double) * (2 * R * (T + 1) + T * T + 48 + R * T);
    cudaFuncSetAttribute(chain2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int xch : {0, 1})
        for (int flags : {0, 3, 3 | 4, 3 | 256, 3 | 4 | 256}) {
            Args p{V, K, T, R, 1e-16, add, out, norms, partials, counters, xch, flags};
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                exchange_reset(0, K, sms, partials, counters);
                void* args[] = {&p};
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void*)chain2<16>, sms, 512, args, smem, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            printf("exchange %d flags %3d (1 prefix 2 publish 4 unroll-red 8 arow 16 loop-s2 32 no-s2 64 no-div 128 no-wsum): %.1f us = %.0f cycles/column (%s)\n",
                   xch, flags, best * 1e3, best * 1e-3 * 1.965e9 / K, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
