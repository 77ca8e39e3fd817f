// The W update's per-column chain in isolation (no look-ahead): 6 row warps
// + 1 exchange warp per CTA, one CTA per SM, 240 columns.  Reports SM cycles
// per column for the intra-CTA part (XCH=0: the exchange replaced by a local
// sqrt) and with the engine's grid exchange (XCH=1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1904_07935_b200/csrc \
//        -o tools/chain_bench.bin tools/chain_bench.cu
#include <cstdio>
#include <cstdlib>

#include "exchange.cuh"
#include "lookahead.cuh"

using namespace plnmf;

template <int XCH, int DIV, int EXTRA, int PRE = 0, int TILE = 0>
__global__ void __launch_bounds__(512, 1) chain(int ncol, double* partials, unsigned* counters, double* out,
                                                long long* cyc, const double* add) {
    __shared__ double red[48];
    __shared__ double prodS[16 * 192];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool xw = warp == 6;
    double val = 1.0 + tid * 1e-3, pre = 0.5, c1 = 0.25, u1 = 3.0;
    for (int j = 0; j < 16; ++j) prodS[j * 192 + (tid % 192)] = 1e-3 * j;
    __syncthreads();
    if (tid >= 224) {  // idle warps (the engine's look-ahead group, here without work)
        __syncthreads();
        return;
    }
    const long long t0 = clock64();
    double add1 = 0.0;
    for (int t = 0; t < ncol; ++t) {
        const int tt = t % 16;
        if (EXTRA && !xw) add1 = add[(blockIdx.x * 192 + tid) * 240 + t];
        if (!xw) {
            const double ss = warp_sum_lane0(plnmf::dmul(val, val));
            if (lane == 0) red[warp] = ss;
        }
        named_sync(1, 224);
        if (PRE && !xw) {  // the engine's norm-independent prefix work during the exchange
            double pr = 0.0;
            for (int j = 0; j < 16; ++j) {
                if (j < tt) pr = plnmf::dadd(pr, plnmf::dmul(prodS[j * 192 + (tid % 192)], 0.5));
                if (j > tt) prodS[j * 192 + (tid % 192)] = plnmf::dmul(prodS[j * 192 + (tid % 192)], 1.0);
            }
            pre = pr * 1e-9 + 0.5;
        }
        if (xw) {
            double blk = 0.0;
            if (lane == 0) {
                blk = red[0];
                for (int i = 1; i < 6; ++i) blk = plnmf::dadd(blk, red[i]);
            }
            blk = __shfl_sync(0xffffffffu, blk, 0);
            const double norm = XCH ? grid_exchange(blk, t, gridDim.x, partials, counters) : __dsqrt_rn(blk);
            if (lane == 0) red[40] = norm;
        }
        named_sync(1, 224);
        const double nv = DIV ? clamp_floor(1e-16, __ddiv_rn(val, red[40])) : clamp_floor(1e-16, plnmf::dmul(val, red[40]));
        double s2 = plnmf::dadd(pre, plnmf::dmul(nv, c1));
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j > tt) s2 = plnmf::dadd(s2, prodS[j * 192 + (tid % 192)]);
        val = clamp_floor(1e-16, plnmf::dsub(EXTRA ? plnmf::dadd(u1, add1) : u1, s2)) * 1e-3 + 1.0;
        if (TILE && tt == 15) {  // tile boundary: publish + CTA-wide barriers (idle warps join)
            out[blockIdx.x * 256 + tid] = val;
            named_sync(2, 224);
            named_sync(2, 224);
        }
    }
    const long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    __syncthreads();
    if (val == 12345.0) out[0] = val;
}

int main(int argc, char** argv) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ncol = 240, g = sms;
    double *partials, *out;
    unsigned* counters;
    cudaMalloc(&partials, sizeof(double) * xch_partials(ncol, g));
    cudaMalloc(&counters, sizeof(unsigned) * xch_counters(ncol));
    cudaMalloc(&out, 8 * 256 * 256);
    long long* cyc;
    cudaMalloc(&cyc, 8 * 256);
    double* add;
    cudaMalloc(&add, sizeof(double) * 148 * 192 * 240);
    const char* names[] = {"no exchange, mul", "no exchange, ddiv", "grid exchange, ddiv", "grid exchange, ddiv, LDG",
                           "+ prefix work", "+ prefix + tile barriers"};
    void* fns[] = {(void*)chain<0, 0, 0>, (void*)chain<0, 1, 0>, (void*)chain<1, 1, 0>, (void*)chain<1, 1, 1>,
                   (void*)chain<1, 1, 1, 1>, (void*)chain<1, 1, 1, 1, 1>};
    const int dyn = argc > 1 ? atoi(argv[1]) : 0;  // dynamic smem to shrink L1 like the engine kernel
    for (int v = 0; v < 6; ++v) {
        if (dyn) cudaFuncSetAttribute(fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        for (int rep = 0; rep < 2; ++rep) {
            exchange_reset(0, ncol, g, partials, counters);
            int nc = ncol;
            void* args[] = {&nc, &partials, &counters, &out, &cyc, &add};
            cudaLaunchCooperativeKernel(fns[v], g, 512, args, dyn, 0);
            cudaDeviceSynchronize();
        }
        long long h[256];
        cudaMemcpy(h, cyc, 8 * g, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int c = 0; c < g; ++c) m += h[c];
        printf("%-22s: %.0f SM cycles per column (%s)\n", names[v], m / g / ncol, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
