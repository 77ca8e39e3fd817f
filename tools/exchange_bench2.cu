// Grid-wide deterministic sum exchange variants (one CTA per SM, cooperative),
// the per-column critical step of the W update.  Each column: `gap` cycles of
// per-CTA work (+ jitter), then the exchange; reports us per column.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/exchange_bench2.bin tools/exchange_bench2.cu
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ double ldr(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void str(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned ldru(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double wsum(double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
    return v;
}
constexpr int MAXL = 5;  // g <= 160
constexpr int REP = 8;

__device__ __forceinline__ double ldcg(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
// read g NaN-sentinel slots (lane l: l, l+32, ...), fixed-order sum, all lanes get it
template <bool WEAK = false>
__device__ __forceinline__ double read_sum(const double* col, int g) {
    const int lane = threadIdx.x & 31;
    double v[MAXL];
#pragma unroll
    for (int i = 0; i < MAXL; ++i) v[i] = (lane + 32 * i < g) ? (WEAK ? ldcg(col + lane + 32 * i) : ldr(col + lane + 32 * i)) : 0.0;
    for (;;) {
        bool pend = false;
#pragma unroll
        for (int i = 0; i < MAXL; ++i) pend |= isnan(v[i]);
        if (!__any_sync(~0u, pend)) break;
#pragma unroll
        for (int i = 0; i < MAXL; ++i)
            if (isnan(v[i])) v[i] = ldr(col + lane + 32 * i);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < MAXL; ++i) s += v[i];
    return __shfl_sync(~0u, wsum(s), 0);
}

// VAR 0: 8 replicas, red counters, lane-0 poll, then read partials (the engine's grid_exchange)
// VAR 1: reducer CTA (column t -> CTA t % g) polls all partials, publishes 8 replicas of the total
// VAR 2: 12-way groups: group leaders poll their members, publish group sums; all read the group sums
// VAR 3: all CTAs poll all partials (16 replicas of each slot written by its owner)
template <int VAR>
__global__ void xk(int ncol, double* slots, double* totals, unsigned* counters, double* out, int gap, int jitter,
                   long long* ph) {
    long long p1 = 0, p2 = 0;
    const int g = gridDim.x, lane = threadIdx.x & 31, cta = blockIdx.x;
    double acc = 0;
    if (threadIdx.x >= 32) return;
    const int stride = 192;
    for (int t = 0; t < ncol; ++t) {
        {
            const long long t0 = clock64();
            const int my_gap = gap + (jitter ? (int)(((cta * 7919u + t * 104729u) % 1000u) * jitter / 1000) : 0);
            while (clock64() - t0 < my_gap) {
            }
        }
        const double blk = 1.0 + cta + t;
        double norm;
        if (VAR == 0 || VAR == 5 || VAR == 6) {
            double* base = slots + (size_t)t * REP * stride;
            unsigned* cb = counters + (size_t)t * REP * 64;
            if (lane < REP) {
                str(base + lane * stride + cta, blk);
                if (VAR != 5) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cb + lane * 64) : "memory");
                else asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cb + lane * 64) : "memory");
            }
            const int rep = cta % REP;
            const long long c0 = clock64();
            if (lane == 0) {
                if (VAR != 5) {
                    while (ldru(cb + rep * 64) < (unsigned)g) {
                    }
                } else {
                    unsigned v;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cb + rep * 64) : "memory");
                    } while (v < (unsigned)g);
                }
            }
            __syncwarp();
            const long long c1 = clock64();
            norm = VAR == 6 ? read_sum<true>(base + rep * stride, g) : read_sum(base + rep * stride, g);
            const long long c2 = clock64();
            p1 += c1 - c0;
            p2 += c2 - c1;
        } else if (VAR == 1) {
            double* col = slots + (size_t)t * stride;
            double* tot = totals + (size_t)t * REP * 32;
            if (lane == 0) str(col + cta, blk);
            const int red = t % g;
            if (cta == red) {
                const double s = read_sum(col, g);
                if (lane < REP) str(tot + lane * 32, s);
                norm = s;
            } else {
                double s = 0;
                if (lane == 0) {
                    s = ldr(tot + (cta % REP) * 32);
                    while (isnan(s)) s = ldr(tot + (cta % REP) * 32);
                }
                norm = __shfl_sync(~0u, s, 0);
            }
        } else if (VAR == 2) {
            constexpr int GS = 12;
            const int ng = (g + GS - 1) / GS;
            double* col = slots + (size_t)t * stride;
            double* gsum = totals + (size_t)t * REP * 32;  // REP replicas of ng group sums (ng <= 32)
            if (lane == 0) str(col + cta, blk);
            const int grp = cta / GS;
            if (cta % GS == 0) {  // leader
                const int n = min(GS, g - grp * GS);
                double v = lane < n ? ldr(col + grp * GS + lane) : 0.0;
                while (__any_sync(~0u, isnan(v))) {
                    if (isnan(v)) v = ldr(col + grp * GS + lane);
                }
                const double s = __shfl_sync(~0u, wsum(v), 0);
                if (lane < REP) str(gsum + lane * 32 + grp, s);
            }
            const double* mine = gsum + (cta % REP) * 32;
            double v = lane < ng ? ldr(mine + lane) : 0.0;
            while (__any_sync(~0u, isnan(v))) {
                if (isnan(v)) v = ldr(mine + lane);
            }
            norm = __shfl_sync(~0u, wsum(v), 0);
        } else if (VAR == 4) {
            // private mailboxes: CTA c's column-t box = slots[(t * g + c) * stride + sender]
            for (int dst = lane; dst < g; dst += 32) str(slots + ((size_t)t * g + dst) * stride + cta, blk);
            norm = read_sum(slots + ((size_t)t * g + cta) * stride, g);
        } else {
            constexpr int R3 = 16;
            double* base = slots + (size_t)t * R3 * stride;
            if (lane < R3) str(base + lane * stride + cta, blk);
            norm = read_sum(base + (cta % R3) * stride, g);
        }
        acc += norm;
    }
    if (lane == 0) { out[cta] = acc; ph[2 * cta] = p1; ph[2 * cta + 1] = p2; }
}

int main(int argc, char** argv) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ncol = 240, g = argc > 1 ? atoi(argv[1]) : sms;
    double *slots, *totals, *out;
    unsigned* counters;
    const size_t nslots = (size_t)ncol * 160 * 192, ntot = (size_t)ncol * REP * 32;
    cudaMalloc(&slots, nslots * 8);
    cudaMalloc(&totals, ntot * 8);
    cudaMalloc(&out, sizeof(double) * g);
    cudaMalloc(&counters, sizeof(unsigned) * ncol * REP * 64);
    long long* ph;
    cudaMalloc(&ph, 16 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"counter + read partials (engine)", "reducer CTA + broadcast", "12-way group leaders",
                           "all-poll, 16 replicas", "private mailboxes", "counter release/acquire", "counter, weak .cg partial reads"};
    void* fns[] = {(void*)xk<0>, (void*)xk<1>, (void*)xk<2>, (void*)xk<3>, (void*)xk<4>, (void*)xk<5>, (void*)xk<6>};
    for (int gap : {0, 1000}) {
        for (int jit : {0, 300}) {
            if (gap == 0 && jit) continue;
            for (int v = 0; v < 7; ++v) {
                float best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaMemset(slots, 0xFF, nslots * 8);
                    cudaMemset(totals, 0xFF, ntot * 8);
                    cudaMemset(counters, 0, sizeof(unsigned) * ncol * REP * 64);
                    int nc = ncol;
                    void* args[] = {&nc, &slots, &totals, &counters, &out, &gap, &jit, &ph};
                    cudaEventRecord(a);
                    cudaLaunchCooperativeKernel(fns[v], g, 512, args, 0, 0);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                long long hp[2 * 160];
                cudaMemcpy(hp, ph, sizeof(long long) * 2 * g, cudaMemcpyDeviceToHost);
                double m1 = 0, m2 = 0;
                for (int c = 0; c < g; ++c) { m1 += hp[2 * c]; m2 += hp[2 * c + 1]; }
                printf("gap %4d jitter %3d  %-34s: %6.3f us/column (%s)", gap, jit, names[v], best * 1e3 / ncol,
                       cudaGetErrorString(cudaGetLastError()));
                if (v == 0 || v >= 5) printf("  poll %.0f cyc, read %.0f cyc per column", m1 / g / ncol, m2 / g / ncol);
                printf("\n");
            }
        }
    }
    return 0;
}
