// Microbenchmark of grid-wide deterministic sum exchanges (one CTA per SM),
// the per-column critical step of the W update.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/xb tools/exchange_bench.cu && /tmp/xb
#include <cstdio>
#include <cuda_runtime.h>

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

constexpr int MAXL = 8;

// variant 0: acq_rel atomic, last arriver sums, publish, poll total
// variant 1: relaxed atomic + NaN-sentinel partials (no fences), last sums, poll total
// variant 2: all CTAs poll all NaN-sentinel partials (with backoff)
// variant 3: relaxed red arrival; lane 0 polls counter; then all read partials (NaN-guarded)
__device__ volatile int g_stop;

template <int VAR, int REP = 8>
__global__ void xkernel(int ncol, double* partials, unsigned* counters, double* totals, double* out, int sleep_ns,
                        int gap, int busy) {
    const int g = gridDim.x, lane = threadIdx.x & 31;
    double acc = 0;
    if (busy && threadIdx.x >= 64) {  // sibling warps: fp64 work + L2 loads until warp 0 is done
        double x = threadIdx.x, y = 1.0000001;
        const double* src = partials;
        int it = 0;
        while (!g_stop) {
            for (int i = 0; i < 64; ++i) x = fma(x, y, 1e-9);
            if (busy > 1) x += src[(threadIdx.x * 97 + it * 131) % 4096];
            ++it;
        }
        if (threadIdx.x == 64) out[blockIdx.x + gridDim.x] = x;
        return;
    }
    for (int t = 0; t < ncol; ++t) {
        if (gap) {
            const long long t0 = clock64();
            while (clock64() - t0 < gap) {
            }
        }
        const double blk = 1.0 + blockIdx.x + t;
        if (threadIdx.x < 32) {
            double* col = partials + (size_t)t * g;
            double norm = 0;
            if (VAR == 0 || VAR == 1) {
                unsigned prev = 0;
                if (lane == 0) {
                    str(col + blockIdx.x, blk);
                    if (VAR == 0)
                        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counters + t) : "memory");
                    else
                        asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counters + t) : "memory");
                }
                prev = __shfl_sync(~0u, prev, 0);
                if (prev == (unsigned)g - 1) {
                    double v[MAXL];
                    for (int i = 0; i < MAXL; ++i) v[i] = (lane + 32 * i < g) ? ldr(col + lane + 32 * i) : 0.0;
                    for (;;) {
                        bool pend = false;
                        for (int i = 0; i < MAXL; ++i) pend |= isnan(v[i]);
                        if (!__any_sync(~0u, pend)) break;
                        for (int i = 0; i < MAXL; ++i)
                            if (isnan(v[i])) v[i] = ldr(col + lane + 32 * i);
                    }
                    double s = 0;
                    for (int i = 0; i < MAXL; ++i) s += v[i];
                    s = wsum(s);
                    if (lane == 0) str(totals + t, s);
                }
                if (lane == 0) {
                    norm = ldr(totals + t);
                    while (isnan(norm)) {
                        if (sleep_ns) __nanosleep(sleep_ns);
                        norm = ldr(totals + t);
                    }
                }
                norm = __shfl_sync(~0u, norm, 0);
            } else if (VAR == 2) {
                if (lane == 0) str(col + blockIdx.x, blk);
                double v[MAXL];
                for (int i = 0; i < MAXL; ++i) v[i] = (lane + 32 * i < g) ? ldr(col + lane + 32 * i) : 0.0;
                for (;;) {
                    bool pend = false;
                    for (int i = 0; i < MAXL; ++i) pend |= isnan(v[i]);
                    if (!__any_sync(~0u, pend)) break;
                    if (sleep_ns) __nanosleep(sleep_ns);
                    for (int i = 0; i < MAXL; ++i)
                        if (isnan(v[i])) v[i] = ldr(col + lane + 32 * i);
                }
                double s = 0;
                for (int i = 0; i < MAXL; ++i) s += v[i];
                norm = __shfl_sync(~0u, wsum(s), 0);
            } else if (VAR == 4 || VAR == 5) {
                const int stride = ((g + 31) / 32) * 32 + 32;
                double* base = partials + (size_t)t * REP * stride;
                unsigned* cb = counters + (size_t)t * REP * 64;
                if (lane < REP) {
                    str(base + lane * stride + blockIdx.x, blk);
                    if (VAR == 4) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cb + lane * 64) : "memory");
                }
                const int rep = blockIdx.x % REP;
                if (VAR == 4 && lane == 0)
                    while (ldru(cb + rep * 64) < (unsigned)g) {
                    }
                __syncwarp();
                const double* c2 = base + rep * stride;
                double v[MAXL];
                for (int i = 0; i < MAXL; ++i) v[i] = (lane + 32 * i < g) ? ldr(c2 + lane + 32 * i) : 0.0;
                for (;;) {
                    bool pend = false;
                    for (int i = 0; i < MAXL; ++i) pend |= isnan(v[i]);
                    if (!__any_sync(~0u, pend)) break;
                    if (sleep_ns) __nanosleep(sleep_ns);
                    for (int i = 0; i < MAXL; ++i)
                        if (isnan(v[i])) v[i] = ldr(c2 + lane + 32 * i);
                }
                double s = 0;
                for (int i = 0; i < MAXL; ++i) s += v[i];
                norm = __shfl_sync(~0u, wsum(s), 0);
            } else {
                if (lane == 0) {
                    str(col + blockIdx.x, blk);
                    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(counters + t) : "memory");
                    while (ldru(counters + t) < (unsigned)g)
                        if (sleep_ns) __nanosleep(sleep_ns);
                }
                __syncwarp();
                double v[MAXL];
                for (int i = 0; i < MAXL; ++i) v[i] = (lane + 32 * i < g) ? ldr(col + lane + 32 * i) : 0.0;
                for (;;) {
                    bool pend = false;
                    for (int i = 0; i < MAXL; ++i) pend |= isnan(v[i]);
                    if (!__any_sync(~0u, pend)) break;
                    for (int i = 0; i < MAXL; ++i)
                        if (isnan(v[i])) v[i] = ldr(col + lane + 32 * i);
                }
                double s = 0;
                for (int i = 0; i < MAXL; ++i) s += v[i];
                norm = __shfl_sync(~0u, wsum(s), 0);
            }
            acc += norm;
        }
        if (busy) asm volatile("bar.sync 1, 64;"); else __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
    if (busy && threadIdx.x == 0) {
        __threadfence();
        atomicAdd((unsigned*)&counters[ncol * 32 * 64], 1u);
        if (atomicAdd((unsigned*)&counters[ncol * 32 * 64], 0u) == (unsigned)gridDim.x) g_stop = 1;
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ncol = 240, g = sms;
    double *partials, *totals, *out;
    unsigned* counters;
    cudaMalloc(&partials, sizeof(double) * ncol * 32 * (g + 64));
    cudaMalloc(&totals, sizeof(double) * ncol);
    cudaMalloc(&out, sizeof(double) * g);
    cudaMalloc(&counters, sizeof(unsigned) * (ncol * 32 * 64 + 1));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[4] = {"acq_rel atomic + last sums", "relaxed atomic + NaN partials", "all poll all partials",
                            "red arrive + counter poll + read"};
    struct Cfg { int var, sleep, gap, busy, smem; const char* what; void* fn; };
    Cfg cfgs[] = {{3, 0, 2800, 0, 0, "counter+read, 1 copy", (void*)xkernel<3>},
                  {4, 0, 2800, 0, 0, "counter+read, 8 replicas", (void*)xkernel<4, 8>},
                  {4, 0, 2800, 0, 0, "counter+read, 16 replicas", (void*)xkernel<4, 16>},
                  {5, 0, 2800, 0, 0, "all-poll, 8 replicas", (void*)xkernel<5, 8>},
                  {5, 32, 2800, 0, 0, "all-poll, 8 replicas, sleep32", (void*)xkernel<5, 8>},
                  {5, 0, 2800, 0, 0, "all-poll, 16 replicas", (void*)xkernel<5, 16>},
                  {5, 0, 2800, 0, 0, "all-poll, 32 replicas", (void*)xkernel<5, 32>},
                  {5, 0, 0, 0, 0, "all-poll, 16 replicas, no gap", (void*)xkernel<5, 16>},
                  {4, 0, 0, 0, 0, "counter+read, 8 replicas, no gap", (void*)xkernel<4, 8>}};
    for (auto c : cfgs) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(partials, 0xFF, sizeof(double) * ncol * 32 * (g + 64));
            cudaMemset(totals, 0xFF, sizeof(double) * ncol);
            cudaMemset(counters, 0, sizeof(unsigned) * (ncol * 32 * 64 + 1));
            int zero = 0;
            cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
            void* args[] = {(void*)&ncol, &partials, &counters, &totals, &out, &c.sleep, &c.gap, &c.busy};
            void* fn = c.fn;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(fn, g, 512, args, c.smem, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-42s: %7.3f us per column (%s)\n", c.what, best * 1e3 / ncol, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
