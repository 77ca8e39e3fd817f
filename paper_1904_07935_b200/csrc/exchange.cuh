// The deterministic grid-wide sum exchange used by the persistent W updates
// (update.cu, stream.cu).
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {

// ---------------------------------------------------------------- grid exchange
// Deterministic grid-wide sum for column t.  Each CTA stores its partial into
// every one of kReplicas copies of the column's partial array (NaN until
// written: the value is its own ready flag, so no fences are needed) and bumps
// every replica's arrival counter with a relaxed red; it then polls the
// counter of replica (cta % kReplicas) until all g CTAs have arrived, loads
// that replica's g partials at once (re-polling any slot still NaN) and sums
// them in one fixed order — lane l adds partials l, l+32, ... in a pairwise
// tree, then an xor butterfly over the lanes (warp_sum_all) — so every CTA
// computes the bit-identical sum, run to run.  Replication
// spreads the 148-way read of the same bytes over kReplicas groups of L2
// lines (one copy per ~18 CTAs): with a single copy, those reads serialise at
// the L2 slices and skew the next column's arrivals by ~2.5 us (measured with
// PLNMF_TRACE_EXCHANGE).
// Layout: partials[(t * kReplicas + rep) * stride + cta], counters[(t * kReplicas + rep) * 64].
constexpr int kMaxPartialsPerLane = 8;  // g <= 256 CTAs
constexpr int kReplicas = 8;
constexpr int kCounterStride = 64;      // 256 B between replica counters
constexpr int kTraceSlots = 16;         // PLNMF_TRACE_EXCHANGE stamps per (column, CTA)

__host__ __device__ inline int64_t partial_stride(int g) { return ((g + 31) / 32) * 32 + 32; }
inline int64_t xch_partials(int64_t k, int g) { return k * kReplicas * partial_stride(g); }
inline int64_t xch_counters(int64_t k) { return k * kReplicas * kCounterStride; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Called by one full warp; returns the grid's sum in every lane.  trace (debug,
// PLNMF_TRACE_EXCHANGE): per column and CTA the SM clock at arrival, at
// counter completion, and after the partials are read.
__device__ __forceinline__ double grid_exchange_sum(double blk, int t, int g, double* partials, unsigned* counters,
                                                    unsigned long long* trace = nullptr) {
    static_assert(kMaxPartialsPerLane == 8, "tree8 sums the partials of one lane");
    const int lane = lane_id();
    const int64_t stride = partial_stride(g);
    double* base = partials + (int64_t)t * kReplicas * stride;
    unsigned* cbase = counters + (int64_t)t * kReplicas * kCounterStride;
    unsigned long long* tr = trace ? trace + ((int64_t)t * g + blockIdx.x) * kTraceSlots : nullptr;
    if (tr && lane == 0) tr[0] = clock64();
    if (lane < kReplicas) {
        st_relaxed_f64(base + lane * stride + blockIdx.x, blk);
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cbase + lane * kCounterStride) : "memory");
    }
    const int rep = blockIdx.x % kReplicas;
    if (lane == 0) {
        unsigned n;
        do {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(n) : "l"(cbase + rep * kCounterStride) : "memory");
        } while (n < (unsigned)g);
        if (tr) tr[1] = clock64();
    }
    __syncwarp();
    const double* col = base + rep * stride;
    double v[kMaxPartialsPerLane];
#pragma unroll
    for (int i = 0; i < kMaxPartialsPerLane; ++i)  // all loads in flight at once
        v[i] = (lane + kWarp * i < g) ? ld_relaxed_f64(col + lane + kWarp * i) : 0.0;
    for (;;) {
        bool pending = false;
#pragma unroll
        for (int i = 0; i < kMaxPartialsPerLane; ++i) pending |= isnan(v[i]);
        if (!__any_sync(0xffffffffu, pending)) break;
#pragma unroll
        for (int i = 0; i < kMaxPartialsPerLane; ++i)
            if (isnan(v[i])) v[i] = ld_relaxed_f64(col + lane + kWarp * i);
    }
    const double s = warp_sum_all(tree8(v));
    if (tr && lane == 0) tr[2] = clock64();
    return s;
}

// sqrt of the grid's sum (the column norm, tiled.cpp:137).
__device__ __forceinline__ double grid_exchange(double blk, int t, int g, double* partials, unsigned* counters,
                                                unsigned long long* trace = nullptr) {
    return __dsqrt_rn(grid_exchange_sum(blk, t, g, partials, counters, trace));
}


// NaN-fill the partial slots and zero the arrival counters before a launch.
inline void exchange_reset(cudaStream_t s, int64_t k, int g, double* partials, unsigned* counters) {
    PLNMF_CUDA_CHECK(cudaMemsetAsync(counters, 0, sizeof(unsigned) * (size_t)xch_counters(k), s));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(partials, 0xFF, sizeof(double) * (size_t)xch_partials(k, g), s));
}

}  // namespace plnmf
