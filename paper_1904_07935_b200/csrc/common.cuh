// Shared device helpers for the PL-NMF engine (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace plnmf {

constexpr int kWarp = 32;

// Timing/diagnostic knobs (PLNMF_DBG, PLNMF_PROFILE, PLNMF_TRACE_EXCHANGE, ...)
// exist only in a developer build compiled with -DPLNMF_DEBUG_KNOBS
// (PLNMF_NVCC_EXTRA=-DPLNMF_DEBUG_KNOBS python -m paper_1904_07935_b200.build);
// the production library never reads the environment and its kernels carry
// none of the experiment branches.
#ifdef PLNMF_DEBUG_KNOBS
constexpr bool kDebugKnobs = true;
#else
constexpr bool kDebugKnobs = false;
#endif

// Arithmetic policy.  Exact: separate round-to-nearest multiply and add, the
// reference's Release-build arithmetic (no FMA contraction), so per-element
// sums in the reference's order are bit-identical.  Fused: one fma per term.
struct MathExact {
    static __device__ __forceinline__ double madd(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
};
struct MathFused {
    static __device__ __forceinline__ double madd(double acc, double a, double b) {
        return __fma_rn(a, b, acc);
    }
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// std::max(eps, x) exactly as the reference evaluates it (x only if eps < x;
// a NaN x therefore yields eps, as in proj/src/hals.cpp:61,84).
__device__ __forceinline__ double clamp_floor(double eps, double x) { return (eps < x) ? x : eps; }

__device__ __forceinline__ int lane_id() { return threadIdx.x & (kWarp - 1); }

// Deterministic warp sum: fixed shfl_down tree, result valid in lane 0.
__device__ __forceinline__ double warp_sum_lane0(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = dadd(v, __shfl_down_sync(0xffffffffu, v, off));
    return v;
}

// a / b, correctly rounded, as an out-of-line call: for rare paths inside
// latency-critical loops whose code must stay small (the instruction cache)
static __device__ __noinline__ double div_outlined(double a, double b) { return __ddiv_rn(a, b); }

// Fixed pairwise tree over 8 values (3 dependent adds instead of 7).
__device__ __forceinline__ double tree8(const double (&v)[8]) {
    return dadd(dadd(dadd(v[0], v[1]), dadd(v[2], v[3])), dadd(dadd(v[4], v[5]), dadd(v[6], v[7])));
}

// Deterministic warp sum with the result in every lane: an xor butterfly.
// IEEE addition is commutative, so lanes l and l^off form the same sum at
// every level and all lanes end with identical bits (no broadcast shuffle).
// Shared-memory trees are slower here: the exchange warp shares the MIO pipe
// with the look-ahead warps' shared-memory traffic (measured: +400 us per W
// update with a 32-load tree).
__device__ __forceinline__ double warp_sum_all(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// Deterministic block sum (fixed tree); every thread gets the value.
// scratch must hold >= blockDim.x/32 + 1 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int nwarps = (blockDim.x + 31) >> 5;
    v = warp_sum_lane0(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double s = (lane < nwarps) ? scratch[lane] : 0.0;
        s = warp_sum_lane0(s);
        if (lane == 0) scratch[nwarps] = s;
    }
    __syncthreads();
    return scratch[nwarps];
}

__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace plnmf

#define PLNMF_CUDA_CHECK(expr)                                                    \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) throw ::plnmf::CudaError(_e, #expr, __FILE__, __LINE__); \
    } while (0)
