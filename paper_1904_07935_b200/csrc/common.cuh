// Shared device helpers for the PL-NMF engine (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace plnmf {

constexpr int kWarp = 32;

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
