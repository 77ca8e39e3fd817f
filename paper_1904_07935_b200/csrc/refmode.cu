// Math::reference_order — the reductions of the W update and of the error in
// the reference's own summation order, so whole iterate() trajectories are
// bit-identical to the reference.  A verification mode:
// every other kernel already reproduces the reference's per-element order
// (SpMM, Gram, both H updaters, init/phase 1/phase 2 values/phase 3); only
// these sums differ in the fast path, where they are fixed-order trees.
//
//   ordered_ss      column t's sum of squares as the reference forms it:
//                   nth = 1: one serial sum over the rows, v ascending
//                   (update_w_reference, proj/src/hals.cpp:97-100);
//                   nth > 1: the tiled path's per-OpenMP-thread partials —
//                   thread i sums rows [i*chunk, (i+1)*chunk) serially with
//                   chunk = ceil(n/nth), then the partials are added in thread
//                   order starting from 0.0 (proj/src/tiled.cpp:103-106,
//                   129-142).  Each term is RN(val*val), then RN(+) (no FMA).
//   ref_w_values    column kk of update_w_reference before its normalisation
//                   (hals.cpp:88-96), one thread per row.
//   serial_dot_cm   sum_i a[i]*b[i] over the column-major order of two
//                   row-major matrices, one serial chain
//                   (relative_error_gram's pw / sq loops, metrics.cpp:104-115).
//                   The block stages products (exact RN multiplies) in shared
//                   memory; thread 0 adds them in order.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

constexpr int kOrderedMaxThreads = 1024;

__global__ void __launch_bounds__(kOrderedMaxThreads) ordered_ss_kernel(int64_t n, int k, int t, int nth,
                                                                        const double* __restrict__ col_src,
                                                                        double* __restrict__ ss_out) {
    __shared__ double part[kOrderedMaxThreads];
    const int i = threadIdx.x;
    if (i < nth) {
        const int64_t chunk = (n + nth - 1) / nth;
        const int64_t v0 = std::min<int64_t>(n, (int64_t)i * chunk);
        const int64_t v1 = std::min<int64_t>(n, v0 + chunk);
        const double* src = col_src + t;
        double s = 0.0;
        int64_t v = v0;
        // loads run ahead of the dependent adds: 8 in flight per step
        for (; v + 8 <= v1; v += 8) {
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = __ldg(src + (v + u) * k);
#pragma unroll
            for (int u = 0; u < 8; ++u) s = dadd(s, dmul(x[u], x[u]));
        }
        for (; v < v1; ++v) {
            const double x = __ldg(src + v * k);
            s = dadd(s, dmul(x, x));
        }
        part[i] = s;
    }
    __syncthreads();
    if (i == 0) {
        double tot = 0.0;
        for (int j = 0; j < nth; ++j) tot = dadd(tot, part[j]);
        *ss_out = tot;
    }
}

constexpr int kRefValThreads = 128;

__global__ void __launch_bounds__(kRefValThreads) ref_w_values_kernel(int64_t v, int k, int kk, double eps,
                                                                      double* __restrict__ w,
                                                                      const double* __restrict__ p,
                                                                      const double* __restrict__ q) {
    const int64_t row = (int64_t)blockIdx.x * kRefValThreads + threadIdx.x;
    if (row >= v) return;
    double* wr = w + row * k;
    const double qkk = __ldg(q + (int64_t)kk * k + kk);
    double dot = 0.0;
    for (int j = 0; j < k; ++j) dot = dadd(dot, dmul(wr[j], __ldg(q + (int64_t)j * k + kk)));
    wr[kk] = clamp_floor(eps, dsub(dadd(dmul(wr[kk], qkk), p[row * k + kk]), dot));  // hals.cpp:95
}

constexpr int kDotThreads = 256, kDotChunk = 4096;

__global__ void __launch_bounds__(kDotThreads) serial_dot_cm_kernel(int64_t rows, int64_t cols,
                                                                    const double* __restrict__ a,
                                                                    const double* __restrict__ b,
                                                                    double* __restrict__ out) {
    __shared__ double buf[kDotChunk];
    const int64_t n = rows * cols;
    double s = 0.0;
    for (int64_t base = 0; base < n; base += kDotChunk) {
        const int m = (int)std::min<int64_t>(kDotChunk, n - base);
        for (int j = threadIdx.x; j < m; j += kDotThreads) {
            const int64_t i = base + j;  // column-major element i = (i % rows, i / rows)
            const int64_t r = i % rows, c = i / rows;
            buf[j] = dmul(a[r * cols + c], b[r * cols + c]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int j = 0;
            for (; j + 8 <= m; j += 8) {
                double x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = buf[j + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) s = dadd(s, x[u]);
            }
            for (; j < m; ++j) s = dadd(s, buf[j]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s;
}

}  // namespace

namespace kern {

int ordered_ss(cudaStream_t s, int64_t n, int64_t k, int64_t t, int nth, const double* col_src, double* ss_out) {
    if (nth < 1 || nth > kOrderedMaxThreads)
        throw std::invalid_argument("reference-order norm: thread count must be in [1, 1024]");
    const int threads = ((nth + 31) / 32) * 32;
    ordered_ss_kernel<<<1, threads, 0, s>>>(n, (int)k, (int)t, nth, col_src, ss_out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int ref_w_values(cudaStream_t s, int64_t v, int64_t k, int64_t kk, double eps, double* w, const double* p,
                 const double* q) {
    if (v <= 0) return 0;
    ref_w_values_kernel<<<(unsigned)((v + kRefValThreads - 1) / kRefValThreads), kRefValThreads, 0, s>>>(
        v, (int)k, (int)kk, eps, w, p, q);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int serial_dot_colmajor(cudaStream_t s, int64_t rows, int64_t cols, const double* a, const double* b, double* out) {
    serial_dot_cm_kernel<<<1, kDotThreads, 0, s>>>(rows, cols, a, b, out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

}  // namespace kern
}  // namespace plnmf
