// Column-stepped pieces of the tiled W update, one launch per piece, for the
// reference-order verification mode (Math::reference_order, refmode.cu /
// engine.cu: update_w_reference_order), which forms each column's norm in the
// reference's own summation order between the steps:
//
//   shard_col_step   phase 2 of column t (tiled.cpp:103-128): writes the clamped
//                    values and a fixed-order partial sum of squares
//   shard_normalize  norm = sqrt(sum of the given partials in order), column t /=
//                    norm, clamp (tiled.cpp:137-146)
//   shard_phase3     the tile's phase-3 rank-T update (tiled.cpp:158-174)
// Phase A (init + phase 1) is the streaming path's stream_phase_a.
#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

constexpr int kColThreads = 256;
constexpr int kColBlocks = 296;

template <class M>
__global__ void __launch_bounds__(kColThreads) col_step_kernel(int64_t n, int k, int b, int e, int t, double eps,
                                                               const double* __restrict__ old_m, double* nb,
                                                               const double* __restrict__ coeff,
                                                               const double* __restrict__ add,
                                                               double* __restrict__ partials) {
    __shared__ double red[40];
    const int tt = t - b, w = e - b;
    double ss = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * kColThreads + threadIdx.x; r < n; r += (int64_t)gridDim.x * kColThreads) {
        const double* nr = nb + r * k + b;
        const double* orow = old_m + r * k + b;
        double s = 0.0;
        for (int j0 = 0; j0 < w; j0 += 8) {
            double x[8], c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = j0 + u;
                x[u] = (j < w) ? (j < tt ? nr[j] : orow[j]) : 0.0;
                c[u] = (j < w) ? __ldg(coeff + (int64_t)(b + j) * k + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (j0 + u < w) s = M::madd(s, x[u], c[u]);
        }
        const double val = clamp_floor(eps, dsub(dadd(nr[tt], add[r * k + t]), s));
        nb[r * k + t] = val;
        ss = M::madd(ss, val, val);
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = ss;
}

__global__ void sum_fixed_kernel(int n, const double* __restrict__ x, double* __restrict__ out) {
    __shared__ double red[40];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s = dadd(s, x[i]);
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

// world_partials[0..world) summed in rank order -> norm; normalise column t.
__global__ void normalize_col_kernel(int64_t n, int k, int t, double eps, int world,
                                     const double* __restrict__ world_partials, double* nb,
                                     double* __restrict__ norms) {
    double s = 0.0;
    for (int i = 0; i < world; ++i) s = dadd(s, world_partials[i]);
    const double norm = __dsqrt_rn(s);
    if (blockIdx.x == 0 && threadIdx.x == 0) norms[t] = norm;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        double* x = nb + r * k + t;
        *x = clamp_floor(eps, __ddiv_rn(*x, norm));
    }
}

template <class M>
__global__ void __launch_bounds__(256) phase3_kernel(int64_t n, int k, int b, int e, double* nb,
                                                     const double* __restrict__ coeff) {
    const int w = e - b, rest = k - e;
    const int ng = (rest + 3) / 4;
    const int64_t items = n * ng;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = it / ng;
        const int c0 = e + (int)(it % ng) * 4;
        double* row = nb + r * k;
        double a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = (c0 + u < k) ? row[c0 + u] : 0.0;
        for (int j0 = 0; j0 < w; j0 += 8) {
            double x[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) x[v] = (j0 + v < w) ? row[b + j0 + v] : 0.0;
#pragma unroll
            for (int v = 0; v < 8; ++v)
                if (j0 + v < w) {
                    const double* cf = coeff + (int64_t)(b + j0 + v) * k + c0;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (c0 + u < k) a[u] = M::madd(a[u], -1.0 * __ldg(cf + u), x[v]);
                }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (c0 + u < k) row[c0 + u] = a[u];
    }
}

}  // namespace

namespace kern {

int shard_col_step(cudaStream_t s, Math m, int64_t n, int64_t k, int64_t b, int64_t e, int64_t t, double eps,
                   const double* old_m, double* nb, const double* coeff, const double* add, double* block_partials,
                   double* ss_out) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(kColBlocks, (n + kColThreads - 1) / kColThreads));
    if (m == Math::exact)
        col_step_kernel<MathExact><<<grid, kColThreads, 0, s>>>(n, (int)k, (int)b, (int)e, (int)t, eps, old_m, nb,
                                                                coeff, add, block_partials);
    else
        col_step_kernel<MathFused><<<grid, kColThreads, 0, s>>>(n, (int)k, (int)b, (int)e, (int)t, eps, old_m, nb,
                                                                coeff, add, block_partials);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    if (!ss_out) return 1;  // reference-order mode forms the sum itself (refmode.cu)
    sum_fixed_kernel<<<1, 256, 0, s>>>((int)grid, block_partials, ss_out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 2;
}

int shard_normalize(cudaStream_t s, int64_t n, int64_t k, int64_t t, double eps, int world,
                    const double* world_partials, double* nb, double* norms) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256));
    normalize_col_kernel<<<grid, 256, 0, s>>>(n, (int)k, (int)t, eps, world, world_partials, nb, norms);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int shard_phase3(cudaStream_t s, Math m, int64_t n, int64_t k, int64_t b, int64_t e, double* nb,
                 const double* coeff) {
    if (e >= k || n <= 0) return 0;
    const int64_t items = n * ((k - e + 3) / 4);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(2368, (items + 255) / 256));
    if (m == Math::exact)
        phase3_kernel<MathExact><<<grid, 256, 0, s>>>(n, (int)k, (int)b, (int)e, nb, coeff);
    else
        phase3_kernel<MathFused><<<grid, 256, 0, s>>>(n, (int)k, (int)b, (int)e, nb, coeff);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

}  // namespace kern
}  // namespace plnmf
