// K7 error evaluation, layout conversion, and the device CSR transpose (K9).
//
// dot / error_finalize: the Gram-identity error of relative_error_gram
// (proj/src/metrics.cpp:94-127): <P,W> and <S,Q> as fixed-order two-pass
// reductions (the reference sums them serially; ours is a fixed tree, so
// run-to-run deterministic), then frob = a2 - 2*pw + sq in the reference's
// operation order, clamped at 0 with the cancellation flag.
//
// direct_residual: relative_error_direct (metrics.cpp:49-92) — a 64x64-tiled
// W*Ht^T product whose per-element sums run in the reference's k order, minus
// A's stored entries, squared and reduced in a fixed tree.
//
// csr_transpose: transpose() (proj/src/csr_matrix.cpp:30-50) on the device — a
// stable radix sort of the column indices (CUB) keeps each output row's
// entries in ascending source-row order, exactly the reference's order.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

template <class M>
__global__ void __launch_bounds__(256) dot_partial_kernel(int64_t n, const double* __restrict__ a,
                                                          const double* __restrict__ b,
                                                          double* __restrict__ partials) {
    __shared__ double red[40];
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        s = M::madd(s, a[i], b[i]);
    s = block_sum(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(int n, const double* __restrict__ partials, double* __restrict__ out) {
    __shared__ double red[40];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s = dadd(s, partials[i]);
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

__global__ void error_finalize_kernel(double a2, const double* __restrict__ pw,
                                      const double* __restrict__ sq, double* __restrict__ out3) {
    // metrics.cpp:120: a_norm_sq - 2.0 * pw + sq
    double frob = dadd(dsub(a2, dmul(2.0, *pw)), *sq);
    double cancel = 0.0;
    if (frob < 0.0) {
        frob = 0.0;
        cancel = 1.0;
    }
    out3[0] = frob;
    out3[1] = __dsqrt_rn(__ddiv_rn(frob, a2));
    out3[2] = cancel;
}

// ---- direct residual ------------------------------------------------------------------
constexpr int kDirTile = 64, kDirK = 16, kDirThreads = 256;

__device__ __forceinline__ double sparse_lookup(const int64_t* rp, const int32_t* ci,
                                                const double* val, int64_t row, int64_t col,
                                                bool* found) {
    int64_t lo = rp[row], hi = rp[row + 1];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int64_t c = ci[mid];
        if (c == col) {
            *found = true;
            return val[mid];
        }
        if (c < col) lo = mid + 1; else hi = mid;
    }
    *found = false;
    return 0.0;
}

template <class M>
__global__ void __launch_bounds__(kDirThreads) direct_residual_kernel(
    int64_t v, int64_t d, int k, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const double* __restrict__ val, const double* __restrict__ a_dense, const double* __restrict__ w,
    const double* __restrict__ ht, double* __restrict__ partials) {
    __shared__ double Ws[kDirK][kDirTile + 1];  // w(r0+rr, k0+kk) at [kk][rr]
    __shared__ double Hs[kDirK][kDirTile + 1];  // ht(c0+cc, k0+kk) at [kk][cc]
    __shared__ double red[40];
    const int64_t r0 = (int64_t)blockIdx.y * kDirTile, c0 = (int64_t)blockIdx.x * kDirTile;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < k; k0 += kDirK) {
        for (int idx = threadIdx.x; idx < kDirK * kDirTile; idx += kDirThreads) {
            const int rr = idx / kDirK, kk = idx % kDirK;
            Ws[kk][rr] = (r0 + rr < v && k0 + kk < k) ? w[(r0 + rr) * k + k0 + kk] : 0.0;
            Hs[kk][rr] = (c0 + rr < d && k0 + kk < k) ? ht[(c0 + rr) * k + k0 + kk] : 0.0;
        }
        __syncthreads();
        const int kmax = (k - k0) < kDirK ? (k - k0) : kDirK;
        for (int kk = 0; kk < kmax; ++kk) {
            double wv[4], hv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) wv[i] = Ws[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) hv[j] = Hs[kk][tx + 16 * j];
            // metrics.cpp:57: wh[d] += hc[d] * f, f = w(v,k)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = M::madd(acc[i][j], hv[j], wv[i]);
        }
        __syncthreads();
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
            if (r < v && c < d) {
                double x = acc[i][j];
                if (a_dense) {
                    x = dsub(a_dense[r * d + c], x);  // metrics.cpp:32: a - wh
                } else {
                    bool found;
                    const double av = sparse_lookup(rp, ci, val, r, c, &found);
                    if (found) x = dsub(x, av);  // metrics.cpp:59: wh -= a
                }
                s = M::madd(s, x, x);
            }
        }
    s = block_sum(s, red);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
}

// ---- layout ---------------------------------------------------------------------------
constexpr int kTr = 32;

// dst(r, c) at dst[r*cols + c]  :=  src(r, c) at src[r + c*rows]
__global__ void col_to_row_kernel(int64_t rows, int64_t cols, const double* __restrict__ src,
                                  double* __restrict__ dst) {
    __shared__ double t[kTr][kTr + 1];
    const int64_t r0 = (int64_t)blockIdx.x * kTr, c0 = (int64_t)blockIdx.y * kTr;
    for (int j = threadIdx.y; j < kTr; j += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + j;
        if (r < rows && c < cols) t[j][threadIdx.x] = src[r + c * rows];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < kTr; j += blockDim.y) {
        const int64_t r = r0 + j, c = c0 + threadIdx.x;
        if (r < rows && c < cols) dst[r * cols + c] = t[threadIdx.x][j];
    }
}

__global__ void row_to_col_kernel(int64_t rows, int64_t cols, const double* __restrict__ src,
                                  double* __restrict__ dst) {
    __shared__ double t[kTr][kTr + 1];
    const int64_t r0 = (int64_t)blockIdx.x * kTr, c0 = (int64_t)blockIdx.y * kTr;
    for (int j = threadIdx.y; j < kTr; j += blockDim.y) {
        const int64_t r = r0 + j, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[j][threadIdx.x] = src[r * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < kTr; j += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + j;
        if (r < rows && c < cols) dst[r + c * rows] = t[threadIdx.x][j];
    }
}

// ---- CSR transpose -----------------------------------------------------------------------
__global__ void expand_rows_kernel(int64_t rows, const int64_t* __restrict__ rp, int32_t* __restrict__ rowid) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) rowid[e] = (int32_t)r;
}

__global__ void iota_kernel(int64_t n, int32_t* __restrict__ x) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = (int32_t)i;
}

__global__ void gather_kernel(int64_t nnz, const int32_t* __restrict__ perm, const int32_t* __restrict__ rowid,
                              const double* __restrict__ val, int32_t* __restrict__ tci, double* __restrict__ tval) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nnz) return;
    const int32_t e = perm[i];
    tci[i] = rowid[e];
    tval[i] = val[e];
}

// trp[c] = first position with key >= c (keys sorted ascending), trp[cols] = nnz
__global__ void row_ptr_from_sorted_kernel(int64_t cols, int64_t nnz, const int32_t* __restrict__ keys,
                                           int64_t* __restrict__ trp) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > cols) return;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < c) lo = mid + 1; else hi = mid;
    }
    trp[c] = lo;
}

}  // namespace

namespace kern {

int dot(cudaStream_t s, Math m, int64_t n, const double* a, const double* b, double* partials, double* out) {
    if (m == Math::exact)
        dot_partial_kernel<MathExact><<<kDotBlocks, 256, 0, s>>>(n, a, b, partials);
    else
        dot_partial_kernel<MathFused><<<kDotBlocks, 256, 0, s>>>(n, a, b, partials);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    sum_partials_kernel<<<1, 256, 0, s>>>(kDotBlocks, partials, out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 2;
}

int error_finalize(cudaStream_t s, double a2, const double* pw, const double* sq, double* out3) {
    error_finalize_kernel<<<1, 1, 0, s>>>(a2, pw, sq, out3);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int64_t direct_residual_partials(int64_t v, int64_t d) {
    return ((v + kDirTile - 1) / kDirTile) * ((d + kDirTile - 1) / kDirTile);
}

int direct_residual(cudaStream_t s, Math m, int64_t v, int64_t d, int64_t k, const int64_t* rp,
                    const int32_t* ci, const double* val, const double* a_dense, const double* w,
                    const double* ht, double* partials, int64_t n_partials, double* out) {
    const dim3 grid((unsigned)((d + kDirTile - 1) / kDirTile), (unsigned)((v + kDirTile - 1) / kDirTile));
    if (m == Math::exact)
        direct_residual_kernel<MathExact><<<grid, kDirThreads, 0, s>>>(v, d, (int)k, rp, ci, val, a_dense, w, ht, partials);
    else
        direct_residual_kernel<MathFused><<<grid, kDirThreads, 0, s>>>(v, d, (int)k, rp, ci, val, a_dense, w, ht, partials);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    sum_partials_kernel<<<1, 1024, 0, s>>>((int)n_partials, partials, out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 2;
}

int colmajor_to_rowmajor(cudaStream_t s, int64_t rows, int64_t cols, const double* src, double* dst) {
    if (rows <= 0 || cols <= 0) return 0;
    const dim3 grid((unsigned)((rows + kTr - 1) / kTr), (unsigned)((cols + kTr - 1) / kTr)), block(kTr, 8);
    col_to_row_kernel<<<grid, block, 0, s>>>(rows, cols, src, dst);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int rowmajor_to_colmajor(cudaStream_t s, int64_t rows, int64_t cols, const double* src, double* dst) {
    if (rows <= 0 || cols <= 0) return 0;
    const dim3 grid((unsigned)((rows + kTr - 1) / kTr), (unsigned)((cols + kTr - 1) / kTr)), block(kTr, 8);
    row_to_col_kernel<<<grid, block, 0, s>>>(rows, cols, src, dst);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int csr_transpose(cudaStream_t s, int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp,
                  const int32_t* ci, const double* val, int64_t* trp, int32_t* tci, double* tval) {
    if (nnz == 0) {
        PLNMF_CUDA_CHECK(cudaMemsetAsync(trp, 0, sizeof(int64_t) * (cols + 1), s));
        return 1;
    }
    if (nnz > INT32_MAX) throw std::invalid_argument("csr_transpose: nnz exceeds int32 indexing");
    int32_t *rowid = nullptr, *idx = nullptr, *keys_out = nullptr, *perm = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    PLNMF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ci, keys_out, idx, perm,
                                                     (int)nnz, 0, 32, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&rowid, sizeof(int32_t) * nnz, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&idx, sizeof(int32_t) * nnz, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&keys_out, sizeof(int32_t) * nnz, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&perm, sizeof(int32_t) * nnz, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&tmp, tmp_bytes, s));
    expand_rows_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(rows, rp, rowid);
    iota_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(nnz, idx);
    int bits = 1;
    while ((int64_t(1) << bits) < cols && bits < 32) ++bits;
    PLNMF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ci, keys_out, idx, perm,
                                                     (int)nnz, 0, bits, s));
    gather_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(nnz, perm, rowid, val, tci, tval);
    row_ptr_from_sorted_kernel<<<(unsigned)((cols + 1 + 255) / 256), 256, 0, s>>>(cols, nnz, keys_out, trp);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    PLNMF_CUDA_CHECK(cudaFreeAsync(rowid, s));
    PLNMF_CUDA_CHECK(cudaFreeAsync(idx, s));
    PLNMF_CUDA_CHECK(cudaFreeAsync(keys_out, s));
    PLNMF_CUDA_CHECK(cudaFreeAsync(perm, s));
    PLNMF_CUDA_CHECK(cudaFreeAsync(tmp, s));
    return 6;
}

}  // namespace kern
}  // namespace plnmf
