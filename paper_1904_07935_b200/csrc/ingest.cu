// Input construction on the device: the synthetic
// workload generator and the Matrix Market coordinate assembly.
//
// synth_csr_device: the counter-based generator of plnmf_synth_csr
//   (host.cpp) run one thread per row — count pass, CUB scan for the row
//   pointers, fill pass — so the large config (C5: 2M x 1M, ~1e9 nonzeros)
//   never exists on the host.  Same stream as the host generator: splitmix64
//   seeded by (seed, row), geometric gaps floor(log(u) / log1p(-p)) with
//   1/log1p(-p) computed on the host, values U(0.1, 2.0) rounded to fp32.
//
// coo_to_csr_device: the assembly half of read_coordinate
//   (proj/src/matrix_market.cpp:147-172) for entries parsed on the host:
//   bucket by row, order each row by column keeping file order among
//   duplicates (one stable radix sort of the key row * cols + col), then sum
//   each run of duplicates in file order (values.back() += v, :163-165).
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Walks row r's cells in ascending column order, calling f(col, value) for
// each; f returns false to stop the walk early.
template <class F>
__device__ void synth_walk(int64_t r, int64_t cols, bool dense, double inv_log_q, uint64_t seed, F&& f) {
    uint64_t s = seed ^ (0xD1B54A32D192ED03ULL * (static_cast<uint64_t>(r) + 1));
    splitmix64(s);
    int64_t c = -1;
    for (;;) {
        int64_t gap = 0;
        if (!dense) {
            const double u = (static_cast<double>(splitmix64(s) >> 11) + 1.0) * 0x1.0p-53;
            const double g = floor(dmul(log(u), inv_log_q));
            if (g >= static_cast<double>(cols)) break;
            gap = static_cast<int64_t>(g);
        }
        c += 1 + gap;
        if (c >= cols) break;
        const double u = static_cast<double>(splitmix64(s) >> 11) * 0x1.0p-53;
        const float value = static_cast<float>(dadd(0.1, dmul(1.9, u)));
        if (!f(c, value)) break;
    }
}

__global__ void synth_count_kernel(int64_t rows, int64_t row0, int64_t cols, int dense, double inv_log_q,
                                   uint64_t seed, int64_t* counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t n = 0;
    synth_walk(row0 + r, cols, dense, inv_log_q, seed, [&](int64_t, float) { ++n; return true; });
    counts[r] = n;
}

__global__ void synth_fill_kernel(int64_t rows, int64_t row0, int64_t cols, int dense, double inv_log_q,
                                  uint64_t seed, const int64_t* __restrict__ rp, int32_t* ci, double* val) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t at = rp[r];
    synth_walk(row0 + r, cols, dense, inv_log_q, seed, [&](int64_t c, float v) {
        ci[at] = static_cast<int32_t>(c);
        val[at] = static_cast<double>(v);
        ++at;
        return true;
    });
}

// the entries of every row with column in [c_lo, c_hi): count, then fill as
// (column - c_lo, source row, value) in row-major order
__global__ void synth_block_count_kernel(int64_t rows, int64_t cols, int dense, double inv_log_q, uint64_t seed,
                                         int64_t c_lo, int64_t c_hi, int64_t* counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t n = 0;
    synth_walk(r, cols, dense, inv_log_q, seed, [&](int64_t c, float) {
        if (c >= c_hi) return false;
        if (c >= c_lo) ++n;
        return true;
    });
    counts[r] = n;
}

__global__ void synth_block_fill_kernel(int64_t rows, int64_t cols, int dense, double inv_log_q, uint64_t seed,
                                        int64_t c_lo, int64_t c_hi, const int64_t* __restrict__ offs, int32_t* key,
                                        int32_t* src, double* val) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    int64_t at = offs[r];
    synth_walk(r, cols, dense, inv_log_q, seed, [&](int64_t c, float v) {
        if (c >= c_hi) return false;
        if (c >= c_lo) {
            key[at] = static_cast<int32_t>(c - c_lo);
            src[at] = static_cast<int32_t>(r);
            val[at] = static_cast<double>(v);
            ++at;
        }
        return true;
    });
}

__global__ void gather_block_kernel(int64_t m, const int32_t* __restrict__ perm, const int32_t* __restrict__ src,
                                    const double* __restrict__ v, int32_t* ci, double* val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = perm[i];
        ci[i] = src[j];
        val[i] = v[j];
    }
}

// rp[r] = first entry whose (sorted) key is >= r
__global__ void key_row_ptr_kernel(int64_t rows, int64_t m, const int32_t* __restrict__ keys, int64_t* rp) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > rows) return;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < r) lo = mid + 1; else hi = mid;
    }
    rp[r] = lo;
}

__global__ void iota_kernel(int64_t m, int32_t* x) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (int32_t)i;
}

__global__ void coo_keys_kernel(int64_t n, int64_t cols, const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                                uint64_t* keys, int64_t* idx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        keys[i] = (uint64_t)r[i] * (uint64_t)cols + (uint64_t)c[i];
        idx[i] = i;
    }
}

// head[i] = 1 when sorted entry i starts a new (row, col) run
__global__ void run_heads_kernel(int64_t n, const uint64_t* __restrict__ keys, int64_t* head) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// one thread per run head: the run's values summed left to right in file order
__global__ void run_sum_kernel(int64_t n, int64_t cols, const uint64_t* __restrict__ keys,
                               const int64_t* __restrict__ perm, const int64_t* __restrict__ pos,
                               const double* __restrict__ v, int32_t* ci, double* val, int64_t* row_of) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (i > 0 && keys[i] == keys[i - 1])) return;
    double acc = v[perm[i]];
    for (int64_t j = i + 1; j < n && keys[j] == keys[i]; ++j) acc = dadd(acc, v[perm[j]]);
    const int64_t o = pos[i] - 1;  // inclusive scan of the heads
    ci[o] = (int32_t)(keys[i] % (uint64_t)cols);
    val[o] = acc;
    row_of[o] = (int64_t)(keys[i] / (uint64_t)cols);
}

// rp[r] = first output entry of row >= r (rows ascending in the sorted output)
__global__ void row_ptr_kernel(int64_t rows, int64_t nnz, const int64_t* __restrict__ row_of, int64_t* rp) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > rows) return;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (row_of[mid] < r) lo = mid + 1; else hi = mid;
    }
    rp[r] = lo;
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace

namespace kern {

int64_t synth_csr_device(cudaStream_t s, int64_t rows, int64_t cols, double density, uint64_t seed,
                         int64_t** rp_out, int32_t** ci_out, double** val_out, int64_t row0) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("synth_csr: negative dimension");
    if (!(density >= 0.0) || density > 1.0) throw std::invalid_argument("synth_csr: density must be in [0, 1]");
    if (cols > INT32_MAX) throw std::invalid_argument("synth_csr: columns exceed int32 indexing");
    const bool dense = density >= 1.0;
    const double inv_log_q = (dense || density <= 0.0) ? 0.0 : 1.0 / std::log1p(-density);  // host, as host.cpp
    int64_t* rp = nullptr;
    PLNMF_CUDA_CHECK(cudaMalloc(&rp, sizeof(int64_t) * (rows + 1)));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(rp, 0, sizeof(int64_t) * (rows + 1), s));
    if (density > 0.0 && rows > 0) {
        synth_count_kernel<<<blocks(rows, 128), 128, 0, s>>>(rows, row0, cols, dense, inv_log_q, seed, rp + 1);
        PLNMF_CUDA_CHECK(cudaGetLastError());
        size_t tmp_bytes = 0;
        PLNMF_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, rp + 1, rp + 1, rows, s));
        void* tmp = nullptr;
        PLNMF_CUDA_CHECK(cudaMallocAsync(&tmp, tmp_bytes, s));
        PLNMF_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, rp + 1, rp + 1, rows, s));
        PLNMF_CUDA_CHECK(cudaFreeAsync(tmp, s));
    }
    int64_t nnz = 0;
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(&nnz, rp + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
    int32_t* ci = nullptr;
    double* val = nullptr;
    PLNMF_CUDA_CHECK(cudaMalloc(&ci, sizeof(int32_t) * std::max<int64_t>(1, nnz)));
    PLNMF_CUDA_CHECK(cudaMalloc(&val, sizeof(double) * std::max<int64_t>(1, nnz)));
    if (nnz > 0) {
        synth_fill_kernel<<<blocks(rows, 128), 128, 0, s>>>(rows, row0, cols, dense, inv_log_q, seed, rp, ci, val);
        PLNMF_CUDA_CHECK(cudaGetLastError());
    }
    *rp_out = rp;
    *ci_out = ci;
    *val_out = val;
    return nnz;
}

int64_t synth_transpose_block_device(cudaStream_t s, int64_t rows, int64_t cols, double density, uint64_t seed,
                                     int64_t c_lo, int64_t c_hi, int64_t** rp_out, int32_t** ci_out,
                                     double** val_out) {
    if (rows < 0 || cols < 0 || c_lo < 0 || c_hi < c_lo || c_hi > cols)
        throw std::invalid_argument("synth_csr: bad column block");
    if (!(density >= 0.0) || density > 1.0) throw std::invalid_argument("synth_csr: density must be in [0, 1]");
    if (rows > INT32_MAX || cols > INT32_MAX) throw std::invalid_argument("synth_csr: dimensions exceed int32 indexing");
    const bool dense = density >= 1.0;
    const double inv_log_q = (dense || density <= 0.0) ? 0.0 : 1.0 / std::log1p(-density);  // host, as host.cpp
    const int64_t nb = c_hi - c_lo;
    int64_t* rp = nullptr;
    PLNMF_CUDA_CHECK(cudaMalloc(&rp, sizeof(int64_t) * (nb + 1)));
    int64_t m = 0;
    int64_t* offs = nullptr;
    PLNMF_CUDA_CHECK(cudaMallocAsync(&offs, sizeof(int64_t) * (rows + 1), s));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(offs, 0, sizeof(int64_t) * (rows + 1), s));
    if (density > 0.0 && rows > 0 && nb > 0) {
        synth_block_count_kernel<<<blocks(rows, 128), 128, 0, s>>>(rows, cols, dense, inv_log_q, seed, c_lo, c_hi,
                                                                   offs + 1);
        PLNMF_CUDA_CHECK(cudaGetLastError());
        size_t tmp_bytes = 0;
        PLNMF_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, offs + 1, offs + 1, rows, s));
        void* tmp = nullptr;
        PLNMF_CUDA_CHECK(cudaMallocAsync(&tmp, tmp_bytes, s));
        PLNMF_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, offs + 1, offs + 1, rows, s));
        PLNMF_CUDA_CHECK(cudaFreeAsync(tmp, s));
        PLNMF_CUDA_CHECK(cudaMemcpyAsync(&m, offs + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    if (m > INT32_MAX) throw std::invalid_argument("synth_csr: column block exceeds int32 entries");
    int32_t* ci = nullptr;
    double* val = nullptr;
    PLNMF_CUDA_CHECK(cudaMalloc(&ci, sizeof(int32_t) * std::max<int64_t>(1, m)));
    PLNMF_CUDA_CHECK(cudaMalloc(&val, sizeof(double) * std::max<int64_t>(1, m)));
    if (m == 0) {
        PLNMF_CUDA_CHECK(cudaMemsetAsync(rp, 0, sizeof(int64_t) * (nb + 1), s));
    } else {
        int32_t *key, *key_sorted, *src, *idx, *perm;
        double* v;
        PLNMF_CUDA_CHECK(cudaMallocAsync(&key, sizeof(int32_t) * m, s));
        PLNMF_CUDA_CHECK(cudaMallocAsync(&key_sorted, sizeof(int32_t) * m, s));
        PLNMF_CUDA_CHECK(cudaMallocAsync(&src, sizeof(int32_t) * m, s));
        PLNMF_CUDA_CHECK(cudaMallocAsync(&idx, sizeof(int32_t) * m, s));
        PLNMF_CUDA_CHECK(cudaMallocAsync(&perm, sizeof(int32_t) * m, s));
        PLNMF_CUDA_CHECK(cudaMallocAsync(&v, sizeof(double) * m, s));
        synth_block_fill_kernel<<<blocks(rows, 128), 128, 0, s>>>(rows, cols, dense, inv_log_q, seed, c_lo, c_hi, offs,
                                                                  key, src, v);
        iota_kernel<<<blocks(m, 256) < 4736 ? blocks(m, 256) : 4736, 256, 0, s>>>(m, idx);
        int bits = 1;
        while (bits < 31 && (int64_t(1) << bits) < nb) ++bits;
        size_t tmp_bytes = 0;
        const int mi = (int)m;
        // stable: equal columns keep ascending source rows (the transpose order)
        PLNMF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key_sorted, idx, perm, mi, 0, bits, s));
        void* tmp = nullptr;
        PLNMF_CUDA_CHECK(cudaMallocAsync(&tmp, tmp_bytes, s));
        PLNMF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_sorted, idx, perm, mi, 0, bits, s));
        gather_block_kernel<<<blocks(m, 256) < 4736 ? blocks(m, 256) : 4736, 256, 0, s>>>(m, perm, src, v, ci, val);
        key_row_ptr_kernel<<<blocks(nb + 1, 256), 256, 0, s>>>(nb, m, key_sorted, rp);
        PLNMF_CUDA_CHECK(cudaGetLastError());
        for (void* p : {(void*)key, (void*)key_sorted, (void*)src, (void*)idx, (void*)perm, (void*)v, tmp})
            PLNMF_CUDA_CHECK(cudaFreeAsync(p, s));
    }
    PLNMF_CUDA_CHECK(cudaFreeAsync(offs, s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
    *rp_out = rp;
    *ci_out = ci;
    *val_out = val;
    return m;
}

int64_t coo_to_csr_device(cudaStream_t s, int64_t rows, int64_t cols, int64_t n, const int64_t* r_host,
                          const int64_t* c_host, const double* v_host, int64_t** rp_out, int32_t** ci_out,
                          double** val_out) {
    if (cols > INT32_MAX) throw std::invalid_argument("read_matrix_market: columns exceed int32 indexing");
    int64_t* rp = nullptr;
    PLNMF_CUDA_CHECK(cudaMalloc(&rp, sizeof(int64_t) * (rows + 1)));
    if (n == 0) {
        PLNMF_CUDA_CHECK(cudaMemsetAsync(rp, 0, sizeof(int64_t) * (rows + 1), s));
        PLNMF_CUDA_CHECK(cudaMalloc(ci_out, sizeof(int32_t)));
        PLNMF_CUDA_CHECK(cudaMalloc(val_out, sizeof(double)));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
        *rp_out = rp;
        return 0;
    }
    int64_t *dr, *dc, *idx, *perm, *head, *row_of;
    uint64_t *keys, *keys_sorted;
    double* dv;
    PLNMF_CUDA_CHECK(cudaMallocAsync(&dr, sizeof(int64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&dc, sizeof(int64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&dv, sizeof(double) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&idx, sizeof(int64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&perm, sizeof(int64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&head, sizeof(int64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&keys, sizeof(uint64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&keys_sorted, sizeof(uint64_t) * n, s));
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(dr, r_host, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(dc, c_host, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(dv, v_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    coo_keys_kernel<<<blocks(n, 256), 256, 0, s>>>(n, cols, dr, dc, keys, idx);
    int bits = 1;
    const uint64_t maxkey = (uint64_t)std::max<int64_t>(1, rows) * (uint64_t)std::max<int64_t>(1, cols);
    while (bits < 64 && (uint64_t(1) << bits) < maxkey) ++bits;
    size_t tmp_bytes = 0;
    PLNMF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, idx, perm, n, 0, bits, s));
    void* tmp = nullptr;
    size_t scan_bytes = 0;
    PLNMF_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, head, head, n, s));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&tmp, std::max(tmp_bytes, scan_bytes), s));
    // radix sort is stable: equal (row, col) keys keep file order
    PLNMF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, idx, perm, n, 0, bits, s));
    run_heads_kernel<<<blocks(n, 256), 256, 0, s>>>(n, keys_sorted, head);
    PLNMF_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp, scan_bytes, head, head, n, s));
    int64_t nnz = 0;
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(&nnz, head + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
    int32_t* ci = nullptr;
    double* val = nullptr;
    PLNMF_CUDA_CHECK(cudaMalloc(&ci, sizeof(int32_t) * nnz));
    PLNMF_CUDA_CHECK(cudaMalloc(&val, sizeof(double) * nnz));
    PLNMF_CUDA_CHECK(cudaMallocAsync(&row_of, sizeof(int64_t) * nnz, s));
    run_sum_kernel<<<blocks(n, 256), 256, 0, s>>>(n, cols, keys_sorted, perm, head, dv, ci, val, row_of);
    row_ptr_kernel<<<blocks(rows + 1, 256), 256, 0, s>>>(rows, nnz, row_of, rp);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    for (void* p : {(void*)dr, (void*)dc, (void*)dv, (void*)idx, (void*)perm, (void*)head, (void*)keys,
                    (void*)keys_sorted, tmp, (void*)row_of})
        PLNMF_CUDA_CHECK(cudaFreeAsync(p, s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
    *rp_out = rp;
    *ci_out = ci;
    *val_out = val;
    return nnz;
}

}  // namespace kern
}  // namespace plnmf
