// K3 Gram products S = W^T W, Q = Ht^T Ht, and K8 dense-A products.
//
// gram: replaces gram_into (proj/src/linalg.cpp:168-204).  The reference sums
// each upper-triangle entry over 2048-row blocks; inside a block its
// `omp simd reduction` runs as two SSE2 lanes (even / odd row offsets, an odd
// tail row into lane 0, combined as (lane0 + 0.0) + lane1 — objdump of the
// Release linalg.o), and the blocks are added to g in order.  Here one CTA
// computes a 32x32 tile of entries for one 2048-row block and one lane parity
// (even or odd rows), each thread a 4x4 register tile, rows streamed through
// shared memory in ascending order — the same per-entry operation sequence.
// A second kernel combines the lanes and adds the per-block partials in block
// order, then mirrors.
//
// dense_a_ht / dense_at_w: replace gemm(..., a.dense(), ...) at
// proj/src/hals.cpp:29,43 (accumulate_nn / accumulate_tn, linalg.cpp:45-79)
// with register-tiled SIMT GEMMs in the same per-element order
// (P: ascending inner index; R: two lanes over all V rows).
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

constexpr int kGramTile = 32;
constexpr int kGramChunk = 32;  // rows of one lane parity staged per shared-memory chunk
constexpr int kGramBlock = 2048;  // proj/src/linalg.cpp:188 kRowBlock
constexpr int kGramThreads = 64;  // 8 x 8 threads, 4 x 4 entries each

__device__ __forceinline__ void decode_upper(int p, int ntile, int& ta, int& tb) {
    ta = 0;
    int row_len = ntile;
    while (p >= row_len) {
        p -= row_len;
        ++ta;
        --row_len;
    }
    tb = ta + p;
}

// One CTA = one 32x32 tile of (a, b) entries, one 2048-row block, ONE lane
// parity: lane 0 (even row offsets) and lane 1 (odd) are independent
// sequential sums in the reference, so they run in separate CTAs (twice the
// parallelism, half the registers); the combine kernel adds them as
// (lane0 + 0.0) + lane1 exactly like the compiled reduction.
// TJ: entries per thread along b (4: 64 threads per CTA; 2: 128 threads, for short
// matrices whose (tile, block, lane) count leaves SMs under-occupied)
// DIAG (a diagonal tile, ta == tb): register entries (i, j) that lie below the
// diagonal for every thread of the CTA are not computed (the combine kernel
// reads only a <= b) — a quarter to three eighths of a diagonal tile's work.
template <int TJ, int TI>
__host__ __device__ constexpr bool below_diag(int i, int j) {
    return (32 / TI) * i > (32 / TJ - 1) + (32 / TJ) * j;
}

// JN (<= TJ): entries along b actually computed — TJ / 2 for a ragged last tile whose
// valid columns (k - b0 <= 16) all lie in the first half (K = 240: tile 7 holds 16)
template <class M, int TJ, int TI, bool DIAG, int JN = TJ>
__device__ __forceinline__ void gram_tile(int64_t n, int k, const double* __restrict__ m, double* __restrict__ part,
                                          int ta, int tb, double (&As)[2][32][32], double (&Bs)[2][32][32]);

template <class M, int TJ = 4, int TI = 4>
__global__ void __launch_bounds__((32 / TI) * (32 / TJ), 8) gram_block_kernel(int64_t n, int k,
                                                                  const double* __restrict__ m,
                                                                  double* __restrict__ part,
                                                                  int ntile) {
    // double-buffered chunks of kGramChunk rows of this lane's parity; cp.async
    // (16-byte pieces) when k is even, so the next chunk's loads overlap this
    // chunk's products instead of stalling on the staging loads
    __shared__ __align__(16) double As[2][kGramChunk][kGramTile];
    __shared__ __align__(16) double Bs[2][kGramChunk][kGramTile];
    int ta, tb;
    decode_upper(blockIdx.x, ntile, ta, tb);
    const bool half_b = tb * kGramTile + 16 >= k;  // columns b0 + 16 .. b0 + 31 are all >= k
    if (ta == tb) {
        if (half_b) gram_tile<M, TJ, TI, true, TJ / 2>(n, k, m, part, ta, tb, As, Bs);
        else gram_tile<M, TJ, TI, true>(n, k, m, part, ta, tb, As, Bs);
    } else {
        if (half_b) gram_tile<M, TJ, TI, false, TJ / 2>(n, k, m, part, ta, tb, As, Bs);
        else gram_tile<M, TJ, TI, false>(n, k, m, part, ta, tb, As, Bs);
    }
}

template <class M, int TJ, int TI, bool DIAG, int JN>
__device__ __forceinline__ void gram_tile(int64_t n, int k, const double* __restrict__ m, double* __restrict__ part,
                                          int ta, int tb, double (&As)[2][32][32], double (&Bs)[2][32][32]) {
    const int64_t blk = blockIdx.y >> 1;
    const int parity = blockIdx.y & 1;
    const int64_t v0 = blk * kGramBlock;
    const int64_t v1 = (v0 + kGramBlock < n) ? v0 + kGramBlock : n;
    // rows of this parity in [v0, v1): v0 + parity + 2i, i < cnt
    const int64_t cnt = (v1 - v0 - parity + 1) / 2;
    constexpr int NX = 32 / TJ, NY = 32 / TI, NT = NY * NX;  // threads along b / a, per CTA
    const int tx = threadIdx.x % NX, ty = threadIdx.x / NX;
    const int a0 = ta * kGramTile, b0 = tb * kGramTile;

    double acc[TI][TJ];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) acc[i][j] = 0.0;

    const bool vec = (k & 1) == 0;
    auto stage = [&](int64_t i0, int buf) {
        const int nr = (int)((cnt - i0) < kGramChunk ? (cnt - i0) : kGramChunk);
        if (vec) {
            // 16 pieces of 16 B per row and slice; columns >= k are never read back
            for (int idx = threadIdx.x; idx < kGramChunk * 32; idx += NT) {
                const int sl = idx >> 4 & 1, rr = idx >> 5, u = idx & 15;
                const int col = (sl ? b0 : a0) + 2 * u;
                if (rr < nr && col < k) {
                    const int64_t row = v0 + parity + 2 * (i0 + rr);
                    double* dst = sl ? &Bs[buf][rr][2 * u] : &As[buf][rr][2 * u];
                    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(m + row * k + col)
                                 : "memory");
                }
            }
        } else {
            for (int idx = threadIdx.x; idx < kGramChunk * kGramTile; idx += NT) {
                const int rr = idx / kGramTile, cc = idx % kGramTile;
                const bool rok = rr < nr;
                const int64_t row = v0 + parity + 2 * (i0 + rr);
                As[buf][rr][cc] = (rok && a0 + cc < k) ? m[row * k + a0 + cc] : 0.0;
                Bs[buf][rr][cc] = (rok && b0 + cc < k) ? m[row * k + b0 + cc] : 0.0;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (cnt > 0) stage(0, 0);
    int cur = 0;
    for (int64_t i0 = 0; i0 < cnt; i0 += kGramChunk, cur ^= 1) {
        const int nr = (int)((cnt - i0) < kGramChunk ? (cnt - i0) : kGramChunk);
        if (i0 + kGramChunk < cnt) {
            stage(i0 + kGramChunk, cur ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double(*Ac)[kGramTile] = As[cur];
        const double(*Bc)[kGramTile] = Bs[cur];
        int rr = 0;
        // one row per step: the 64-register variant keeps every address in registers (the
        // earlier two-rows-with-all-products-first step needed 72 registers of doubles, and
        // the compiler re-derived threadIdx inside the loop: Gram W 183 -> 176 us)
        for (; rr < nr; ++rr) {
            double av[TI], bv[TJ];
#pragma unroll
            for (int i = 0; i < TI; ++i) av[i] = Ac[rr][ty + NY * i];
#pragma unroll
            for (int j = 0; j < JN; ++j) bv[j] = Bc[rr][tx + NX * j];
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < JN; ++j)
                    if (!(DIAG && below_diag<TJ, TI>(i, j))) acc[i][j] = M::madd(acc[i][j], av[i], bv[j]);
        }
        __syncthreads();
    }
    double* pb = part + (int64_t)blockIdx.y * k * k;
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < JN; ++j) {
            const int a = a0 + ty + NY * i, b = b0 + tx + NX * j;
            if (a < k && b < k) pb[(int64_t)a * k + b] = acc[i][j];
        }
}

// g(a,b) = g(b,a) = sum over blocks in order (g starts at 0, g += acc).
__global__ void gram_combine_kernel(int k, int64_t nblk, const double* __restrict__ part,
                                    double* __restrict__ g) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)k * k) return;
    const int a = (int)(idx / k), b = (int)(idx % k);
    if (a > b) return;
    const int64_t kk = (int64_t)k * k;
    double s = 0.0;
#pragma unroll 4  // the loads of 4 blocks in flight at once (the adds stay in block order)
    for (int64_t blk = 0; blk < nblk; ++blk) {
        const double lane0 = part[(2 * blk) * kk + (int64_t)a * k + b];
        const double lane1 = part[(2 * blk + 1) * kk + (int64_t)a * k + b];
        s = dadd(s, dadd(dadd(lane0, 0.0), lane1));  // g += (lane0 + 0.0) + lane1
    }
    g[(int64_t)a * k + b] = s;
    g[(int64_t)b * k + a] = s;
}

// ---- dense-A products --------------------------------------------------------------
constexpr int kGemmTile = 64;
constexpr int kGemmK = 16;
constexpr int kGemmThreads = 256;  // 16 x 16, 4 x 4 outputs each

// p(v, j) = sum_{kk ascending} ht(kk, j) * a(v, kk), from 0 (accumulate_nn with
// alpha = 1: f = alpha*b(kk,j), c += f * a(i,kk)).
template <class M>
__global__ void __launch_bounds__(kGemmThreads) dense_a_ht_kernel(int64_t v, int64_t d, int k,
                                                                  const double* __restrict__ a,
                                                                  const double* __restrict__ ht,
                                                                  double* __restrict__ p) {
    __shared__ double As[kGemmK][kGemmTile + 1];
    __shared__ double Bs[kGemmK][kGemmTile];
    const int64_t r0 = (int64_t)blockIdx.y * kGemmTile;
    const int c0 = blockIdx.x * kGemmTile;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t k0 = 0; k0 < d; k0 += kGemmK) {
        for (int idx = threadIdx.x; idx < kGemmK * kGemmTile; idx += kGemmThreads) {
            const int rr = idx / kGemmK, kk = idx % kGemmK;
            As[kk][rr] = (r0 + rr < v && k0 + kk < d) ? a[(r0 + rr) * d + k0 + kk] : 0.0;
            const int kb = idx / kGemmTile, cc = idx % kGemmTile;
            Bs[kb][cc] = (k0 + kb < d && c0 + cc < k) ? 1.0 * ht[(k0 + kb) * k + c0 + cc] : 0.0;
        }
        __syncthreads();
        const int kmax = (int)((d - k0) < kGemmK ? (d - k0) : kGemmK);
        for (int kk = 0; kk < kmax; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = M::madd(acc[i][j], bv[j], av[i]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t r = r0 + ty + 16 * i;
            const int c = c0 + tx + 16 * j;
            if (r < v && c < k) p[r * k + c] = acc[i][j];
        }
}

// r(dd, j) = 0 + 1.0 * ((lane0 + 0.0) + lane1), lanes = even / odd v over all
// V rows (accumulate_tn's simd reduction, linalg.cpp:71-75, after the beta=0
// zero fill at :31-42).
template <class M>
__global__ void __launch_bounds__(kGemmThreads) dense_at_w_kernel(int64_t v, int64_t d, int k,
                                                                  const double* __restrict__ a,
                                                                  const double* __restrict__ w,
                                                                  double* __restrict__ r) {
    __shared__ double As[kGemmK][kGemmTile];
    __shared__ double Bs[kGemmK][kGemmTile];
    const int64_t r0 = (int64_t)blockIdx.y * kGemmTile;  // output rows = columns of A
    const int c0 = blockIdx.x * kGemmTile;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double e[4][4], o[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) e[i][j] = o[i][j] = 0.0;
    for (int64_t v0 = 0; v0 < v; v0 += kGemmK) {  // kGemmK even: parity of kk == parity of row
        for (int idx = threadIdx.x; idx < kGemmK * kGemmTile; idx += kGemmThreads) {
            const int kk = idx / kGemmTile, cc = idx % kGemmTile;
            As[kk][cc] = (v0 + kk < v && r0 + cc < d) ? a[(v0 + kk) * d + r0 + cc] : 0.0;
            Bs[kk][cc] = (v0 + kk < v && c0 + cc < k) ? w[(v0 + kk) * k + c0 + cc] : 0.0;
        }
        __syncthreads();
        const int kmax = (int)((v - v0) < kGemmK ? (v - v0) : kGemmK);
        for (int kk = 0; kk < kmax; kk += 2) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) e[i][j] = M::madd(e[i][j], av[i], bv[j]);
            if (kk + 1 < kmax) {
#pragma unroll
                for (int i = 0; i < 4; ++i) av[i] = As[kk + 1][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[j] = Bs[kk + 1][tx + 16 * j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) o[i][j] = M::madd(o[i][j], av[i], bv[j]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t rr = r0 + ty + 16 * i;
            const int c = c0 + tx + 16 * j;
            if (rr < d && c < k) r[rr * k + c] = dadd(0.0, dmul(1.0, dadd(dadd(e[i][j], 0.0), o[i][j])));
        }
}

}  // namespace

namespace kern {

int64_t gram_scratch_doubles(int64_t n, int64_t k) {
    const int64_t nblk = (n + kGramBlock - 1) / kGramBlock;
    return 2 * (nblk > 0 ? nblk : 1) * k * k;  // one K x K partial per block and lane
}

int gram(cudaStream_t s, Math m, int64_t n, int64_t k, const double* mat, double* g,
         double* scratch, int sms) {
    if (k <= 0) return 0;
    const int64_t nblk = (n + kGramBlock - 1) / kGramBlock;
    if (nblk == 0) {
        PLNMF_CUDA_CHECK(cudaMemsetAsync(g, 0, sizeof(double) * k * k, s));
        return 0;
    }
    const int ntile = (int)((k + kGramTile - 1) / kGramTile);
    const dim3 grid((unsigned)(ntile * (ntile + 1) / 2), (unsigned)(2 * nblk));
    // fewer than ~4 CTAs per SM of 4x4 threads: use 4x2 threads (twice the warps)
    const bool narrow = (int64_t)grid.x * grid.y < 8LL * sms;  // sms: the engine's device (cached by the caller)
    const int variant = narrow ? 42 : 44;
    if (m == Math::exact) {
        if (variant == 22) gram_block_kernel<MathExact, 2, 2><<<grid, 256, 0, s>>>(n, (int)k, mat, scratch, ntile);
        else if (variant == 42) gram_block_kernel<MathExact, 2, 4><<<grid, 128, 0, s>>>(n, (int)k, mat, scratch, ntile);
        else gram_block_kernel<MathExact, 4, 4><<<grid, 64, 0, s>>>(n, (int)k, mat, scratch, ntile);
    } else {
        if (variant == 22) gram_block_kernel<MathFused, 2, 2><<<grid, 256, 0, s>>>(n, (int)k, mat, scratch, ntile);
        else if (variant == 42) gram_block_kernel<MathFused, 2, 4><<<grid, 128, 0, s>>>(n, (int)k, mat, scratch, ntile);
        else gram_block_kernel<MathFused, 4, 4><<<grid, 64, 0, s>>>(n, (int)k, mat, scratch, ntile);
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
    const int64_t tot = k * k;
    gram_combine_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((int)k, nblk, scratch, g);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 2;
}

int dense_a_ht(cudaStream_t s, Math m, int64_t v, int64_t d, int64_t k, const double* a,
               const double* ht, double* p) {
    const dim3 grid((unsigned)((k + kGemmTile - 1) / kGemmTile), (unsigned)((v + kGemmTile - 1) / kGemmTile));
    if (m == Math::exact)
        dense_a_ht_kernel<MathExact><<<grid, kGemmThreads, 0, s>>>(v, d, (int)k, a, ht, p);
    else
        dense_a_ht_kernel<MathFused><<<grid, kGemmThreads, 0, s>>>(v, d, (int)k, a, ht, p);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int dense_at_w(cudaStream_t s, Math m, int64_t v, int64_t d, int64_t k, const double* a,
               const double* w, double* r) {
    const dim3 grid((unsigned)((k + kGemmTile - 1) / kGemmTile), (unsigned)((d + kGemmTile - 1) / kGemmTile));
    if (m == Math::exact)
        dense_at_w_kernel<MathExact><<<grid, kGemmThreads, 0, s>>>(v, d, (int)k, a, w, r);
    else
        dense_at_w_kernel<MathFused><<<grid, kGemmThreads, 0, s>>>(v, d, (int)k, a, w, r);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

}  // namespace kern
}  // namespace plnmf
