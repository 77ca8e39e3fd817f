// Math::tensor — fp64-accurate products on the 5th-generation tensor cores
// (SURVEY.md 8(d) "inter-tile phases 1/3 and dense C4: tensor cores"; the
// north star's tensor-core GEMM).  sm_100a has no fp64 tcgen05 kind, so the
// dense-A products P = A Ht and R = A^T W (proj/src/hals.cpp:29,43 ->
// gemm / accumulate_nn / accumulate_tn, linalg.cpp:45-79) are computed with
// the Ozaki splitting on tcgen05.mma kind::i8:
//
//   every row x of the left operand (and every column of the right one) is
//   scaled by a power of two 2^e (e = exponent of the row maximum, so x/2^e is
//   in [0, 1)) and cut into S = 6 unsigned 8-bit digits, x/2^e = sum_i d_i 2^-8i
//   + r with r < 2^-48 (exact fp64 arithmetic: multiply by 256, floor,
//   subtract).  The inputs are non-negative (A >= 0, factors >= eps), so
//   unsigned digits carry 8 bits each.  Then
//       C = sa sb sum_{L=2..S+1} 2^-8L sum_{i+j=L} A_i B_j
//   keeps the 21 digit products with i + j <= S + 1: each is an exact u8 x u8
//   tensor-core GEMM accumulated in int32 in TMEM (one accumulator per level
//   L, 6 x N columns), and the levels are combined in fp64 from the smallest.
//   The error is bounded by the operand scales, not by the entry: every
//   digit truncation leaves < 2^-48 of its row's (column's) maximum, so
//   |C - C~|(i,j) <= n 2^-46 sa(i) sb(j) for reduction length n.  For
//   well-scaled non-negative data (no cancellation) that is ~2^-46 relative
//   per entry; an operand column whose entries span many decades (the
//   collapsed columns right after iteration 1) keeps the
//   bound, not the per-entry figure.
//   The reduction dimension is split so no int32 accumulator can overflow
//   (6 products per level x 5024 x 255^2 < 2^31); the splits' fp64 partials
//   are added in split order.
//
// Kernel structure (one CTA = 128 rows x NT columns x one K split, one CTA
// per SM: the 6 accumulators take 6*NT <= 480 of the 512 TMEM columns):
//   warp 0  producer: per 32-wide k step, two bulk-async copies (TMA engine,
//           cp.async.bulk + mbarrier complete_tx) of the step's A and B digit
//           tiles, already stored in the tensor cores' canonical no-swizzle
//           K-major core-matrix order by the slicing kernel
//   warp 1  TMEM owner and MMA issuer: one elected thread issues the 21
//           tcgen05.mma per k step, tcgen05.commit frees the stage
//   warps 2-5  epilogue: tcgen05.ld of the 6 accumulators, fp64 combine, store
#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace ozk {

constexpr int kS = 6;                 // digits per value
constexpr int kLevels = kS;           // L = 2 .. S+1
constexpr int kPairs = kS * (kS + 1) / 2;
constexpr int kMT = 128;              // rows per CTA (MMA M)
constexpr int kKStep = 32;            // bytes of K per MMA (kind::i8)
constexpr int kStages = 5;
constexpr int kSplitK = 5024;         // 157 k steps: 6 * 5024 * 255^2 < 2^31
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// canonical K-major, no swizzle: core matrices of 8 rows x 16 bytes; LBO = 128 B
// (the two 16-byte K halves of a 32-byte k step), SBO = 256 B (8-row groups)
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// digits d_1..d_S of x in [0, 1): exact (x * 256 and the subtraction are exact in fp64)
__device__ __forceinline__ void digits(double x, uint8_t (&d)[kS]) {
#pragma unroll
    for (int i = 0; i < kS; ++i) {
        x = x * 256.0;
        const double f = floor(x);
        d[i] = (uint8_t)f;
        x = x - f;
    }
}

// scale[r] = 2^e with e the exponent of max_k x(r, k) (x/2^e in [0, 1)); x(r, k) at
// base[r * ld + k] (trans = 0) or base[k * ld + r] (trans = 1)
__global__ void row_scale_kernel(int64_t rows, int64_t cols, const double* __restrict__ base, int64_t ld, int trans,
                                 double* __restrict__ scale) {
    if (!trans) {  // one warp per row
        const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int lane = threadIdx.x & 31;
        if (r >= rows) return;
        double m = 0.0;
        for (int64_t k = lane; k < cols; k += 32) m = fmax(m, base[r * ld + k]);
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
            int e = 0;
            frexp(m, &e);
            scale[r] = m > 0.0 ? ldexp(1.0, e) : 1.0;
        }
    } else {  // one thread per row, coalesced across threads
        const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (r >= rows) return;
        double m = 0.0;
        for (int64_t k = 0; k < cols; ++k) m = fmax(m, base[k * ld + r]);
        int e = 0;
        frexp(m, &e);
        scale[r] = m > 0.0 ? ldexp(1.0, e) : 1.0;
    }
}

// Digits of x(r, k) / scale[r] into the tile layout the GEMM streams:
// [row tile][k step][digit][8-row group][16-byte K half][row in group][16 bytes],
// rows padded to a multiple of rt, K to a multiple of 32 (zero digits).
// One thread per (row, 16-wide K chunk).
__global__ void slice_kernel(int64_t rows, int64_t cols, int64_t rows_pad, int64_t nks, const double* __restrict__ base,
                             int64_t ld, int trans, const double* __restrict__ scale, int rt, uint8_t* __restrict__ out) {
    const int64_t nchunk = nks * 2;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows_pad * nchunk) return;
    // trans: consecutive threads take consecutive rows of one chunk (coalesced reads)
    const int64_t r = trans ? idx % rows_pad : idx / nchunk;
    const int64_t ch = trans ? idx / rows_pad : idx % nchunk;
    uint8_t dg[kS][16];
    const double inv = r < rows ? 1.0 / scale[r] : 0.0;  // a power of two: exact
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        const int64_t k = ch * 16 + c;
        double x = 0.0;
        if (r < rows && k < cols) x = (trans ? base[k * ld + r] : base[r * ld + k]) * inv;
        uint8_t d[kS];
        digits(x, d);
#pragma unroll
        for (int i = 0; i < kS; ++i) dg[i][c] = d[i];
    }
    const int64_t tile = r / rt, rr = r % rt, ks = ch >> 1, half = ch & 1;
    uint8_t* t = out + ((tile * nks + ks) * kS) * (int64_t)rt * kKStep;
    const int64_t off = (rr >> 3) * 256 + half * 128 + (rr & 7) * 16;
#pragma unroll
    for (int i = 0; i < kS; ++i) {
        uint4 v;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = (uint32_t)dg[i][4 * q] | ((uint32_t)dg[i][4 * q + 1] << 8) | ((uint32_t)dg[i][4 * q + 2] << 16) |
                   ((uint32_t)dg[i][4 * q + 3] << 24);
        v.x = w[0];
        v.y = w[1];
        v.z = w[2];
        v.w = w[3];
        *reinterpret_cast<uint4*>(t + (int64_t)i * rt * kKStep + off) = v;
    }
}

struct GemmArgs {
    const uint8_t* a;  // digit tiles of the left operand (row tile 128)
    const uint8_t* b;  // digit tiles of the right operand (row tile NT)
    const double* sa;  // power-of-two row scales
    const double* sb;
    double* part;      // [split][M][N] fp64 partial products
    int64_t m, n, nks; // rows, columns (N), k steps of 32
    int nt;            // N per CTA (multiple of 16, <= 80)
    int steps_per_split;
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) ozaki_gemm_kernel(GemmArgs g) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kABytes = kS * kMT * kKStep;  // 24 KB
    constexpr int kBBytes = kS * NT * kKStep;
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t mt = blockIdx.y, ntile = blockIdx.x, split = blockIdx.z;
    const int64_t ks0 = split * g.steps_per_split;
    const int64_t ks1 = (ks0 + g.steps_per_split < g.nks) ? ks0 + g.steps_per_split : g.nks;
    const int nsteps = (int)(ks1 - ks0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: 512 columns (the 6 level accumulators use 6 * NT)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // producer: one bulk copy per operand per k step
            const uint8_t* a0 = g.a + (mt * g.nks) * (int64_t)kABytes;
            const uint8_t* b0 = g.b + (ntile * g.nks) * (int64_t)kBBytes;
            for (int i = 0; i < nsteps; ++i) {
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(empty + s, ((i / kStages) - 1) & 1);
                mbar_expect_tx(full + s, kABytes + kBBytes);
                bulk_g2s(sA + s * kABytes, a0 + (ks0 + i) * (int64_t)kABytes, kABytes, full + s);
                bulk_g2s(sB + s * kBBytes, b0 + (ks0 + i) * (int64_t)kBBytes, kBBytes, full + s);
            }
        }
    } else if (warp == 1) {
        // For one A digit da, the B digits db = 1 .. S+1-da feed the levels L = da+1 .. S+1, whose
        // accumulators sit side by side in TMEM ((L-2) * NT) while the B digit tiles sit side by
        // side in shared memory: one MMA with N = (#db) * NT covers them all (split at N <= 256).
        // 9 MMAs per k step instead of 21, and each A digit tile is read from shared memory once
        // per group instead of once per pair — the same exact integer sums.
        constexpr int kMaxDig = (256 / NT) < kS ? (256 / NT) : kS;  // B digit tiles per MMA
        for (int i = 0; i < nsteps; ++i) {
            const int s = i % kStages;
            mbar_wait(full + s, (i / kStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
#pragma unroll
                for (int da = 1; da <= kS; ++da) {
                    const int nb = kS + 1 - da;  // db = 1 .. nb
#pragma unroll
                    for (int d0 = 1; d0 <= nb; d0 += kMaxDig) {
                        const int cnt = (nb - d0 + 1) < kMaxDig ? (nb - d0 + 1) : kMaxDig;
                        // instruction descriptor: D s32, A/B u8 K-major, N = cnt * NT, M = 128
                        const uint32_t idesc =
                            (2u << 4) | ((uint32_t)((cnt * NT) >> 3) << 17) | ((uint32_t)(kMT >> 4) << 24);
                        const uint64_t ad = smem_desc(sA + s * kABytes + (da - 1) * kMT * kKStep);
                        const uint64_t bd = smem_desc(sB + s * kBBytes + (d0 - 1) * NT * kKStep);
                        // da = 1 is the first digit of every level: at the first k step it initialises
                        const uint32_t acc = (i > 0 || da > 1) ? 1u : 0u;
                        mma_u8(tmem + (uint32_t)((da + d0 - 2) * NT), ad, bd, idesc, acc);
                    }
                }
                mma_commit(empty + s);  // the stage's smem is free once these MMAs have read it
            }
            __syncwarp();
        }
        if (lane == 0) mma_commit(done);
        __syncwarp();
    } else {
        // epilogue: warp w reads TMEM lanes 32 * (w % 4) .. +31 = rows of the tile
        const int quarter = warp & 3;
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int64_t row = mt * kMT + quarter * 32 + lane;
        const double sa = row < g.m ? g.sa[row] : 0.0;
        double* prow = g.part + (split * g.m + row) * g.n;
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 16) {
            double v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.0;
#pragma unroll 1
            for (int L = kS + 1; L >= 2; --L) {  // smallest contributions first
                uint32_t r[16];
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)((L - 2) * NT + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const double w = ldexp(1.0, -8 * L);
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = dadd(v[j], dmul((double)(int32_t)r[j], w));
            }
            if (row < g.m) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int64_t col = ntile * NT + c0 + j;
                    if (col < g.n) prow[col] = dmul(dmul(v[j], sa), g.sb[col]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// out[m][n] = sum over splits in split order (fixed: run-to-run deterministic)
__global__ void split_sum_kernel(int64_t mn, int splits, const double* __restrict__ part, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= mn) return;
    double s = part[i];
    for (int p = 1; p < splits; ++p) s = dadd(s, part[(int64_t)p * mn + i]);
    out[i] = s;
}

// U(kk, c) = coeff(kk, c) for kk in the tiles after c's (kk >= e(c)), else 0: phase 1's
// coefficients (tiled.cpp:52-65) as one matrix
__global__ void phase1_coeff_kernel(int64_t k, int64_t tile, const double* __restrict__ coeff, double* __restrict__ u) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k * k) return;
    const int64_t kk = i / k, c = i % k;
    const int64_t e = ((c / tile) + 1) * tile;
    u[i] = kk >= e ? coeff[i] : 0.0;
}

// nb = init - nb (nb holds old * U on entry): init = old * coeff(c, c) for W (tiled.cpp:44), old for H
__global__ void phase_a_combine_kernel(int64_t n, int64_t k, int use_diag, const double* __restrict__ old_m,
                                       const double* __restrict__ coeff, double* __restrict__ nb) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    const int64_t c = i % k;
    const double init = use_diag ? __dmul_rn(old_m[i], coeff[c * k + c]) : old_m[i];
    nb[i] = __dsub_rn(init, nb[i]);
}

}  // namespace ozk

namespace kern {

int64_t tensor_phase_a_bytes(int64_t n, int64_t k) {
    const int nt = ozaki_nt(k);
    auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
    return al(sizeof(double) * k * k) + al(ozaki_digit_bytes(n, k, ozk::kMT)) + al(sizeof(double) * n) +
           al(ozaki_digit_bytes(k, k, nt)) + al(sizeof(double) * k) + al(sizeof(double) * ozaki_partial_doubles(n, k, k));
}

int tensor_phase_a(cudaStream_t s, int64_t n, int64_t k, int64_t tile, bool use_diag, const double* old_m,
                   const double* coeff, double* nb, void* ws) {
    if (n <= 0 || k <= 0) return 0;
    const int nt = ozaki_nt(k);
    auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
    char* p = static_cast<char*>(ws);
    double* u = reinterpret_cast<double*>(p);
    p += al(sizeof(double) * k * k);
    uint8_t* dl = reinterpret_cast<uint8_t*>(p);
    p += al(ozaki_digit_bytes(n, k, ozk::kMT));
    double* sl = reinterpret_cast<double*>(p);
    p += al(sizeof(double) * n);
    uint8_t* dr = reinterpret_cast<uint8_t*>(p);
    p += al(ozaki_digit_bytes(k, k, nt));
    double* sr = reinterpret_cast<double*>(p);
    p += al(sizeof(double) * k);
    double* part = reinterpret_cast<double*>(p);
    int launches = 0;
    ozk::phase1_coeff_kernel<<<(unsigned)((k * k + 255) / 256), 256, 0, s>>>(k, tile, coeff, u);
    ++launches;
    // left = old (n x k rows), right rows = the columns c of U: element (c, kk) at u[kk * k + c]
    launches += ozaki_slice(s, n, k, old_m, k, false, ozk::kMT, sl, dl);
    launches += ozaki_slice(s, k, k, u, k, true, nt, sr, dr);
    launches += ozaki_gemm(s, n, k, k, dl, sl, dr, sr, part, nb);  // nb := old * U
    ozk::phase_a_combine_kernel<<<(unsigned)((n * k + 255) / 256), 256, 0, s>>>(n, k, use_diag ? 1 : 0, old_m, coeff, nb);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return launches + 1;
}

int64_t ozaki_digit_bytes(int64_t rows, int64_t cols, int rt) {
    const int64_t rp = (rows + rt - 1) / rt * rt, nks = (cols + ozk::kKStep - 1) / ozk::kKStep;
    return rp * nks * ozk::kKStep * ozk::kS;
}

int ozaki_nt(int64_t n) { return n <= 80 ? (int)((n + 15) / 16 * 16) : 80; }

int ozaki_slice(cudaStream_t s, int64_t rows, int64_t cols, const double* base, int64_t ld, bool trans, int rt,
                double* scale, uint8_t* out) {
    if (rows <= 0) return 0;
    const int64_t rp = (rows + rt - 1) / rt * rt, nks = (cols + ozk::kKStep - 1) / ozk::kKStep;
    if (!trans)
        ozk::row_scale_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(rows, cols, base, ld, 0, scale);
    else
        ozk::row_scale_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(rows, cols, base, ld, 1, scale);
    const int64_t work = rp * nks * 2;
    ozk::slice_kernel<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(rows, cols, rp, nks, base, ld, trans ? 1 : 0,
                                                                     scale, rt, out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 2;
}

int64_t ozaki_partial_doubles(int64_t m, int64_t n, int64_t kdim) {
    const int64_t nks = (kdim + ozk::kKStep - 1) / ozk::kKStep;
    const int64_t per = ozk::kSplitK / ozk::kKStep;
    return ((nks + per - 1) / per) * m * n;
}

int ozaki_gemm(cudaStream_t s, int64_t m, int64_t n, int64_t kdim, const uint8_t* a_digits, const double* sa,
               const uint8_t* b_digits, const double* sb, double* part, double* out) {
    if (m <= 0 || n <= 0) return 0;
    const int nt = ozaki_nt(n);
    const int64_t nks = (kdim + ozk::kKStep - 1) / ozk::kKStep;
    const int per = ozk::kSplitK / ozk::kKStep;
    const int splits = (int)((nks + per - 1) / per);
    ozk::GemmArgs g{a_digits, b_digits, sa, sb, part, m, n, nks, nt, per};
    const dim3 grid((unsigned)((n + nt - 1) / nt), (unsigned)((m + ozk::kMT - 1) / ozk::kMT), (unsigned)splits);
    const size_t smem = (size_t)ozk::kStages * ozk::kS * (ozk::kMT + nt) * ozk::kKStep + 256;
    auto launch = [&](auto kern_fn) {
        PLNMF_CUDA_CHECK(cudaFuncSetAttribute(kern_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern_fn<<<grid, ozk::kThreads, smem, s>>>(g);
    };
    switch (nt) {
        case 16: launch(ozk::ozaki_gemm_kernel<16>); break;
        case 32: launch(ozk::ozaki_gemm_kernel<32>); break;
        case 48: launch(ozk::ozaki_gemm_kernel<48>); break;
        case 64: launch(ozk::ozaki_gemm_kernel<64>); break;
        case 80: launch(ozk::ozaki_gemm_kernel<80>); break;
        default: throw std::logic_error("ozaki_gemm: bad N tile");
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
    const int64_t mn = m * n;
    ozk::split_sum_kernel<<<(unsigned)((mn + 255) / 256), 256, 0, s>>>(mn, splits, part, out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 2;
}

}  // namespace kern
}  // namespace plnmf
