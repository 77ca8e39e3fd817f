// K1/K2 — CSR SpMM y := a * x on sm_100a.
//
// Replaces spmm_into (proj/src/linalg.cpp:139-154), called as A*Ht
// (proj/src/hals.cpp:41) and as A^T*W on the cached transpose (hals.cpp:26-27).
//
// One warp per sparse row.  The dense operand is row-major, so each nonzero
// gathers one contiguous K-wide factor row: lane l owns columns l, l+32, ...,
// and a gather is NC coalesced 256-byte warp loads.  The row's (col, val)
// pairs are loaded 32 at a time, coalesced, and broadcast by shuffle.  Each
// output element accumulates its terms in ascending nonzero order starting
// from 0.0 — the reference's order — so with Math::exact the result is
// bit-identical to spmm_into.  Gathers of UNROLL nonzeros are issued before
// their adds to keep NC*UNROLL independent loads in flight per lane.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

constexpr int kSpmmThreads = 256;
constexpr int kUnroll = 4;

template <int NC, class M, int UNR = kUnroll, int MINB = 1>
__global__ void __launch_bounds__(kSpmmThreads, MINB) spmm_csr_kernel(
    int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const double* __restrict__ val, const double* __restrict__ x, int64_t ldx,
    double* __restrict__ y, int64_t ldy, int col0, int ncols) {
    const int64_t row = (int64_t)blockIdx.x * (kSpmmThreads / kWarp) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = lane_id();
    const int64_t e0 = rp[row], e1 = rp[row + 1];

    double acc[NC];
    bool ok[NC];
#pragma unroll
    for (int g = 0; g < NC; ++g) {
        acc[g] = 0.0;
        ok[g] = lane + kWarp * g < ncols;
    }
    const double* xb = x + col0 + lane;

    for (int64_t base = e0; base < e1; base += kWarp) {
        const int cnt = (int)((e1 - base) < kWarp ? (e1 - base) : kWarp);
        int c = 0;
        double a = 0.0;
        if (lane < cnt) {
            c = __ldg(ci + base + lane);
            a = __ldg(val + base + lane);
        }
        int i = 0;
        for (; i + UNR <= cnt; i += UNR) {
            double xv[UNR][NC];
            double av[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int cc = __shfl_sync(0xffffffffu, c, i + u);
                av[u] = __shfl_sync(0xffffffffu, a, i + u);
                const double* xr = xb + (int64_t)cc * ldx;
#pragma unroll
                for (int g = 0; g < NC; ++g) xv[u][g] = ok[g] ? __ldg(xr + kWarp * g) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int g = 0; g < NC; ++g) acc[g] = M::madd(acc[g], av[u], xv[u][g]);
        }
        for (; i < cnt; ++i) {
            const int cc = __shfl_sync(0xffffffffu, c, i);
            const double aa = __shfl_sync(0xffffffffu, a, i);
            const double* xr = xb + (int64_t)cc * ldx;
#pragma unroll
            for (int g = 0; g < NC; ++g)
                acc[g] = M::madd(acc[g], aa, ok[g] ? __ldg(xr + kWarp * g) : 0.0);
        }
    }
    double* yr = y + row * ldy + col0 + lane;
#pragma unroll
    for (int g = 0; g < NC; ++g)
        if (ok[g]) yr[kWarp * g] = acc[g];
}

// 16-byte variant (even K, 16-byte aligned rows): lane l owns the column
// pairs 2l + 64g, so a 240-wide factor row is 4 warp loads of 512 bytes
// instead of 8 of 256 — half the load instructions and L1 requests for the
// same L2 sectors.  Same per-element order as spmm_csr_kernel.
template <int NC2, class M, int UNR = kUnroll, int MINB = 1>
__global__ void __launch_bounds__(kSpmmThreads, MINB) spmm_csr_v2_kernel(
    int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const double* __restrict__ val, const double* __restrict__ x, int64_t ldx,
    double* __restrict__ y, int64_t ldy, int col0, int ncols) {
    const int64_t row = (int64_t)blockIdx.x * (kSpmmThreads / kWarp) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = lane_id();
    const int64_t e0 = rp[row], e1 = rp[row + 1];

    double2 acc[NC2];
    bool ok[NC2];
#pragma unroll
    for (int g = 0; g < NC2; ++g) {
        acc[g] = make_double2(0.0, 0.0);
        ok[g] = 2 * (lane + kWarp * g) < ncols;  // ncols is even
    }
    const double2* xb = reinterpret_cast<const double2*>(x + col0) + lane;
    const int64_t ld2 = ldx / 2;

    for (int64_t base = e0; base < e1; base += kWarp) {
        const int cnt = (int)((e1 - base) < kWarp ? (e1 - base) : kWarp);
        int c = 0;
        double a = 0.0;
        if (lane < cnt) {
            c = __ldg(ci + base + lane);
            a = __ldg(val + base + lane);
        }
        int i = 0;
        for (; i + UNR <= cnt; i += UNR) {
            double2 xv[UNR][NC2];
            double av[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int cc = __shfl_sync(0xffffffffu, c, i + u);
                av[u] = __shfl_sync(0xffffffffu, a, i + u);
                const double2* xr = xb + (int64_t)cc * ld2;
#pragma unroll
                for (int g = 0; g < NC2; ++g) xv[u][g] = ok[g] ? __ldg(xr + kWarp * g) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int g = 0; g < NC2; ++g) {
                    acc[g].x = M::madd(acc[g].x, av[u], xv[u][g].x);
                    acc[g].y = M::madd(acc[g].y, av[u], xv[u][g].y);
                }
        }
        for (; i < cnt; ++i) {
            const int cc = __shfl_sync(0xffffffffu, c, i);
            const double aa = __shfl_sync(0xffffffffu, a, i);
            const double2* xr = xb + (int64_t)cc * ld2;
#pragma unroll
            for (int g = 0; g < NC2; ++g) {
                const double2 t = ok[g] ? __ldg(xr + kWarp * g) : make_double2(0.0, 0.0);
                acc[g].x = M::madd(acc[g].x, aa, t.x);
                acc[g].y = M::madd(acc[g].y, aa, t.y);
            }
        }
    }
    double2* yr = reinterpret_cast<double2*>(y + row * ldy + col0) + lane;
#pragma unroll
    for (int g = 0; g < NC2; ++g)
        if (ok[g]) yr[kWarp * g] = acc[g];
}

// Column-blocked pass for operands far larger than L2 (C5: Ht 2 GB, W 4 GB):
// y += the terms of every row whose column lies in [col_lo, col_hi), from the
// row's cursor on.  A row's entries are sorted by column, so the blocks of one
// row are consecutive runs of its nonzeros; carrying each (row, column)
// accumulator through y from block to block adds the terms in exactly the
// order of one unblocked pass (spmm_into's ascending nonzero order), so the
// result is bit-identical, while every block's operand rows (<= ~48 MB) stay
// resident in L2 for all the rows that gather them.  first: the accumulators
// start at 0.0 and the cursors at the row starts.
template <int NC2, class M, int UNR = kUnroll>
__global__ void __launch_bounds__(kSpmmThreads, 2) spmm_blocked_kernel(
    int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const double* __restrict__ val, const double* __restrict__ x, int64_t ldx,
    double* __restrict__ y, int64_t ldy, int ncols, int col_hi, int64_t* __restrict__ cursor, int first,
    int last) {
    const int64_t row = (int64_t)blockIdx.x * (kSpmmThreads / kWarp) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = lane_id();
    const int64_t e1 = rp[row + 1];
    int64_t e = first ? rp[row] : cursor[row];
    if (e >= e1 || __ldg(ci + e) >= col_hi) {  // nothing in this block: the accumulators stay in y
        if (first) {
            double2* yr = reinterpret_cast<double2*>(y + row * ldy) + lane;
#pragma unroll
            for (int g = 0; g < NC2; ++g)
                if (2 * (lane + kWarp * g) < ncols) yr[kWarp * g] = make_double2(0.0, 0.0);
            if (!last) cursor[row] = e;
        }
        return;
    }
    double2 acc[NC2];
    bool ok[NC2];
    double2* yr = reinterpret_cast<double2*>(y + row * ldy) + lane;
#pragma unroll
    for (int g = 0; g < NC2; ++g) {
        ok[g] = 2 * (lane + kWarp * g) < ncols;
        acc[g] = (first || !ok[g]) ? make_double2(0.0, 0.0) : __ldcs(yr + kWarp * g);
    }
    const double2* xb = reinterpret_cast<const double2*>(x) + lane;
    const int64_t ld2 = ldx / 2;
    for (;;) {
        const int avail = (int)((e1 - e) < kWarp ? (e1 - e) : kWarp);
        int c = col_hi;
        double a = 0.0;
        if (lane < avail) {
            c = __ldcs(ci + e + lane);  // streamed once per block: evict-first, the operand block keeps L2
            a = __ldcs(val + e + lane);
        }
        const int cnt = __popc(__ballot_sync(0xffffffffu, c < col_hi));  // sorted: a prefix
        int i = 0;
        for (; i + UNR <= cnt; i += UNR) {
            double2 xv[UNR][NC2];
            double av[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int cc = __shfl_sync(0xffffffffu, c, i + u);
                av[u] = __shfl_sync(0xffffffffu, a, i + u);
                const double2* xr = xb + (int64_t)cc * ld2;
#pragma unroll
                for (int g = 0; g < NC2; ++g) xv[u][g] = ok[g] ? __ldg(xr + kWarp * g) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int g = 0; g < NC2; ++g) {
                    acc[g].x = M::madd(acc[g].x, av[u], xv[u][g].x);
                    acc[g].y = M::madd(acc[g].y, av[u], xv[u][g].y);
                }
        }
        for (; i < cnt; ++i) {
            const int cc = __shfl_sync(0xffffffffu, c, i);
            const double aa = __shfl_sync(0xffffffffu, a, i);
            const double2* xr = xb + (int64_t)cc * ld2;
#pragma unroll
            for (int g = 0; g < NC2; ++g) {
                const double2 t = ok[g] ? __ldg(xr + kWarp * g) : make_double2(0.0, 0.0);
                acc[g].x = M::madd(acc[g].x, aa, t.x);
                acc[g].y = M::madd(acc[g].y, aa, t.y);
            }
        }
        e += cnt;
        if (cnt < avail || e >= e1) break;
    }
#pragma unroll
    for (int g = 0; g < NC2; ++g)
        if (ok[g]) __stcs(yr + kWarp * g, acc[g]);
    if (!last && lane == 0) cursor[row] = e;
}

template <class M>
void launch_blocked(cudaStream_t s, int nc2, int64_t rows, const int64_t* rp, const int32_t* ci, const double* val,
                    const double* x, int64_t k, double* y, int col_hi, int64_t* cursor, bool first, bool last) {
    const dim3 grid((unsigned)((rows + kSpmmThreads / kWarp - 1) / (kSpmmThreads / kWarp)));
    const int nk = (int)k, f = first ? 1 : 0, l = last ? 1 : 0;
    switch (nc2) {
        case 1: spmm_blocked_kernel<1, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, nk, col_hi, cursor, f, l); break;
        case 2: spmm_blocked_kernel<2, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, nk, col_hi, cursor, f, l); break;
        case 3: spmm_blocked_kernel<3, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, nk, col_hi, cursor, f, l); break;
        case 4: spmm_blocked_kernel<4, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, nk, col_hi, cursor, f, l); break;
        default: throw std::logic_error("spmm: bad column-pair group count");
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
}

template <class M>
void launch_pass_v2(cudaStream_t s, int nc2, int64_t rows, const int64_t* rp, const int32_t* ci,
                    const double* val, const double* x, int64_t k, double* y, int col0, int ncols, bool short_rows,
                    bool lean) {
    const dim3 grid((unsigned)((rows + kSpmmThreads / kWarp - 1) / (kSpmmThreads / kWarp)));
    // 64 registers (4 CTAs, 32 warps per SM): beside a running Gram (lean), and
    // for short rows on its own (A*Ht at C2: 115 vs 125 us for the 80-register
    // 3-CTA variant; A^T*W's longer rows run the same on the 4-deep unroll)
    if (nc2 == 4 && (lean || short_rows)) {
        spmm_csr_v2_kernel<4, M, 2, 4><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, col0, ncols);
    } else {
        switch (nc2) {
            case 1: spmm_csr_v2_kernel<1, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, col0, ncols); break;
            case 2: spmm_csr_v2_kernel<2, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, col0, ncols); break;
            case 3: spmm_csr_v2_kernel<3, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, col0, ncols); break;
            case 4: spmm_csr_v2_kernel<4, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, col0, ncols); break;
            default: throw std::logic_error("spmm: bad column-pair group count");
        }
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
}

template <class M>
void launch_pass(cudaStream_t s, int nc, int64_t rows, const int64_t* rp, const int32_t* ci,
                 const double* val, const double* x, int64_t k, double* y, int col0, int ncols, bool short_rows) {
    const dim3 grid((unsigned)((rows + kSpmmThreads / kWarp - 1) / (kSpmmThreads / kWarp)));
#define PLNMF_SPMM_CASE(N)                                                                   \
    case N:                                                                                  \
        spmm_csr_kernel<N, M><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k,   \
                                                            col0, ncols);                    \
        break;
    // short rows (few nonzeros to unroll over): a 2-deep unroll at 80 registers
    // runs 3 CTAs per SM (24 warps) and keeps more gathers in flight than 2 CTAs
    // of a 4-deep unroll (A*Ht at C2: 126 vs 134 us; A^T*W's longer rows prefer 4)
    if (nc == 8 && short_rows) {
        spmm_csr_kernel<8, M, 2, 3><<<grid, kSpmmThreads, 0, s>>>(rows, rp, ci, val, x, k, y, k, col0, ncols);
        PLNMF_CUDA_CHECK(cudaGetLastError());
        return;
    }
    switch (nc) {
        PLNMF_SPMM_CASE(1)
        PLNMF_SPMM_CASE(2)
        PLNMF_SPMM_CASE(3)
        PLNMF_SPMM_CASE(4)
        PLNMF_SPMM_CASE(5)
        PLNMF_SPMM_CASE(6)
        PLNMF_SPMM_CASE(7)
        PLNMF_SPMM_CASE(8)
        default: throw std::logic_error("spmm: bad column-group count");
    }
#undef PLNMF_SPMM_CASE
    PLNMF_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

namespace kern {

int64_t spmm_block_rows(int64_t k) {
    const char* env = kDebugKnobs ? std::getenv("PLNMF_SPMM_BLOCK_MB") : nullptr;
    const int64_t bytes = (env ? std::atoll(env) : 64) << 20;
    return std::max<int64_t>(1, bytes / (8 * k));
}

int spmm_csr(cudaStream_t s, Math m, int64_t rows, const int64_t* rp, const int32_t* ci,
             const double* val, const double* x, int64_t k, double* y, int64_t nnz, int64_t x_rows,
             int64_t* cursor, int64_t force_block, bool lean) {
    if (rows <= 0 || k <= 0) return 0;
    // an operand much larger than L2: column-blocked passes (bit-identical, see spmm_blocked_kernel)
    const int64_t block = force_block > 0 ? force_block : spmm_block_rows(k);
    if (cursor && (x_rows > 2 * block || (force_block > 0 && x_rows > block)) && k % 2 == 0 && k <= 256 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
        reinterpret_cast<uintptr_t>(y) % 16 == 0 && x_rows <= INT32_MAX) {
        const int nc2 = (int)((k + 2 * kWarp - 1) / (2 * kWarp));
        const int64_t nb = (x_rows + block - 1) / block;
        const int64_t per = (x_rows + nb - 1) / nb;  // equal blocks
        int launches = 0;
        for (int64_t b0 = 0; b0 < x_rows; b0 += per) {
            const int hi = (int)std::min<int64_t>(x_rows, b0 + per);
            const bool first = b0 == 0, last = hi == x_rows;
            if (m == Math::exact) launch_blocked<MathExact>(s, nc2, rows, rp, ci, val, x, k, y, hi, cursor, first, last);
            else launch_blocked<MathFused>(s, nc2, rows, rp, ci, val, x, k, y, hi, cursor, first, last);
            ++launches;
        }
        return launches;
    }
    const bool short_rows = nnz >= 0 && nnz < 60 * rows;  // mean < 60 nonzeros per row
    // Columns are processed in passes of at most 256 (8 warp-wide groups);
    // passes split K evenly so no pass is nearly empty.
    const int64_t passes = (k + 255) / 256;
    const int64_t per = (k + passes - 1) / passes;
    int launches = 0;
    for (int64_t c0 = 0; c0 < k; c0 += per) {
        const int ncols = (int)((k - c0) < per ? (k - c0) : per);
        const int nc = (ncols + kWarp - 1) / kWarp;
        const bool vec = (k % 2 == 0) && (c0 % 2 == 0) && (ncols % 2 == 0) &&
                         reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0;
        if (vec) {
            const int nc2 = (ncols + 2 * kWarp - 1) / (2 * kWarp);
            if (m == Math::exact) launch_pass_v2<MathExact>(s, nc2, rows, rp, ci, val, x, k, y, (int)c0, ncols, short_rows, lean);
            else launch_pass_v2<MathFused>(s, nc2, rows, rp, ci, val, x, k, y, (int)c0, ncols, short_rows, lean);
            ++launches;
            continue;
        }
        if (m == Math::exact)
            launch_pass<MathExact>(s, nc, rows, rp, ci, val, x, k, y, (int)c0, ncols, short_rows);
        else
            launch_pass<MathFused>(s, nc, rows, rp, ci, val, x, k, y, (int)c0, ncols, short_rows);
        ++launches;
    }
    return launches;
}

}  // namespace kern
}  // namespace plnmf
