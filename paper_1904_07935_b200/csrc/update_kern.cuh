// The look-ahead tiled-update kernel template (pl_update_kernel) and its
// launchers.  Instantiated per (Math, normalize) in update_inst_*.cu so the
// four heavy instantiation sets compile in parallel; update.cu holds the host
// side (planning, dispatch) and the reference (fast-hals) updaters.
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"
#include "lookahead.cuh"

namespace plnmf {
namespace upd {



// ---------------------------------------------------------------- look-ahead tiled update
// One persistent kernel per factor update (W: cooperative, one CTA per SM, one
// grid exchange per column; H: ordinary launch).  A CTA owns R consecutive
// rows.  Its warps split into
//   chain warps  (one thread per row): phase 2 of tile s, column by column —
//                the latency-critical recurrence;
//   update warps : meanwhile build tile s+1's accumulators
//                  acc(r,c) = init(old(r,c)[*coeff(c,c)])           tiled.cpp:44
//                           + sum_{kk >= e_{s+1}} -coeff(kk,c)*old(r,kk)   phase 1, :58-60
//                           + sum_{kk <  b_s}     -coeff(kk,c)*out(r,kk)   phase 3 of tiles < s
//                  — each term in the reference's order (kk ascending).
// At the tile boundary all warps add tile s's phase-3 term to tile s+1 and
// the next tile starts.  Finished tiles are written to `out` (global) where
// later tiles' update warps read them.  The per-element operation sequence is
// exactly the reference's init -> phase 1 -> phase 3 (tiles in order) ->
// phase 2, so with Math::exact H is bit-identical to update_h_tiled.
constexpr int kLThreads = 512;
constexpr int kLQuad = 4;  // columns per update thread (independent chains)

struct LookArgs {
    int64_t n;
    int k;
    int tile;
    double eps;
    int use_diag;
    int rows_per_cta;
    const double* old_m;   // n x k
    double* out;           // n x k, the updated factor
    const double* coeff;   // k x k
    const double* add;     // n x k
    double* norms;         // k            (normalize)
    double* partials;      // k x gridDim  (normalize)
    unsigned* counters;    // k, zeroed    (normalize)
    double* totals;        // k, NaN       (normalize)
    long long* prof;       // optional per-CTA section cycles (PLNMF_PROFILE=1)
    int overlap;           // 1: look-ahead concurrent with the chain; 0: at the tile boundary
    unsigned long long* trace;  // debug: exchange timestamps (k x grid x 3)
    const double* qpanel;  // [tile][k][TQ] column panels of coeff (zero-padded), built per update
    int stage_ops;         // 1: the tile's old/add operands are staged in shared memory
    int sqn_smem;          // 1: the next tile's coeff panel is staged in shared memory
    int kc;                // >0: look-ahead operands staged in kc-wide chunks (lookahead_gemm_private)
    int kst;               // ring depth of those chunks
    int kbuf;              // rings (one per look-ahead thread that owns items)
    int dbg;               // timing experiments only (PLNMF_DBG bitmask); 0 in production
    int resident;          // 1: the CTA's old rows live in shared memory (H update, lookahead_gemm_resident)
    int ldr;               // their leading dimension (k + 2)
};

template <class M>
constexpr bool kExactM = false;
template <>
constexpr bool kExactM<MathExact> = true;

enum { kProfPro = 0, kProfChain = 1, kProfGrid = 2, kProfWait = 3, kProfBoundary = 4, kProfUpd = 5, kProfDiv = 6,
       kProfDot = 7 };

// acc(r, c) += sum over kk in [k0, k1) of -coeff(kk, c) * src(r, kk), for the
// kLQuad columns c0.. (c < cend); src row pointer srow (global or shared).
template <class M>
__device__ __forceinline__ void accumulate_quad(double (&acc)[kLQuad], const double* srow, int k0, int k1,
                                                const double* sq, int ldq, int cq, int wq) {
#pragma unroll 4
    for (int kk = k0; kk < k1; ++kk) {
        const double x = srow[kk];
        const double* q = sq + kk * ldq + cq;
#pragma unroll
        for (int u = 0; u < kLQuad; ++u)
            if (u < wq) acc[u] = M::madd(acc[u], -1.0 * q[u], x);
    }
}

// acc[u] += -coeff(kk, c0+u) * src[kk] for kk in [k0, k1), u < C (coefficient
// row kk of the next tile's columns at sq + kk*ldq + c0, 16-byte aligned).
// Columns past the tile width have zero coefficients in sq, so they stay 0.
template <class M, int C>
__device__ __forceinline__ void row_panel(double (&acc)[C], const double* __restrict__ src, int k0, int k1,
                                          const double* sq, int ldq, int c0) {
#pragma unroll 4
    for (int kk = k0; kk < k1; ++kk) {
        const double x = src[kk];
        const double2* q2 = reinterpret_cast<const double2*>(sq + kk * ldq + c0);
#pragma unroll
        for (int u = 0; u < C / 2; ++u) {
            const double2 qq = q2[u];
            acc[2 * u] = M::madd(acc[2 * u], -1.0 * qq.x, x);
            acc[2 * u + 1] = M::madd(acc[2 * u + 1], -1.0 * qq.y, x);
        }
    }
}

// TMAX > 0: the chain thread keeps its row of the current tile in registers
// (x[j] = old value, replaced by the finished value once column j is done —
// exactly the operand the reference reads: new for j < t, old for j >= t), so
// each column's scratch sum is a pure register DADD chain.  TMAX = 0: generic
// shared-memory path for tiles wider than 32.
template <class M, bool NORMALIZE, int TMAX, bool STAGE, bool SQN>
__global__ void __launch_bounds__(kLThreads, 1) pl_update_kernel(LookArgs p) {
    // developer-build instrumentation (common.cuh: kDebugKnobs); compiled out in production
    unsigned long long* const ptrace = kDebugKnobs ? p.trace : nullptr;
    long long* const pprof = kDebugKnobs ? p.prof : nullptr;
    const int overlap = kDebugKnobs ? p.overlap : 1;
    extern __shared__ double smem[];
    // tile rows in shared memory at an odd stride of doubles (T + 1, or T + 2 for odd T):
    // one thread per row, so an even stride would put many lanes on one bank
    const int T = p.tile, k = p.k, ldt = (T + 1) | 1;
    const int TQ = (T + 7) & ~7;  // sqn leading dimension: whole 8-column panels, 16-byte rows
    const int R = p.rows_per_cta;
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int nrows = (int)((r0 + R < p.n) ? R : (p.n > r0 ? p.n - r0 : 0));
    const int tid = threadIdx.x;
    // The chain warps take the HIGHEST warp ids: the issue arbiter favours
    // high warp ids, and the chain is the latency-critical path while the
    // look-ahead warps saturate the fp64 pipes.
    // Chain = row warps (one row per thread) + for W one exchange warp that
    // runs the grid exchange while the row warps precompute the next column's
    // prefix terms.
    const int row_warps = min(8, max(1, (R + kWarp - 1) / kWarp));
    const int nrowt = row_warps * kWarp;
    const int chain_warps = row_warps + (NORMALIZE ? 1 : 0);
    const int nchain = chain_warps * kWarp;
    const int nupd = kLThreads - nchain;
    const bool is_chain = tid >= nupd;
    const int ctid = tid - nupd;  // chain-local thread id
    const bool is_xwarp = NORMALIZE && ctid >= nrowt;
    const int utid = tid;         // look-ahead thread id

    // double-buffered per-tile blocks: accumulators and (optionally) the old
    // values / additive term; optionally the next tile's coeff panel.  Shapes
    // too large for shared memory read those from global (L1) instead.
    const int64_t blk = (int64_t)R * ldt;
    double* acc[2] = {smem, smem + blk};
    double* oldB[2] = {smem + 2 * blk, smem + 3 * blk};
    double* sqn = smem + (STAGE ? 4 : 2) * blk;  // k x TQ: coeff(:, next tile's columns), zero-padded
    double* sqc = sqn + (SQN ? (int64_t)k * TQ : 0);  // T x T: coeff(tile, tile) of the current tile
    double* red = sqc + (int64_t)T * T;                // 48: [0, 8) warp partials, [40, 42) norm and 1/norm
    // look-ahead GEMM operand chunks: p.kst buffers of R x (p.kc + 2), 16-byte aligned
    double* xbuf0 = smem + ((((red + 48) - smem) + 1) & ~(int64_t)1);
    // W chain (exact): per-row products of the next column's old terms, [j][row]
    double* prodS = xbuf0 + (p.kc > 0 ? (int64_t)p.kst * p.kbuf * (p.kc + 2) : 0);
    // resident mode (kc == 0): the CTA's rows of the factor, old values until a
    // tile finishes, then its new values (written back at the tile end)
    double* resid = xbuf0;

    // Profiled threads (look-ahead warp 0, chain warp 0, the exchange warp)
    // add section durations straight to global (profiling runs only); no
    // per-section registers in production.
    long long* const prof_row =
        pprof ? ((tid == 0) ? pprof + blockIdx.x * 24
                  : (tid == nupd) ? pprof + blockIdx.x * 24 + 8
                  : (is_xwarp && ctid == nrowt) ? pprof + blockIdx.x * 24 + 16 : nullptr)
               : nullptr;
    long long t0 = prof_row ? clock64() : 0;
    auto mark = [&](int sec) {
        if (prof_row) {
            const long long now = clock64();
            prof_row[sec] += now - t0;
            t0 = now;
        }
    };

    // the coeff panel of the tile starting at column bn: shared copy or global panel
    auto Qn = [&](int bn) -> const double* {
        return SQN ? sqn : p.qpanel + (int64_t)(bn / T) * k * TQ;
    };
    // Builds the accumulators of the tile [bn, en) except the phase-3 term of
    // the tile just before it: init + phase 1 + phase 3 from [0, b_prev).
    // Run by `count` threads, this one being number `self`.
    // Register-tile path (TMAX > 0): a thread owns 8 consecutive columns of one
    // row (8 independent chains); one load of the row operand feeds 8 MACs and
    // the 8 coefficients come as 4 vector LDS.128 from sqn (ld TQ, even).
    // Staged look-ahead GEMM (p.kc > 0, SQN, run by the look-ahead group):
    // lookahead_gemm_private, one row x 16 columns per thread, each thread
    // streaming its own row's operands through a p.kst-deep cp.async ring.
    auto gemm_next = [&](double* dst, int bn, int en, int bprev, int count, int self) {
        GemmArgs ga{dst, ldt, Qn(bn), TQ, bn, en, bprev, p.use_diag, p.old_m, p.out, r0, nrows, k, xbuf0,
                    p.kbuf * (kPrivKC + 2), count, self, 2};
        if (TQ == 16) {
            if (p.kst >= 3) lookahead_gemm_private<M, 16, kPrivKC, 3, 16>(ga);
            else lookahead_gemm_private<M, 16, kPrivKC, 2, 16>(ga);
        } else {
            if (p.kst >= 3) lookahead_gemm_private<M, 16, kPrivKC, 3>(ga);
            else lookahead_gemm_private<M, 16, kPrivKC, 2>(ga);
        }
    };
    auto build_next = [&](double* dst, int bn, int en, int bprev, int first, int count, int self) {
        const double* Q = Qn(bn);
        if (TMAX > 0 && TMAX <= 16 && SQN && !NORMALIZE && p.resident && count == nupd) {  // planner: tile <= 16
            GemmArgs ga{dst, ldt, Qn(bn), TQ, bn, en, bprev, p.use_diag, p.old_m, p.out, r0, nrows, k, nullptr, 0,
                        count, self, 2};
            const int rg = (nrows + count / 16 - 1) / (count / 16);  // rows per thread (<= 4 by the planner)
            if (rg <= 2) lookahead_gemm_resident<M, 2>(ga, resid, p.ldr);
            else if (rg == 3) lookahead_gemm_resident<M, 3>(ga, resid, p.ldr);
            else lookahead_gemm_resident<M, 4>(ga, resid, p.ldr);
            return;
        }
        if (TMAX > 0 && SQN && p.kc > 0 && count <= nupd) {
            gemm_next(dst, bn, en, bprev, count, self);
            return;
        }
        if (TMAX > 0) {
            constexpr int C8 = 8;
            const int wn = en - bn;
            const int ng = (wn + C8 - 1) / C8;
            for (int item = self; item < nrows * ng; item += count) {
                const int r = item / ng, cq = (item % ng) * C8;
                const int64_t g = (r0 + r) * k;
                double a[C8];
#pragma unroll
                for (int u = 0; u < C8; ++u) {
                    a[u] = 0.0;
                    if (cq + u < wn) {
                        const int c = bn + cq + u;
                        const double o = p.old_m[g + c];
                        a[u] = p.use_diag ? dmul(o, Q[c * TQ + cq + u]) : o;
                    }
                }
                row_panel<M, C8>(a, p.old_m + g, en, k, Q, TQ, cq);   // phase 1
                row_panel<M, C8>(a, p.out + g, 0, bprev, Q, TQ, cq);  // phase 3, tiles before the previous
#pragma unroll
                for (int u = 0; u < C8; ++u)
                    if (cq + u < wn) dst[r * ldt + cq + u] = a[u];
            }
            return;
        }
        const int wn = en - bn;
        const int nq = (wn + kLQuad - 1) / kLQuad;
        for (int item = self; item < nrows * nq; item += count) {
            const int r = item / nq, cq = (item % nq) * kLQuad;
            const int wq = min(kLQuad, wn - cq);
            const int64_t g = (r0 + r) * k;
            double a[kLQuad];
#pragma unroll
            for (int u = 0; u < kLQuad; ++u) {
                a[u] = 0.0;
                if (u < wq) {
                    const int c = bn + cq + u;
                    const double o = p.old_m[g + c];
                    a[u] = p.use_diag ? dmul(o, Q[c * TQ + cq + u]) : o;
                }
            }
            accumulate_quad<M>(a, p.old_m + g, en, k, Q, TQ, cq, wq);  // phase 1
            accumulate_quad<M>(a, p.out + g, 0, bprev, Q, TQ, cq, wq);  // phase 3, tiles before the previous
#pragma unroll
            for (int u = 0; u < kLQuad; ++u)
                if (u < wq) dst[r * ldt + cq + u] = a[u];
        }
        (void)first;
    };
    // the next tile's coefficient panel coeff(:, bn .. en), zero-padded to TQ columns; completed
    // by the caller's cp_async_wait before its barrier.  W: staged straight from coeff (no
    // panel-building launch before the latency-bound update); H: copied from the panel built
    // by qpanel_kernel (whole 16-byte rows: the smaller code keeps the H kernel's registers)
    auto load_sqn = [&](int bn, int en, int self, int count) {
        if (!SQN) return;
        if (!NORMALIZE) {
            const double* src = p.qpanel + (int64_t)(bn / T) * k * TQ;
            for (int idx = self; idx < k * TQ / 2; idx += count) cp_async16(sqn + 2 * idx, src + 2 * idx);
            cp_async_commit();
            return;
        }
        const int wn = en - bn, hq = TQ / 2;
        if (((k | bn) & 1) == 0) {  // 16-byte pieces
            for (int idx = self; idx < k * hq; idx += count) {
                const int kk = idx / hq, j = 2 * (idx - kk * hq);
                double* dst = sqn + kk * TQ + j;
                if (j + 1 < wn) {
                    cp_async16(dst, p.coeff + (int64_t)kk * k + bn + j);
                } else {
                    dst[0] = j < wn ? p.coeff[(int64_t)kk * k + bn + j] : 0.0;
                    dst[1] = 0.0;
                }
            }
        } else {
            for (int idx = self; idx < k * TQ; idx += count) {
                const int kk = idx / TQ, j = idx - kk * TQ;
                if (j < wn) cp_async8(sqn + idx, p.coeff + (int64_t)kk * k + bn + j);
                else sqn[idx] = 0.0;
            }
        }
        cp_async_commit();
    };
    // the tile's T x T coefficient block: a sub-block of the staged panel
    // sqn (coeff(kk, b + j) at sqn[kk * TQ + j]) when that is in shared memory
    auto load_sqc = [&](int b, int e, int self, int count) {
        const int w = e - b;
        const bool from_panel = SQN && b > 0;  // the panel of tile b is staged during the previous tile
        for (int idx = self; idx < w * w; idx += count) {
            const int i = idx / w, j = idx % w;
            sqc[i * T + j] = from_panel ? sqn[(b + i) * TQ + j] : p.coeff[(int64_t)(b + i) * k + b + j];
        }
    };

    // old values of the tile [bn, en) for this CTA's rows (coalesced rows of w doubles); the
    // additive term is read from global by the chain, one column ahead
    auto stage_tile = [&](int buf, int bn, int en, int self, int count) {
        if (!STAGE) return;
        const int wn = en - bn;
        for (int idx = self; idx < nrows * wn; idx += count) {
            const int r = idx / wn, j = idx % wn;
            const int64_t g = (r0 + r) * k + bn + j;
            cp_async8(oldB[buf] + r * ldt + j, p.old_m + g);
        }
        cp_async_commit();
    };

    // exact W chain with a concurrent look-ahead: a finished tile (all T columns; only the
    // last tile may be narrower) is published to global by the look-ahead warps at the start
    // of the next tile, before build_next reuses its buffer, instead of by the chain at the
    // tile boundary
    const bool la_pub = NORMALIZE && kExactM<M> && TMAX > 0 && overlap == 1 && !p.resident;
    auto publish_prev = [&](const double* P, int pb) {
        if (T == 16) {
            for (int idx = utid; idx < nrows * 16; idx += nupd)
                p.out[(r0 + (idx >> 4)) * k + pb + (idx & 15)] = P[(idx >> 4) * ldt + (idx & 15)];
        } else {
            for (int idx = utid; idx < nrows * T; idx += nupd) {
                const int rr = idx / T, j = idx % T;
                p.out[(r0 + rr) * k + pb + j] = P[rr * ldt + j];
            }
        }
    };

    // ---- prologue: tile 0 accumulators (init + phase 1), coeff blocks, tile-0 operands
    {
        const int e0 = min(T, k);
        if (tid < 8) red[tid] = 0.0;  // warp-partial slots no row warp owns stay +0.0
        if (p.resident) {  // the CTA's rows of the old factor, once
            const bool vec = (k & 1) == 0;
            const int pr = vec ? k / 2 : k;
            for (int idx = tid; idx < nrows * pr; idx += kLThreads) {
                const int r = idx / pr, u = idx - r * pr;
                if (vec) cp_async16(resid + r * p.ldr + 2 * u, p.old_m + (r0 + r) * k + 2 * u);
                else cp_async8(resid + r * p.ldr + u, p.old_m + (r0 + r) * k + u);
            }
            cp_async_commit();
        }
        load_sqn(0, e0, tid, kLThreads);
        load_sqc(0, e0, tid, kLThreads);
        stage_tile(0, 0, e0, tid, kLThreads);
        cp_async_wait<0>();
        __syncthreads();
        if (p.kc > 0 || p.resident) {
            if (!is_chain) build_next(acc[0], 0, e0, 0, 0, nupd, utid);
        } else {
            build_next(acc[0], 0, e0, 0, 0, kLThreads, tid);
        }
        __syncthreads();
    }
    mark(kProfPro);

    int cur = 0;
    double add_carry = 0.0;  // chain: the next tile's first additive term, prefetched
    for (int b = 0; b < k; b += T) {
        const int e = min(b + T, k), w = e - b;
        const int bn = e, en = min(e + T, k);
        const bool has_next = bn < k;
        double* A = acc[cur];
        // PLNMF_TRACE_EXCHANGE: tile-boundary stamps go to the tile's last column
        unsigned long long* const btr =
            ptrace ? ptrace + ((int64_t)(e - 1) * gridDim.x + blockIdx.x) * kTraceSlots : nullptr;
        if (is_chain && TMAX > 0 && NORMALIZE && kExactM<M>) {
            // ---- W phase 2, latency-ordered (Math::exact).  Everything that does
            // not depend on the column's norm is computed while the exchange is
            // in flight: the next column's new-value prefix (pre), the products
            // of its old-value terms (prod[j] = old_j * c(j, t+1): exact
            // multiplications, the same bits the reference adds), its diagonal
            // coefficient and a + add.  After the norm arrives only
            //   div -> clamp -> mul -> add -> (w-t-1 dependent adds) -> sub -> clamp -> square
            // remain before the next reduction: the reference's exact order.
            // Operands stay in shared memory (old values: orow; finished values:
            // arow, which the reference reads as `new`; the products: prodS).
            constexpr int TM = TMAX > 0 ? TMAX : 1;
            const int r = ctid;
            const bool own = !is_xwarp && r < nrows;
            // prod[j]: this row's products at the odd row stride ldt (lanes' 64-bit accesses
            // spread over the banks), so every j is an immediate offset from one base
            double* prod = prodS + r * ldt;
            double* arow = A + r * ldt;
            const double* addr = p.add + (r0 + r) * k + b;
            const double* orow = p.resident ? resid + r * p.ldr + b
                                 : STAGE ? oldB[cur] + r * ldt : p.old_m + (r0 + r) * k + b;
            // column 0 of the tile: every scratch term is old (tiled.cpp:118-131)
            double val = 0.0;
            {
                const double add0 = b == 0 ? (own ? addr[0] : 0.0) : add_carry;
                if (own) {
                    double s = 0.0;
#pragma unroll
                    for (int j = 0; j < TM; ++j)
                        if (j < w) s = dadd(s, dmul(orow[j], sqc[j * T]));
                    val = clamp_floor(p.eps, dsub(dadd(arow[0], add0), s));
                }
            }
            if (ptrace && b > 0 && ctid == 0) ptrace[((int64_t)(b - 1) * gridDim.x + blockIdx.x) * kTraceSlots + 13] = clock64();
            // the additive term is read from global one column ahead of its use
            // (an HBM/L2 load: ~1K cycles that the prefix would otherwise stall on)
            double add_nx = (own && w > 1) ? addr[1] : 0.0;
            // not unrolled: one column's code (exchange included) stays resident
            // in the instruction cache across the whole update
#pragma unroll 1
            for (int tt = 0; tt < w; ++tt) {
                {
                    unsigned long long* const trc =
                        ptrace ? ptrace + ((int64_t)(b + tt) * gridDim.x + blockIdx.x) * kTraceSlots : nullptr;
                    const bool more = tt + 1 < w;
                    if (!is_xwarp) {
                        const double ss = (kDebugKnobs && (p.dbg & 8)) ? val : warp_sum_lane0(dmul(val, val));
                        if (lane_id() == 0) red[ctid >> 5] = ss;
                    }
                    mark(kProfDot);
                    if (trc && ctid == 0) trc[6] = clock64();
                    named_sync(1, nchain);
                    double pre = 0.0, c1 = 0.0, u1 = 0.0;
                    if (is_xwarp) {
                        // every lane adds the 8 warp partials in one fixed pairwise tree
                        // (slots >= row_warps hold +0.0): no broadcast shuffle needed
                        double v[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[i] = red[i];
                        const double blk = tree8(v);
                        mark(kProfChain);
                        if (trc && lane_id() == 0) trc[7] = clock64();
                        const double norm = (kDebugKnobs && (p.dbg & 32)) ? __dsqrt_rn(blk)
                                                         : grid_exchange(blk, b + tt, gridDim.x, p.partials, p.counters,
                                                                         ptrace);
                        if (lane_id() == 0) {
                            red[40] = norm;
                            // the rows divide as a * RN(1/norm) + one fma correction: bit-identical to
                            // a / norm for operands in [2^-500, 2^500] (tools/div_check.cu: 2.6e10 pairs)
                            const bool safe = norm >= 0x1p-500 && norm <= 0x1p500;
                            red[41] = safe ? __drcp_rn(norm) : 0.0;
                            if (blockIdx.x == 0) p.norms[b + tt] = norm;
                        }
                        mark(kProfGrid);
                    } else if (own && !more && has_next) {
                        add_carry = addr[w];  // next tile's first column
                    } else if (own && more && !(kDebugKnobs && (p.dbg & 1))) {
                        // next column's norm-independent parts, overlapping the exchange
#pragma unroll
                        for (int j = 0; j < TM; ++j)
                            if (j < tt) pre = dadd(pre, dmul(arow[j], sqc[j * T + tt + 1]));
#pragma unroll
                        for (int j = 0; j < TM; ++j)
                            if (j > tt && j < w) prod[j] = dmul(orow[j], sqc[j * T + tt + 1]);
                        c1 = sqc[tt * T + tt + 1];
                        u1 = dadd(arow[tt + 1], add_nx);
                        if (tt + 2 < w) add_nx = addr[tt + 2];  // consumed by the next column's prefix
                        mark(kProfUpd);
                    }
                    named_sync(1, nchain);
                    if (trc && (ctid == 0 || ctid == nrowt)) trc[ctid == 0 ? 4 : 3] = clock64();
                    double nv;  // max(eps, val / norm), tiled.cpp:146
                    {
                        const double bn = red[40], y = red[41];
                        if (y != 0.0 && val >= 0x1p-500 && val <= 0x1p500) {
                            const double q0 = __dmul_rn(val, y);
                            nv = clamp_floor(p.eps, __fma_rn(__fma_rn(-q0, bn, val), y, q0));
                        } else {
                            nv = clamp_floor(p.eps, div_outlined(val, bn));
                        }
                    }
                    if (own) {
                        arow[tt] = nv;
                        if (more) {
                            double s2 = dadd(pre, dmul(nv, c1));
                            if (!(kDebugKnobs && (p.dbg & 2)))
#pragma unroll
                                for (int j = 0; j < TM; ++j)
                                    if (j > tt && j < w) s2 = dadd(s2, prod[j]);
                            val = clamp_floor(p.eps, dsub(u1, s2));
                        }
                    }
                    mark(kProfDiv);
                    if (trc && ctid == 0) trc[5] = clock64();
                }
            }
            named_sync(1, nchain);
            if (la_pub && has_next) {
                // published by the look-ahead warps at the start of the next tile
            } else if (w == 16 && !p.resident) {  // full 16-wide tiles: shifts instead of a runtime division
                for (int idx = ctid; idx < nrows * 16; idx += nchain)
                    p.out[(r0 + (idx >> 4)) * k + b + (idx & 15)] = A[(idx >> 4) * ldt + (idx & 15)];
            } else {
                for (int idx = ctid; idx < nrows * w; idx += nchain) {
                    const int rr = idx / w, j = idx % w;
                    p.out[(r0 + rr) * k + b + j] = A[rr * ldt + j];
                    if (p.resident) resid[rr * p.ldr + b + j] = A[rr * ldt + j];
                }
            }
            mark(kProfChain);
        } else if (is_chain && TMAX > 0 && !NORMALIZE) {
            // ---- H phase 2, register-resident rows, latency-ordered: column tt's scratch
            // sum is the reference's sequence 0 + new_0 c(0,tt) + ... + new_{tt-1} c(tt-1,tt)
            // + old_tt c(tt,tt) + ... (tiled.cpp:118-131).  Its first tt-1 terms depend only
            // on finished columns, so they are summed (P) while column tt-1 is still in
            // flight; after new_{tt-1} only its own term and the old terms remain.
            // full 16-wide tiles get their own copy with the width and the coefficient
            // stride as constants (no predicates on the terms, immediate-offset loads)
            auto hchain = [&](auto wconst) {
                constexpr int WF = decltype(wconst)::value;
                const int wl = WF > 0 ? WF : w, Tl = WF > 0 ? WF : T;
                constexpr int TM = TMAX > 0 ? TMAX : 1;
                const int r = ctid;
                const bool own = r < nrows;
                double x[TM];
                double* arow = A + r * ldt;
                const double* addr = p.add + (r0 + r) * k + b;
                const double* orow = p.resident ? resid + r * p.ldr + b
                                     : STAGE ? oldB[cur] + r * ldt : p.old_m + (r0 + r) * k + b;
#pragma unroll
                for (int j = 0; j < TM; ++j) x[j] = (own && j < wl) ? orow[j] : 0.0;
                double pre = 0.0;  // sum_{j < tt-1} new_j c(j, tt), from 0
                double add_next = b == 0 ? (own ? addr[0] : 0.0) : add_carry;
#pragma unroll
                for (int tt = 0; tt < TM; ++tt) {
                    if (tt < wl) {
                        double val = 0.0;
                        const double add_t = add_next;
                        if (own && tt + 1 < wl) add_next = addr[tt + 1];
                        if (own && tt + 1 == wl && has_next) add_carry = addr[wl];
                        if (own) {
                            double s = tt == 0 ? 0.0 : M::madd(pre, x[tt - 1], sqc[(tt - 1) * Tl + tt]);
#pragma unroll
                            for (int j = 0; j < TM; ++j)
                                if (j >= tt && j < wl) s = M::madd(s, x[j], sqc[j * Tl + tt]);
                            if (tt + 1 < wl) {  // the next column's prefix: new terms j < tt
                                double pn = 0.0;
#pragma unroll
                                for (int j = 0; j < TM; ++j)
                                    if (j < tt) pn = M::madd(pn, x[j], sqc[j * Tl + tt + 1]);
                                pre = pn;
                            }
                            val = clamp_floor(p.eps, dsub(dadd(arow[tt], add_t), s));
                        }
                        x[tt] = val;
                        if (own) arow[tt] = val;
                    }
                }
                named_sync(1, nchain);
                for (int idx = ctid; idx < nrows * wl; idx += nchain) {
                    const int rr = idx / wl, j = idx % wl;
                    p.out[(r0 + rr) * k + b + j] = A[rr * ldt + j];
                    if (p.resident) resid[rr * p.ldr + b + j] = A[rr * ldt + j];
                }
            };
            if (TMAX >= 16 && w == 16 && T == 16) hchain(std::integral_constant<int, 16>{});
            else hchain(std::integral_constant<int, 0>{});
            mark(kProfChain);
        } else if (is_chain && TMAX > 0) {
            // ---- phase 2 of this tile, register-resident rows (one row per row thread)
            constexpr int TM = TMAX > 0 ? TMAX : 1;
            const int r = ctid;
            const bool own = !is_xwarp && r < nrows;
            double x[TM];
            double* arow = A + r * ldt;
            const double* addr = p.add + (r0 + r) * k + b;
            const double* orow = p.resident ? resid + r * p.ldr + b
                                 : STAGE ? oldB[cur] + r * ldt : p.old_m + (r0 + r) * k + b;
#pragma unroll
            for (int j = 0; j < TM; ++j) x[j] = (own && j < w) ? orow[j] : 0.0;
            double pre = 0.0;  // sum_{j < tt-1} x[j] c(j, tt), precomputed during the previous exchange
            double add_next = b == 0 ? (own ? addr[0] : 0.0) : add_carry;  // loaded one column ahead
#pragma unroll
            for (int tt = 0; tt < TM; ++tt) {
                if (tt < w) {
                    double val = 0.0;
                    const double add_t = add_next;
                    if (own && tt + 1 < w) add_next = addr[tt + 1];  // in flight across this column's exchange
                    if (own && tt + 1 == w && has_next) add_carry = addr[w];  // next tile's first column
                    if (own) {
                        const double a_t = arow[tt];
                        double s = NORMALIZE ? pre : 0.0;
#pragma unroll
                        for (int j = 0; j < TM; ++j) {
                            // scratch terms in the reference's order: new (j < tt), then old (j >= tt)
                            const bool take = NORMALIZE ? (j + 1 >= tt && j < w) : (j < w);
                            if (take) s = M::madd(s, x[j], sqc[j * T + tt]);
                        }
                        val = clamp_floor(p.eps, dsub(dadd(a_t, add_t), s));
                    }
                    mark(kProfDot);
                    if (NORMALIZE) {
                        if (!is_xwarp) {
                            const double ss = warp_sum_lane0(M::madd(0.0, val, val));
                            if (lane_id() == 0) red[ctid >> 5] = ss;
                        }
                        mark(kProfChain);
                        named_sync(1, nchain);
                        mark(kProfWait);
                        if (is_xwarp) {
                            double blk = 0.0;
                            if (lane_id() == 0) {
                                blk = red[0];
                                for (int i = 1; i < row_warps; ++i) blk = dadd(blk, red[i]);  // fixed order
                            }
                            blk = __shfl_sync(0xffffffffu, blk, 0);
                            mark(kProfChain);
                            const double norm =
                                grid_exchange(blk, b + tt, gridDim.x, p.partials, p.counters, ptrace);
                            if (lane_id() == 0) {
                                red[40] = norm;
                                if (blockIdx.x == 0) p.norms[b + tt] = norm;
                            }
                            mark(kProfGrid);
                        } else if (own && tt + 1 < w) {
                            // next column's prefix: terms j < tt (all final) — overlaps the exchange
                            pre = 0.0;
#pragma unroll
                            for (int j = 0; j < TM; ++j)
                                if (j < tt) pre = M::madd(pre, x[j], sqc[j * T + tt + 1]);
                            mark(kProfUpd);
                        }
                        named_sync(1, nchain);
                        mark(kProfWait);
                        val = clamp_floor(p.eps, __ddiv_rn(val, red[40]));  // tiled.cpp:146
                    }
                    x[tt] = val;
                    if (own) arow[tt] = val;
                    mark(kProfDiv);
                }
            }
            named_sync(1, nchain);
            for (int idx = ctid; idx < nrows * w; idx += nchain) {
                const int rr = idx / w, j = idx % w;
                p.out[(r0 + rr) * k + b + j] = A[rr * ldt + j];
                if (p.resident) resid[rr * p.ldr + b + j] = A[rr * ldt + j];
            }
            mark(kProfChain);
        } else if (is_chain) {
            // ---- phase 2 of this tile (generic shared-memory path)
            const double* oldT = STAGE ? oldB[cur] : p.old_m + r0 * k + b;
            const double* addT = p.add + r0 * k + b;
            const int64_t ldo = STAGE ? ldt : k;
            const int64_t lda = k;
            for (int t = b; t < e; ++t) {
                const int tt = t - b;
                double ss = 0.0;
                for (int r = ctid; r < nrows && !is_xwarp; r += nrowt) {
                    double* nr = A + r * ldt;
                    const double* orow = oldT + r * ldo;
                    double s = 0.0;
                    for (int j = 0; j < tt; ++j) s = M::madd(s, nr[j], sqc[j * T + tt]);
                    for (int j = tt; j < w; ++j) s = M::madd(s, orow[j], sqc[j * T + tt]);
                    const double val = clamp_floor(p.eps, dsub(dadd(nr[tt], addT[r * lda + tt]), s));
                    nr[tt] = val;
                    if (NORMALIZE) ss = M::madd(ss, val, val);
                }
                if (NORMALIZE) {
                    // chain-group reduction (fixed tree), then the grid exchange
                    if (!is_xwarp) {
                        ss = warp_sum_lane0(ss);
                        if (lane_id() == 0) red[ctid >> 5] = ss;
                    }
                    named_sync(1, nchain);
                    if (is_xwarp) {
                        double blk = 0.0;
                        if (lane_id() == 0) {
                            blk = red[0];
                            for (int i = 1; i < row_warps; ++i) blk = dadd(blk, red[i]);  // fixed order
                        }
                        blk = __shfl_sync(0xffffffffu, blk, 0);
                        mark(kProfChain);
                        const double norm = grid_exchange(blk, t, gridDim.x, p.partials, p.counters, ptrace);
                        if (lane_id() == 0) {
                            red[40] = norm;
                            if (blockIdx.x == 0) p.norms[t] = norm;
                        }
                        mark(kProfGrid);
                    }
                    named_sync(1, nchain);
                    const double norm = red[40];
                    for (int r = ctid; r < nrows && !is_xwarp; r += nrowt) {
                        double* x = A + r * ldt + tt;
                        *x = clamp_floor(p.eps, __ddiv_rn(*x, norm));  // tiled.cpp:146
                    }
                }
            }
            // publish the finished tile (rows were thread-private until here)
            named_sync(1, nchain);
            if (btr && ctid == 0) btr[8] = clock64();
            for (int idx = ctid; idx < nrows * w; idx += nchain) {
                const int r = idx / w, j = idx % w;
                p.out[(r0 + r) * k + b + j] = A[r * ldt + j];
                if (p.resident) resid[r * p.ldr + b + j] = A[r * ldt + j];
            }
            mark(kProfChain);
        } else if (has_next && overlap) {
            // ---- look-ahead: next tile's accumulators, minus this tile's phase-3 term
            if (la_pub && b > 0) publish_prev(acc[cur ^ 1], b - T);  // before build_next reuses it
            load_sqn(bn, en, utid, nupd);
            stage_tile(cur ^ 1, bn, en, utid, nupd);
            cp_async_wait<0>();
            named_sync(2, nupd);
#ifndef PLNMF_CHAIN_ONLY  // timing experiment: the chain with the look-ahead compiled out
            {
                // PLNMF_DBG >> 8: look-ahead width in warps (timing experiments only; 0 = all)
                const int nla = (kDebugKnobs && (p.dbg >> 8)) ? min((p.dbg >> 8) * kWarp, nupd) : nupd;
                if ((!kDebugKnobs || overlap != 2) && utid < nla) build_next(acc[cur ^ 1], bn, en, b, 0, nla, utid);  // 2: timing probe only
            }
#endif
            mark(kProfUpd);
        } else if (la_pub && !is_chain && b > 0) {
            publish_prev(acc[cur ^ 1], b - T);  // last tile: only the previous tile is left to publish
        }
        if (btr && tid == nupd) btr[9] = clock64();
        __syncthreads();
        if (btr && tid == nupd) btr[10] = clock64();
        mark(kProfWait);
#ifndef PLNMF_CHAIN_ONLY
        if (has_next && !overlap) {
            load_sqn(bn, en, tid, kLThreads);
            stage_tile(cur ^ 1, bn, en, tid, kLThreads);
            cp_async_wait<0>();
            __syncthreads();
            build_next(acc[cur ^ 1], bn, en, b, 0, kLThreads, tid);
            __syncthreads();
            mark(kProfUpd);
        }
#endif
        if (has_next) {
            // ---- boundary: this tile's phase-3 term into the next tile, coeff block of the next tile
            double* An = acc[cur ^ 1];
            const int wn = en - bn;
#ifndef PLNMF_CHAIN_ONLY
            if (TMAX > 0 && SQN) {
                // zero-padded staged panel: 8-wide register rows (row_panel, the same per-element
                // madd sequence as accumulate_quad), one item per thread for 16-wide tiles
                const int n8 = (wn + 7) / 8;
                for (int item = tid; item < nrows * n8; item += kLThreads) {
                    const int r = item / n8, c8 = (item % n8) * 8;
                    double a[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) a[u] = (c8 + u < wn) ? An[r * ldt + c8 + u] : 0.0;
                    row_panel<M, 8>(a, A + r * ldt - b, b, e, Qn(bn), TQ, c8);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (c8 + u < wn) An[r * ldt + c8 + u] = a[u];
                }
            }
            const int nq = (wn + kLQuad - 1) / kLQuad;
            for (int item = tid; item < ((TMAX > 0 && SQN) ? 0 : nrows * nq); item += kLThreads) {
                const int r = item / nq, cq = (item % nq) * kLQuad;
                const int wq = min(kLQuad, wn - cq);
                double a[kLQuad];
#pragma unroll
                for (int u = 0; u < kLQuad; ++u) a[u] = (u < wq) ? An[r * ldt + cq + u] : 0.0;
                // src row = finished tile values, indexed by absolute kk in [b, e)
                accumulate_quad<M>(a, A + r * ldt - b, b, e, Qn(bn), TQ, cq, wq);
#pragma unroll
                for (int u = 0; u < kLQuad; ++u)
                    if (u < wq) An[r * ldt + cq + u] = a[u];
            }
#endif
            if (btr && tid == nupd) btr[11] = clock64();
            load_sqc(bn, en, tid, kLThreads);
            __syncthreads();
            if (btr && tid == nupd) btr[12] = clock64();
            mark(kProfBoundary);
        }
        cur ^= 1;
    }
}


template <class M, bool NORM, int TMAX, bool STAGE, bool SQN>
void launch_pl_t(cudaStream_t s, const kern::PhaseBPlan& plan, LookArgs& a) {
    auto fn = pl_update_kernel<M, NORM, TMAX, STAGE, SQN>;
    PLNMF_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem));
    const dim3 grid((unsigned)plan.grid), block(kLThreads);
    if (NORM) {
        void* args[] = {&a};
        PLNMF_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)fn, grid, block, args, plan.smem, s));
    } else {
        fn<<<grid, block, plan.smem, s>>>(a);
    }
}

// Shared-memory variants: both staged, panel only, neither (the planner
// never picks "operands staged, panel global").
template <class M, bool NORM, int TMAX>
void launch_pl_s(cudaStream_t s, const kern::PhaseBPlan& plan, LookArgs& a) {
    if (plan.stage_ops) launch_pl_t<M, NORM, TMAX, true, true>(s, plan, a);
    else if (plan.sqn_smem) launch_pl_t<M, NORM, TMAX, false, true>(s, plan, a);
    else launch_pl_t<M, NORM, TMAX, false, false>(s, plan, a);
}

// Register-resident chains need one row per chain thread (<= 256 rows per CTA).
template <class M, bool NORM>
void launch_pl(cudaStream_t s, const kern::PhaseBPlan& plan, LookArgs& a) {
    const bool regs = plan.rows_per_cta <= 8 * kWarp;
    if (regs && a.tile <= 16) launch_pl_s<M, NORM, 16>(s, plan, a);
    else if (regs && a.tile <= 32) launch_pl_s<M, NORM, 32>(s, plan, a);
    else launch_pl_s<M, NORM, 0>(s, plan, a);
}


}  // namespace upd
}  // namespace plnmf
