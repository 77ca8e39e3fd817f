// K4/K5/K6 — the factor updates on sm_100a.
//
// Tiled (PL-NMF) update, proj/src/tiled.cpp:176-214, in two launches:
//
//   phase A  init_new_accumulator (:28-50) + phase1_left_contributions (:52-65)
//            A register-tiled SIMT GEMM: nb(v,c) = old(v,c)[*coeff(c,c)], then
//            nb(v,c) += (-coeff(kk,c)) * old(v,kk) for every kk in the tiles
//            strictly right of c's tile, kk ascending — each thread walks its
//            4x4 outputs through kk in the reference's order.  Row-local.
//
//   phase B  for each tile: phase2_in_tile (:67-156) then
//            phase3_right_contributions (:158-174).  Each CTA owns a block of
//            rows; the tile's columns of nb/old/add for those rows are staged
//            in shared memory, the in-tile recurrence runs one thread per row
//            (its scratch sums run in the reference's k order), and the rank-T
//            phase-3 update of the columns right of the tile is done by the
//            whole CTA (4 independent columns per thread).  When the CTA's rows
//            fit in shared memory they stay resident for the whole update.  For
//            W (normalize) each column needs the global sum of squares before
//            the next column may start: the launch is cooperative and
//            persistent (one CTA per SM) and each column costs one grid-wide
//            exchange (grid_norm below: NaN-sentinel slots, no atomics, no
//            fences), after which every CTA sums the same partials in the same
//            fixed order, so the norm is bit-identical in every CTA and
//            run-to-run deterministic.  (The reference sums per-OpenMP-thread
//            partials instead; that order is thread-count dependent,
//            tiled.cpp:97-99.)  For H there is no norm: an ordinary launch.
//
// Reference (fast-hals) updaters, proj/src/hals.cpp:51-108: thread per row,
// exact per-row dot order; the W updater is persistent with one grid_norm per
// column for its serial norm (hals.cpp:97-102, here a fixed-order tree).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

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
};

enum { kProfPro = 0, kProfChain = 1, kProfGrid = 2, kProfWait = 3, kProfBoundary = 4, kProfUpd = 5 };

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
    extern __shared__ double smem[];
    const int T = p.tile, k = p.k, ldt = T + 1;
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
    double* addB[2] = {smem + 4 * blk, smem + 5 * blk};
    double* sqn = smem + (STAGE ? 6 : 2) * blk;  // k x TQ: coeff(:, next tile's columns), zero-padded
    double* sqc = sqn + (SQN ? (int64_t)k * TQ : 0);  // T x T: coeff(tile, tile) of the current tile
    double* red = sqc + (int64_t)T * T;                // 48

    // Section timers stay in registers (no memory traffic on the critical
    // path) and are written once at the end; look-ahead warp 0 records the
    // prologue / wait / look-ahead / boundary sections, chain warp 0 the chain,
    // grid-exchange and chain-side wait sections.
    long long t0 = clock64();
    long long sec_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto mark = [&](int sec) {
        if (p.prof) {
            const long long now = clock64();
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i == sec) sec_t[i] += now - t0;
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
    auto build_next = [&](double* dst, int bn, int en, int bprev, int first, int count, int self) {
        const double* Q = Qn(bn);
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
    auto load_sqn = [&](int bn, int en, int self, int count) {
        (void)en;
        if (!SQN) return;
        const double* src = p.qpanel + (int64_t)(bn / T) * k * TQ;
        for (int idx = self; idx < k * TQ; idx += count) sqn[idx] = src[idx];
    };
    auto load_sqc = [&](int b, int e, int self, int count) {
        const int w = e - b;
        for (int idx = self; idx < w * w; idx += count) {
            const int i = idx / w, j = idx % w;
            sqc[i * T + j] = p.coeff[(int64_t)(b + i) * k + b + j];
        }
    };

    // old / additive values of the tile [bn, en) for this CTA's rows (coalesced rows of w doubles)
    auto stage_tile = [&](int buf, int bn, int en, int self, int count) {
        if (!STAGE) return;
        const int wn = en - bn;
        for (int idx = self; idx < nrows * wn; idx += count) {
            const int r = idx / wn, j = idx % wn;
            const int64_t g = (r0 + r) * k + bn + j;
            oldB[buf][r * ldt + j] = p.old_m[g];
            addB[buf][r * ldt + j] = p.add[g];
        }
    };

    // ---- prologue: tile 0 accumulators (init + phase 1), coeff blocks, tile-0 operands
    {
        const int e0 = min(T, k);
        load_sqn(0, e0, tid, kLThreads);
        load_sqc(0, e0, tid, kLThreads);
        stage_tile(0, 0, e0, tid, kLThreads);
        __syncthreads();
        build_next(acc[0], 0, e0, 0, 0, kLThreads, tid);
        __syncthreads();
    }
    mark(kProfPro);

    int cur = 0;
    for (int b = 0; b < k; b += T) {
        const int e = min(b + T, k), w = e - b;
        const int bn = e, en = min(e + T, k);
        const bool has_next = bn < k;
        double* A = acc[cur];
        if (is_chain && TMAX > 0) {
            // ---- phase 2 of this tile, register-resident rows (one row per row thread)
            constexpr int TM = TMAX > 0 ? TMAX : 1;
            const int r = ctid;
            const bool own = !is_xwarp && r < nrows;
            double x[TM];
            double* arow = A + r * ldt;
            const double* addr = STAGE ? addB[cur] + r * ldt : p.add + (r0 + r) * k + b;
            const double* orow = STAGE ? oldB[cur] + r * ldt : p.old_m + (r0 + r) * k + b;
#pragma unroll
            for (int j = 0; j < TM; ++j) x[j] = (own && j < w) ? orow[j] : 0.0;
            double pre = 0.0;  // sum_{j < tt-1} x[j] c(j, tt), precomputed during the previous exchange
            double add_next = own ? addr[0] : 0.0;  // additive term, loaded one column ahead
#pragma unroll
            for (int tt = 0; tt < TM; ++tt) {
                if (tt < w) {
                    double val = 0.0;
                    const double add_t = add_next;
                    if (own && tt + 1 < w) add_next = addr[tt + 1];  // in flight across this column's exchange
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
                    if (NORMALIZE) {
                        if (!is_xwarp) {
                            const double ss = warp_sum_lane0(M::madd(0.0, val, val));
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
                            const double norm =
                                grid_exchange(blk, b + tt, gridDim.x, p.partials, p.counters, p.trace);
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
                        }
                        named_sync(1, nchain);
                        val = clamp_floor(p.eps, __ddiv_rn(val, red[40]));  // tiled.cpp:146
                    }
                    x[tt] = val;
                    if (own) arow[tt] = val;
                }
            }
            named_sync(1, nchain);
            for (int idx = ctid; idx < nrows * w; idx += nchain) {
                const int rr = idx / w, j = idx % w;
                p.out[(r0 + rr) * k + b + j] = A[rr * ldt + j];
            }
            mark(kProfChain);
        } else if (is_chain) {
            // ---- phase 2 of this tile (generic shared-memory path)
            const double* oldT = STAGE ? oldB[cur] : p.old_m + r0 * k + b;
            const double* addT = STAGE ? addB[cur] : p.add + r0 * k + b;
            const int64_t ldo = STAGE ? ldt : k;
            for (int t = b; t < e; ++t) {
                const int tt = t - b;
                double ss = 0.0;
                for (int r = ctid; r < nrows && !is_xwarp; r += nrowt) {
                    double* nr = A + r * ldt;
                    const double* orow = oldT + r * ldo;
                    double s = 0.0;
                    for (int j = 0; j < tt; ++j) s = M::madd(s, nr[j], sqc[j * T + tt]);
                    for (int j = tt; j < w; ++j) s = M::madd(s, orow[j], sqc[j * T + tt]);
                    const double val = clamp_floor(p.eps, dsub(dadd(nr[tt], addT[r * ldo + tt]), s));
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
                        const double norm = grid_exchange(blk, t, gridDim.x, p.partials, p.counters, p.trace);
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
            for (int idx = ctid; idx < nrows * w; idx += nchain) {
                const int r = idx / w, j = idx % w;
                p.out[(r0 + r) * k + b + j] = A[r * ldt + j];
            }
            mark(kProfChain);
        } else if (has_next && p.overlap) {
            // ---- look-ahead: next tile's accumulators, minus this tile's phase-3 term
            load_sqn(bn, en, utid, nupd);
            stage_tile(cur ^ 1, bn, en, utid, nupd);
            named_sync(2, nupd);
            build_next(acc[cur ^ 1], bn, en, b, 0, nupd, utid);
            mark(kProfUpd);
        }
        __syncthreads();
        mark(kProfWait);
        if (has_next && !p.overlap) {
            load_sqn(bn, en, tid, kLThreads);
            stage_tile(cur ^ 1, bn, en, tid, kLThreads);
            __syncthreads();
            build_next(acc[cur ^ 1], bn, en, b, 0, kLThreads, tid);
            __syncthreads();
            mark(kProfUpd);
        }
        if (has_next) {
            // ---- boundary: this tile's phase-3 term into the next tile, coeff block of the next tile
            double* An = acc[cur ^ 1];
            const int wn = en - bn, nq = (wn + kLQuad - 1) / kLQuad;
            for (int item = tid; item < nrows * nq; item += kLThreads) {
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
            load_sqc(bn, en, tid, kLThreads);
            __syncthreads();
            mark(kProfBoundary);
        }
        cur ^= 1;
    }
    if (p.prof && (tid == 0 || tid == nupd)) {
        const int slot = (tid == 0) ? 0 : 8;  // look-ahead view, chain view
#pragma unroll
        for (int i = 0; i < 8; ++i) p.prof[blockIdx.x * 16 + slot + i] = sec_t[i];
    }
}

int sm_count(int device) {
    int n = 0;
    PLNMF_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

size_t pl_smem(int64_t rows, int64_t k, int64_t tile, bool stage_ops, bool sqn_smem) {
    const int64_t tq = (tile + 7) & ~int64_t(7);
    return sizeof(double) * (size_t)((stage_ops ? 6 : 2) * rows * (tile + 1) + (sqn_smem ? k * tq : 0) +
                                     tile * tile + 48);
}

// qpanel[tau][kk][j] = coeff(kk, b_tau + j) for j < width(tau), 0 up to TQ.
__global__ void qpanel_kernel(int k, int tile, int tq, const double* __restrict__ coeff, double* __restrict__ qp) {
    const int64_t gamma = (k + tile - 1) / tile;
    const int64_t total = gamma * k * tq;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tau = i / ((int64_t)k * tq);
        const int kk = (int)((i / tq) % k), j = (int)(i % tq);
        const int64_t b = tau * tile;
        qp[i] = (j < tile && b + j < k) ? coeff[(int64_t)kk * k + b + j] : 0.0;
    }
}

// ---------------------------------------------------------------- reference H
constexpr int kRefHRows = 32;

template <class M>
__global__ void __launch_bounds__(kRefHRows) ref_update_h_kernel(int64_t d, int k, double eps,
                                                                 double* __restrict__ ht,
                                                                 const double* __restrict__ r,
                                                                 const double* __restrict__ s) {
    extern __shared__ double sh[];
    const int ld = k + 1;
    const int64_t row0 = (int64_t)blockIdx.x * kRefHRows;
    const int nrows = (int)((d - row0) < kRefHRows ? (d - row0) : kRefHRows);
    for (int idx = threadIdx.x; idx < nrows * k; idx += kRefHRows)
        sh[(idx / k) * ld + idx % k] = ht[row0 * k + idx];
    __syncthreads();
    if (threadIdx.x < nrows) {
        double* h = sh + threadIdx.x * ld;
        const double* rr = r + (row0 + threadIdx.x) * k;
        for (int kk = 0; kk < k; ++kk) {
            double dot = 0.0;
            for (int j = 0; j < k; ++j) dot = M::madd(dot, h[j], __ldg(&s[(int64_t)j * k + kk]));
            h[kk] = clamp_floor(eps, dsub(dadd(h[kk], rr[kk]), dot));  // hals.cpp:61
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrows * k; idx += kRefHRows)
        ht[row0 * k + idx] = sh[(idx / k) * ld + idx % k];
}

// ---------------------------------------------------------------- reference W
constexpr int kRefWThreads = 256;

struct RefWArgs {
    int64_t v;
    int k;
    double eps;
    int64_t rows_per_cta;
    double* w;
    const double* p;
    const double* q;
    double* norms;
    double* partials;
    unsigned* counters;
    double* totals;
};

template <class M>
__global__ void __launch_bounds__(kRefWThreads) ref_update_w_kernel(RefWArgs a) {
    __shared__ double red[48];
    const int k = a.k;
    const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
    const int64_t r1 = (r0 + a.rows_per_cta < a.v) ? r0 + a.rows_per_cta : a.v;
    for (int kk = 0; kk < k; ++kk) {
        const double qkk = a.q[(int64_t)kk * k + kk];
        double ss = 0.0;
        for (int64_t row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
            double* wr = a.w + row * k;
            double dot = 0.0;
            for (int j = 0; j < k; ++j) dot = M::madd(dot, wr[j], __ldg(&a.q[(int64_t)j * k + kk]));
            // hals.cpp:95: w*qkk + p - dot
            const double u = clamp_floor(a.eps, dsub(dadd(dmul(wr[kk], qkk), a.p[row * k + kk]), dot));
            wr[kk] = u;
            ss = M::madd(ss, u, u);
        }
        const double blk = block_sum(ss, red);
        if (threadIdx.x < kWarp) {
            const double nrm = grid_exchange(blk, kk, gridDim.x, a.partials, a.counters);
            if (threadIdx.x == 0) red[40] = nrm;
        }
        __syncthreads();
        const double norm = red[40];
        if (blockIdx.x == 0 && threadIdx.x == 0) a.norms[kk] = norm;
        for (int64_t row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
            double* x = a.w + row * k + kk;
            *x = clamp_floor(a.eps, __ddiv_rn(*x, norm));  // hals.cpp:102
        }
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

}  // namespace

namespace kern {

int64_t exchange_partials_doubles(int64_t k, int g) { return xch_partials(k, g); }
int64_t exchange_counters(int64_t k) { return xch_counters(k); }

PhaseBPlan plan_tiled_update(int64_t n, int64_t k, int64_t tile, bool normalize, int device) {
    PhaseBPlan plan;
    int max_smem = 0;
    PLNMF_CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    const int sms = sm_count(device);
    int64_t rpc = n > 0 ? (n + sms - 1) / sms : 1;  // one SM's share of rows
    if (std::getenv("PLNMF_FORCE_STREAMING")) return plan_stream_update(n, k, tile, normalize, device);
    // shared-memory variants, most staged first
    const bool variants[3][2] = {{true, true}, {false, true}, {false, false}};
    auto pick = [&](int64_t rows) -> int {
        for (int v = 0; v < 3; ++v)
            if (pl_smem(rows, k, tile, variants[v][0], variants[v][1]) <= (size_t)max_smem) return v;
        return -1;
    };
    int v = -1;
    if (normalize) {
        // persistent + grid-synchronised: exactly one resident CTA per SM with
        // one SM's rows (one row per chain thread); otherwise the streaming path
        v = rpc <= 8 * 32 ? pick(rpc) : -1;
        if (v < 0) return plan_stream_update(n, k, tile, normalize, device);
        plan.grid = sms;
        plan.cooperative = true;
    } else {
        while (rpc > 1 && pick(rpc) != 0 && rpc > 32) rpc = (rpc + 1) / 2;
        v = pick(rpc);
        if (v < 0) return plan_stream_update(n, k, tile, normalize, device);
        plan.grid = (int)((n + rpc - 1) / rpc);
    }
    plan.stage_ops = variants[v][0];
    plan.sqn_smem = variants[v][1];
    plan.rows_per_cta = rpc;
    plan.smem = pl_smem(rpc, k, tile, plan.stage_ops, plan.sqn_smem);
    return plan;
}

int64_t qpanel_doubles(int64_t k, int64_t tile) {
    const int64_t tq = (tile + 7) & ~int64_t(7);
    return ((k + tile - 1) / tile) * k * tq;
}

int tiled_update(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t n, int64_t k, int64_t tile,
                 double eps, bool w_update, const double* old_m, double* out, const double* coeff,
                 const double* add, double* norms, double* partials, unsigned* counters, double* totals,
                 long long* prof, double* qpanel) {
    if (n <= 0 || k <= 0) return 0;
    if (plan.streaming)
        return stream_update(s, m, plan, n, k, tile, eps, w_update, old_m, out, coeff, add, norms, partials,
                             counters);
    LookArgs a{n, (int)k, (int)tile, eps, w_update ? 1 : 0, (int)plan.rows_per_cta, old_m, out, coeff, add,
               norms, partials, counters, totals, prof, std::getenv("PLNMF_NO_OVERLAP") ? 0 : 1, nullptr,
               qpanel, plan.stage_ops ? 1 : 0, plan.sqn_smem ? 1 : 0};
    {
        const int tq = (int)((tile + 7) & ~int64_t(7));
        qpanel_kernel<<<(unsigned)std::min<int64_t>(1024, (qpanel_doubles(k, tile) + 255) / 256), 256, 0, s>>>(
            (int)k, (int)tile, tq, coeff, qpanel);
        PLNMF_CUDA_CHECK(cudaGetLastError());
    }
    static unsigned long long* trace_buf = nullptr;
    if (w_update && std::getenv("PLNMF_TRACE_EXCHANGE")) {
        if (!trace_buf) PLNMF_CUDA_CHECK(cudaMalloc(&trace_buf, sizeof(unsigned long long) * 3 * 1024 * 512));
        a.trace = trace_buf;
    }
    if (w_update) {
        exchange_reset(s, k, plan.grid, partials, counters);
        if (m == Math::exact) launch_pl<MathExact, true>(s, plan, a);
        else launch_pl<MathFused, true>(s, plan, a);
    } else {
        if (m == Math::exact) launch_pl<MathExact, false>(s, plan, a);
        else launch_pl<MathFused, false>(s, plan, a);
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
    if (a.trace) {
        const int g = plan.grid;
        std::vector<unsigned long long> h((size_t)3 * k * g);
        PLNMF_CUDA_CHECK(cudaMemcpyAsync(h.data(), a.trace, sizeof(unsigned long long) * h.size(),
                                         cudaMemcpyDeviceToHost, s));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
        double skew = 0, poll = 0, read = 0, gap = 0;
        for (int64_t t = 0; t < k; ++t) {
            unsigned long long amin = ~0ull, amax = 0, cmin = ~0ull, cmax = 0, rmax = 0;
            for (int c = 0; c < g; ++c) {
                const unsigned long long* x = &h[(size_t)(t * g + c) * 3];
                amin = std::min(amin, x[0]); amax = std::max(amax, x[0]);
                cmin = std::min(cmin, x[1]); cmax = std::max(cmax, x[1]);
                rmax = std::max(rmax, x[2]);
            }
            skew += double(amax - amin);
            poll += double(cmax - amax);
            read += double(rmax - cmax);
            if (t > 0) {
                unsigned long long pmax = 0;
                for (int c = 0; c < g; ++c) pmax = std::max(pmax, h[(size_t)((t - 1) * g + c) * 3 + 2]);
                gap += double(amin - pmax);
            }
        }
        std::fprintf(stderr, "[plnmf] exchange trace (ns/column): arrival skew %.0f, last-arrival->all-complete %.0f, "
                     "complete->partials read %.0f, prev-done->first-arrival %.0f\n",
                     skew / k, poll / k, read / k, gap / (k - 1));
    }
    return 1;
}

int reference_update_h(cudaStream_t s, Math m, int64_t d, int64_t k, double eps, double* ht,
                       const double* r, const double* sm) {
    if (d <= 0 || k <= 0) return 0;
    const size_t smem = sizeof(double) * (size_t)kRefHRows * (size_t)(k + 1);
    const dim3 grid((unsigned)((d + kRefHRows - 1) / kRefHRows));
    if (m == Math::exact) {
        PLNMF_CUDA_CHECK(cudaFuncSetAttribute(ref_update_h_kernel<MathExact>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ref_update_h_kernel<MathExact><<<grid, kRefHRows, smem, s>>>(d, (int)k, eps, ht, r, sm);
    } else {
        PLNMF_CUDA_CHECK(cudaFuncSetAttribute(ref_update_h_kernel<MathFused>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ref_update_h_kernel<MathFused><<<grid, kRefHRows, smem, s>>>(d, (int)k, eps, ht, r, sm);
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

PhaseBPlan plan_reference_w(int64_t v, int device) {
    PhaseBPlan plan;
    plan.grid = sm_count(device);
    plan.rows_per_cta = v > 0 ? (v + plan.grid - 1) / plan.grid : 1;
    plan.cooperative = true;
    return plan;
}

int reference_update_w(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t v, int64_t k, double eps,
                       double* w, const double* p, const double* q, double* norms, double* partials,
                       unsigned* counters, double* totals) {
    if (v <= 0 || k <= 0) return 0;
    exchange_reset(s, k, plan.grid, partials, counters);
    RefWArgs a{v, (int)k, eps, plan.rows_per_cta, w, p, q, norms, partials, counters, totals};
    void* args[] = {&a};
    const void* fn = (m == Math::exact) ? (const void*)ref_update_w_kernel<MathExact>
                                        : (const void*)ref_update_w_kernel<MathFused>;
    PLNMF_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, dim3((unsigned)plan.grid), dim3(kRefWThreads), args, 0, s));
    return 1;
}

}  // namespace kern
}  // namespace plnmf
