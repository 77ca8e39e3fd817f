// Streaming tiled (PL-NMF) update — the general fallback of the look-ahead
// kernel (update.cu) for shapes whose per-SM tile state does not fit in shared
// memory (large V and/or K: C3, C5).  Same per-element operation order as the
// reference (proj/src/tiled.cpp), so H is bit-identical and W differs only in
// the column-norm reduction order, exactly like the look-ahead path.
//
//   stream_phase_a  init_new_accumulator (:28-50) + phase1_left_contributions
//                   (:52-65) as a register-tiled SIMT GEMM into nb (global).
//   stream_update   one persistent launch (cooperative for W): for each tile,
//                   phase 2 (:67-156) one thread per row with the row's tile
//                   operands streamed from global/L1, the column norm through
//                   the grid exchange, then phase 3 (:158-174) over the CTA's
//                   own rows (4 independent columns per thread).
#include "common.cuh"
#include "exchange.cuh"
#include "kernels.cuh"

namespace plnmf {
namespace {

constexpr int kTileRows = 64, kTileCols = 64, kTileK = 16, kPhaseAThreads = 256;

template <class M>
__global__ void __launch_bounds__(kPhaseAThreads) stream_phase_a_kernel(int64_t n, int k, int tile,
                                                                        int use_diag,
                                                                        const double* __restrict__ old_m,
                                                                        const double* __restrict__ coeff,
                                                                        double* __restrict__ nb) {
    __shared__ double As[kTileK][kTileRows + 1];  // old(r0+rr, k0+kk) at [kk][rr]
    __shared__ double Bs[kTileK][kTileCols];      // -coeff(k0+kk, c0+cc)
    const int c0 = blockIdx.x * kTileCols;
    const int64_t r0 = (int64_t)blockIdx.y * kTileRows;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
    int estart[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = c0 + tx + 16 * j;
        const int e = (c / tile + 1) * tile;  // first column right of c's tile
        estart[j] = e < k ? e : k;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t r = r0 + ty + 16 * i;
            const int c = c0 + tx + 16 * j;
            double x = 0.0;
            if (r < n && c < k) {
                x = old_m[r * k + c];
                if (use_diag) x = dmul(x, coeff[(int64_t)c * k + c]);  // tiled.cpp:44
            }
            acc[i][j] = x;
        }
    const int kbeg = ((c0 / tile + 1) * tile) < k ? (c0 / tile + 1) * tile : k;
    for (int k0 = kbeg; k0 < k; k0 += kTileK) {
        for (int idx = threadIdx.x; idx < kTileK * kTileRows; idx += kPhaseAThreads) {
            const int rr = idx / kTileK, kk = idx % kTileK;
            As[kk][rr] = (r0 + rr < n && k0 + kk < k) ? old_m[(r0 + rr) * k + k0 + kk] : 0.0;
            const int kb = idx / kTileCols, cc = idx % kTileCols;
            // f = alpha * b(kk, j) with alpha = -1 (tiled.cpp:58-60, linalg.cpp:52)
            Bs[kb][cc] = (k0 + kb < k && c0 + cc < k) ? -1.0 * coeff[(int64_t)(k0 + kb) * k + c0 + cc] : 0.0;
        }
        __syncthreads();
        const int kmax = (k - k0) < kTileK ? (k - k0) : kTileK;
        for (int kk = 0; kk < kmax; ++kk) {
            const int kabs = k0 + kk;
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (kabs >= estart[j]) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[i][j] = M::madd(acc[i][j], bv[j], av[i]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t r = r0 + ty + 16 * i;
            const int c = c0 + tx + 16 * j;
            if (r < n && c < k) nb[r * k + c] = acc[i][j];
        }
}

constexpr int kSThreads = 512;

struct StreamArgs {
    int64_t n;
    int k;
    int tile;
    double eps;
    int64_t rows_per_cta;
    const double* old_m;
    double* nb;
    const double* coeff;
    const double* add;
    double* norms;
    double* partials;
    unsigned* counters;
    WorldXch xch;  // WORLD: the other ranks' windows (sharded engine)
    double* xs;    // stream_w_kernel: per-CTA column-major tile scratch, 3 x tile x ldx doubles per CTA
    int64_t ldx;
    FusedPush push;  // WORLD: the finished tiles also go to every other rank's window (all-gather)
};

template <class M, bool NORMALIZE, bool WORLD = false>
__global__ void __launch_bounds__(kSThreads, 1) stream_update_kernel(StreamArgs p) {
    __shared__ double red[48];
    const int k = p.k, T = p.tile, tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_cta;
    const int64_t r1 = (r0 + p.rows_per_cta < p.n) ? r0 + p.rows_per_cta : p.n;
    for (int b = 0; b < k; b += T) {
        const int e = (b + T < k) ? b + T : k, w = e - b;
        // ---- phase 2: columns in order; each thread keeps the same rows throughout
        for (int t = b; t < e; ++t) {
            const int tt = t - b;
            double ss = 0.0;
            for (int64_t r = r0 + tid; r < r1; r += kSThreads) {
                const double* nr = p.nb + r * k + b;
                const double* orow = p.old_m + r * k + b;
                const double a_t = nr[tt], add_t = p.add[r * k + t];
                double s = 0.0;
                // operands in batches of 8 independent loads (new for j < tt, old for j >= tt),
                // then the scratch terms in the reference's order
                for (int j0 = 0; j0 < w; j0 += 8) {
                    double x[8], c[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + u;
                        x[u] = (j < w) ? (j < tt ? nr[j] : orow[j]) : 0.0;
                        c[u] = (j < w) ? __ldg(p.coeff + (int64_t)(b + j) * k + t) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (j0 + u < w) s = M::madd(s, x[u], c[u]);
                }
                const double val = clamp_floor(p.eps, dsub(dadd(a_t, add_t), s));
                p.nb[r * k + t] = val;
                if (NORMALIZE) ss = M::madd(ss, val, val);
            }
            if (NORMALIZE) {
                const double blk = block_sum(ss, red);
                if (tid < kWarp) {
                    const double nrm =
                        WORLD ? __dsqrt_rn(world_sum(grid_exchange_sum(blk, t, gridDim.x, p.partials, p.counters), t,
                                                     p.xch))
                              : grid_exchange(blk, t, gridDim.x, p.partials, p.counters);
                    if (tid == 0) {
                        red[40] = nrm;
                        if (blockIdx.x == 0) p.norms[t] = nrm;
                    }
                }
                __syncthreads();
                const double norm = red[40];
                for (int64_t r = r0 + tid; r < r1; r += kSThreads) {
                    double* x = p.nb + r * k + t;
                    *x = clamp_floor(p.eps, __ddiv_rn(*x, norm));  // tiled.cpp:146
                }
            }
        }
        __syncthreads();
        // ---- phase 3 over this CTA's rows: nb(r,c) += (-coeff(kk,c)) * nb(r,kk), kk in the tile
        const int rest = k - e;
        if (rest > 0) {
            const int ng = (rest + 3) / 4;
            const int64_t items = (r1 - r0) * ng;
            for (int64_t it = tid; it < items; it += kSThreads) {
                const int64_t r = r0 + it / ng;
                const int c0 = e + (int)(it % ng) * 4;
                double* row = p.nb + r * k;
                double a[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = (c0 + u < k) ? row[c0 + u] : 0.0;
                for (int j0 = 0; j0 < w; j0 += 8) {
                    double x[8];
#pragma unroll
                    for (int v = 0; v < 8; ++v) x[v] = (j0 + v < w) ? row[b + j0 + v] : 0.0;
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        if (j0 + v < w) {
                            const double* cf = p.coeff + (int64_t)(b + j0 + v) * k + c0;
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (c0 + u < k) a[u] = M::madd(a[u], -1.0 * __ldg(cf + u), x[v]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (c0 + u < k) row[c0 + u] = a[u];
            }
        }
        __syncthreads();
    }
}

// The W update of the streaming plan with its phase 2 on a column-major copy of
// the tile.  Phase 2 needs, for every column t, all w tile values of every row
// (new for j < t, old for j >= t, tiled.cpp:103-128).  Read from the row-major
// factor those are 32 scattered rows per warp load, re-fetched for every
// column (ncu at C5: 361 GB of DRAM traffic per update for 12 GB of compulsory
// bytes).  Here each CTA first copies its rows' tile into X (old values, then
// overwritten in place by the new values: exactly the operands the reference
// reads), the accumulators into AC and the additive term into AD, all
// column-major, so every phase-2 load is a coalesced column read; the finished
// tile is copied back to the row-major factor.  Phase 3 runs as a look-ahead:
// only the next tile's accumulators are built (their phase-A values plus every
// finished tile's terms, in tile order), so the far columns are read but never
// rewritten.  Same per-element operation order as stream_update_kernel.
constexpr int kSWarps = kSThreads / kWarp;

// NORMALIZE: the W update (every column normalised through the grid exchange); without it
// the H update.  WORLD (sharded): W's norm exchange spans the ranks, and the finished tiles
// are pushed into every other rank's window (the factor all-gather fused into the update).
template <class M, bool NORMALIZE, bool WORLD>
__global__ void __launch_bounds__(kSThreads, 1) stream_w_kernel(StreamArgs p) {
    __shared__ double red[48];
    // dynamic: phase 3's negated coefficient rows (w x (k - e)); the transposes' per-warp stages
    // (T x 33 each) — never live at the same time
    extern __shared__ __align__(16) double cq[];
    const int k = p.k, T = p.tile, tid = threadIdx.x;
    const int warp = tid / kWarp, lane = lane_id();
    double* st = cq + (int64_t)warp * T * (kWarp + 1);
    const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_cta;
    const int64_t r1 = (r0 + p.rows_per_cta < p.n) ? r0 + p.rows_per_cta : p.n;
    const int64_t nl = r1 > r0 ? r1 - r0 : 0;
    const int64_t ld = p.ldx;
    double* X = p.xs + (int64_t)blockIdx.x * 3 * T * ld;
    double* AC = X + (int64_t)T * ld;
    double* AD = AC + (int64_t)T * ld;
    // Phase 3, two ways.  Many rows per CTA (C5: 13.5 K): as a look-ahead that builds only the
    // next tile's accumulators (the far columns read, never rewritten: 35 instead of 61 GB at C5).
    // Few rows (TDT2, K=480: 249): the per-tile read-modify-write of the later columns, whose
    // (row, 4-column) items keep every thread busy (measured: 5.2 vs 5.9 ms per W update).
    const bool narrow = nl < 2 * kSThreads;
    for (int b = 0; b < k; b += T) {
        const int e = (b + T < k) ? b + T : k, w = e - b;
        // ---- the tile, column-major: each warp transposes 32-row chunks through its own
        // shared-memory stage (row segments in, coalesced 32-row column pieces out).  The
        // accumulators AC of tiles after the first were built by the previous tile's look-ahead.
        for (int64_t i0 = (int64_t)warp * kWarp; i0 < nl; i0 += (int64_t)kSWarps * kWarp) {
            const double* src[3] = {p.old_m, p.add, p.nb};
            double* dst[3] = {X, AD, AC};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (a == 2 && b > 0 && !narrow) break;  // built by the previous tile's look-ahead
                for (int idx = lane; idx < kWarp * w; idx += kWarp) {
                    const int ii = idx / w, j = idx - ii * w;
                    if (i0 + ii < nl) st[j * (kWarp + 1) + ii] = src[a][(r0 + i0 + ii) * k + b + j];
                }
                __syncwarp();
                if (i0 + lane < nl)
                    for (int j = 0; j < w; ++j) dst[a][j * ld + i0 + lane] = st[j * (kWarp + 1) + lane];
                __syncwarp();
            }
        }
        __syncthreads();
        // ---- phase 2: columns in order; each thread keeps the same rows throughout
        for (int t = b; t < e; ++t) {
            const int tt = t - b;
            double ss = 0.0;
            if (w <= 16) {
                double c[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) c[j] = (j < w) ? __ldg(p.coeff + (int64_t)(b + j) * k + t) : 0.0;
                for (int64_t i = tid; i < nl; i += kSThreads) {
                    double x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) x[j] = (j < w) ? X[j * ld + i] : 0.0;
                    double s = 0.0;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < w) s = M::madd(s, x[j], c[j]);
                    const double val = clamp_floor(p.eps, dsub(dadd(AC[tt * ld + i], AD[tt * ld + i]), s));
                    X[tt * ld + i] = val;
                    ss = M::madd(ss, val, val);
                }
            } else {
                for (int64_t i = tid; i < nl; i += kSThreads) {
                    double s = 0.0;
                    for (int j0 = 0; j0 < w; j0 += 8) {
                        double x[8], c[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = j0 + u;
                            x[u] = (j < w) ? X[j * ld + i] : 0.0;
                            c[u] = (j < w) ? __ldg(p.coeff + (int64_t)(b + j) * k + t) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (j0 + u < w) s = M::madd(s, x[u], c[u]);
                    }
                    const double val = clamp_floor(p.eps, dsub(dadd(AC[tt * ld + i], AD[tt * ld + i]), s));
                    X[tt * ld + i] = val;
                    if (NORMALIZE) ss = M::madd(ss, val, val);
                }
            }
            if (NORMALIZE) {
                const double blk = block_sum(ss, red);
                if (tid < kWarp) {
                    const double nrm =
                        WORLD ? __dsqrt_rn(world_sum(grid_exchange_sum(blk, t, gridDim.x, p.partials, p.counters), t,
                                                     p.xch))
                              : grid_exchange(blk, t, gridDim.x, p.partials, p.counters);
                    if (tid == 0) {
                        red[40] = nrm;
                        if (blockIdx.x == 0) p.norms[t] = nrm;
                    }
                }
                __syncthreads();
                const double norm = red[40];
                for (int64_t i = tid; i < nl; i += kSThreads)
                    X[tt * ld + i] = clamp_floor(p.eps, __ddiv_rn(X[tt * ld + i], norm));  // tiled.cpp:146
            }
        }
        if (narrow) {
            // ---- phase 3 (tiled.cpp:158-174): nb(r, c) += (-coeff(b+j, c)) * new(r, b+j), j ascending,
            // for every c >= e.  One thread per row: the row's w new values (a coalesced column read of X)
            // stay in registers for all its columns; the tile's coefficient rows are staged in shared
            // memory (every thread reads the same entry: broadcast); 4 columns of the row per step
            // (32-byte sector-sized accesses of the row-major factor).
            if (e < k) {
                const int rest = k - e;
                for (int idx = tid; idx < w * rest; idx += kSThreads) {
                    const int j = idx / rest, c = idx - j * rest;
                    cq[j * rest + c] = -1.0 * p.coeff[(int64_t)(b + j) * k + e + c];
                }
                __syncthreads();
                const bool vec4 = (k % 2 == 0) && (e % 2 == 0);
                for (int64_t i = tid; i < nl; i += kSThreads) {
                    double x[16];
                    const bool small = w <= 16;
                    if (small) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) x[j] = (j < w) ? X[j * ld + i] : 0.0;
                    }
                    double* row = p.nb + (r0 + i) * k + e;
                    auto load4 = [&](int c0, double (&a)[4]) {
                        if (c0 + 4 <= rest && vec4) {
                            const double2 lo = *reinterpret_cast<const double2*>(row + c0);
                            const double2 hi = *reinterpret_cast<const double2*>(row + c0 + 2);
                            a[0] = lo.x; a[1] = lo.y; a[2] = hi.x; a[3] = hi.y;
                        } else {
#pragma unroll
                            for (int u = 0; u < 4; ++u) a[u] = (c0 + u < rest) ? row[c0 + u] : 0.0;
                        }
                    };
                    double an[4];
                    load4(0, an);
                    for (int c0 = 0; c0 < rest; c0 += 4) {
                        double a[4];
                        const bool full = c0 + 4 <= rest;
#pragma unroll
                        for (int u = 0; u < 4; ++u) a[u] = an[u];
                        if (c0 + 4 < rest) load4(c0 + 4, an);  // the next group's loads in flight during this one
                        if (small) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                if (j < w) {
                                    const double* q = cq + j * rest + c0;
#pragma unroll
                                    for (int u = 0; u < 4; ++u)
                                        if (c0 + u < rest) a[u] = M::madd(a[u], q[u], x[j]);
                                }
                            }
                        } else {
                            for (int j = 0; j < w; ++j) {
                                const double xj = X[j * ld + i];
                                const double* q = cq + j * rest + c0;
#pragma unroll
                                for (int u = 0; u < 4; ++u)
                                    if (c0 + u < rest) a[u] = M::madd(a[u], q[u], xj);
                            }
                        }
                        if (full && vec4) {
                            *reinterpret_cast<double2*>(row + c0) = make_double2(a[0], a[1]);
                            *reinterpret_cast<double2*>(row + c0 + 2) = make_double2(a[2], a[3]);
                        } else {
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (c0 + u < rest) row[c0 + u] = a[u];
                        }
                    }
                }
            }
            __syncthreads();
        }
        // ---- the finished tile back to the row-major factor (the same warp-level transpose);
        // sharded: also into every other rank's window — the W all-gather fused into the update,
        // each tile's rows travelling over NVLink while the later tiles compute
        for (int64_t i0 = (int64_t)warp * kWarp; i0 < nl; i0 += (int64_t)kSWarps * kWarp) {
            if (i0 + lane < nl)
                for (int j = 0; j < w; ++j) st[j * (kWarp + 1) + lane] = X[j * ld + i0 + lane];
            __syncwarp();
            for (int idx = lane; idx < kWarp * w; idx += kWarp) {
                const int ii = idx / w, j = idx - ii * w;
                if (i0 + ii < nl) {
                    const int64_t g = (r0 + i0 + ii) * k + b + j;
                    const double v = st[j * (kWarp + 1) + ii];
                    p.nb[g] = v;
                    if (WORLD) {
#pragma unroll
                        for (int q = 0; q < kMaxWorld; ++q)
                            if (q < p.push.world && q != p.push.rank) p.push.dst[q][g] = v;
                    }
                }
            }
            __syncwarp();
        }
        __syncthreads();
        // ---- phase 3 as a look-ahead (tiled.cpp:158-174): phase 3 of every finished tile adds to
        // the later columns in tile order; the next tile's columns are the only ones the next phase
        // 2 reads, so they are built here — their phase-A values (in nb, never rewritten) plus the
        // sum over kk < e of (-coeff(kk, c)) * new(r, kk), kk ascending: the reference's order —
        // straight into the column-major AC.  The far columns are read, never rewritten.  One
        // thread per row; the next tile's coefficient panel in shared memory (broadcast reads).
        if (!narrow && e < k) {
            const int bn = e, wn = (bn + T < k) ? T : k - bn;
            for (int idx = tid; idx < e * wn; idx += kSThreads) {
                const int kk = idx / wn, c = idx - kk * wn;
                cq[kk * wn + c] = -1.0 * p.coeff[(int64_t)kk * k + bn + c];
            }
            __syncthreads();
            for (int64_t i = tid; i < nl; i += kSThreads) {
                const double* row = p.nb + (r0 + i) * k;
                if (wn <= 16) {
                    double a[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) a[c] = (c < wn) ? row[bn + c] : 0.0;
                    for (int kk = 0; kk < e; ++kk) {
                        const double xv = row[kk];
                        const double* q = cq + kk * wn;
#pragma unroll
                        for (int c = 0; c < 16; ++c)
                            if (c < wn) a[c] = M::madd(a[c], q[c], xv);
                    }
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        if (c < wn) AC[c * ld + i] = a[c];
                } else {
                    for (int c0 = 0; c0 < wn; c0 += 8) {
                        double a[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) a[c] = (c0 + c < wn) ? row[bn + c0 + c] : 0.0;
                        for (int kk = 0; kk < e; ++kk) {
                            const double xv = row[kk];
                            const double* q = cq + kk * wn + c0;
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                if (c0 + c < wn) a[c] = M::madd(a[c], q[c], xv);
                        }
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            if (c0 + c < wn) AC[(c0 + c) * ld + i] = a[c];
                    }
                }
            }
        }
        __syncthreads();
    }
    if (WORLD) fused_push_finish(p.push);
}

int sm_count(int device) {
    int n = 0;
    PLNMF_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

}  // namespace

namespace kern {

int stream_phase_a(cudaStream_t s, Math m, int64_t n, int64_t k, int64_t tile, bool use_diag, const double* old_m,
                   const double* coeff, double* nb) {
    if (n <= 0 || k <= 0) return 0;
    const dim3 ga((unsigned)((k + kTileCols - 1) / kTileCols), (unsigned)((n + kTileRows - 1) / kTileRows));
    if (m == Math::exact)
        stream_phase_a_kernel<MathExact><<<ga, kPhaseAThreads, 0, s>>>(n, (int)k, (int)tile, use_diag, old_m, coeff, nb);
    else
        stream_phase_a_kernel<MathFused><<<ga, kPhaseAThreads, 0, s>>>(n, (int)k, (int)tile, use_diag, old_m, coeff, nb);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

PhaseBPlan plan_stream_update(int64_t n, int64_t k, int64_t tile, bool normalize, int device) {
    (void)k;
    (void)tile;
    PhaseBPlan plan;
    const int sms = sm_count(device);
    if (normalize) {
        plan.grid = sms;  // one resident CTA per SM, grid exchange per column
        plan.cooperative = true;
    } else {
        plan.grid = (int)std::min<int64_t>(std::max<int64_t>(1, (n + 63) / 64), 4 * (int64_t)sms);
    }
    plan.rows_per_cta = n > 0 ? (n + plan.grid - 1) / plan.grid : 1;
    plan.streaming = true;
    return plan;
}

int64_t stream_w_scratch_doubles(const PhaseBPlan& plan, int64_t tile) {
    return (int64_t)plan.grid * 3 * tile * plan.rows_per_cta;
}

bool stream_fuses_push(int64_t k, int64_t tile) {
    const size_t w_smem = sizeof(double) * (size_t)std::max<int64_t>(tile * k, (int64_t)kSWarps * tile * (kWarp + 1));
    return tile <= 32 && w_smem <= 200 * 1024;
}

int stream_update(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t n, int64_t k, int64_t tile,
                  double eps, bool w_update, const double* old_m, double* out, const double* coeff,
                  const double* add, double* norms, double* partials, unsigned* counters, const WorldXch* xch,
                  double* scratch, const FusedPush* push, void* tensor_ws) {
    if (n <= 0 || k <= 0) return 0;
    // phase A: init + phase 1 into `out` (used as the accumulator nb)
    int launches = 2;
    if (tensor_ws) {
        launches += tensor_phase_a(s, n, k, tile, w_update, old_m, coeff, out, tensor_ws) - 1;
    } else {
        const dim3 ga((unsigned)((k + kTileCols - 1) / kTileCols), (unsigned)((n + kTileRows - 1) / kTileRows));
        if (m == Math::exact)
            stream_phase_a_kernel<MathExact><<<ga, kPhaseAThreads, 0, s>>>(n, (int)k, (int)tile, w_update, old_m, coeff, out);
        else
            stream_phase_a_kernel<MathFused><<<ga, kPhaseAThreads, 0, s>>>(n, (int)k, (int)tile, w_update, old_m, coeff, out);
        PLNMF_CUDA_CHECK(cudaGetLastError());
    }
    const bool world = xch && xch->world > 1;
    // stream_w_kernel: tiles up to 32 wide; shared memory for the coefficient rows and the stages
    const size_t w_smem = sizeof(double) * (size_t)std::max<int64_t>(tile * k, (int64_t)kSWarps * tile * (kWarp + 1));
    if (scratch && !stream_fuses_push(k, tile)) scratch = nullptr;
    if (push && push->world > 1 && !scratch) throw std::logic_error("stream_update: a fused push needs stream_w_kernel");
    StreamArgs a{n, (int)k, (int)tile, eps, plan.rows_per_cta, old_m, out, coeff, add, norms, partials, counters,
                 world ? *xch : WorldXch{}, scratch, plan.rows_per_cta, push ? *push : FusedPush{}};
    const dim3 grid((unsigned)plan.grid), block(kSThreads);
    const bool pushing = push && push->world > 1;
    const size_t smem = scratch ? w_smem : 0;
    void* args[] = {&a};
    auto launch = [&](const void* fn, bool cooperative) {
        // stream_w_kernel: the tile's coefficient rows for phase 3 in dynamic shared memory
        if (smem > 48 * 1024) PLNMF_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // a plan with fewer CTAs than SMs (ranks sharing one GPU) is co-resident with
        // the other ranks' kernels only under a plain launch
        if (cooperative) PLNMF_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, grid, block, args, smem, s));
        else PLNMF_CUDA_CHECK(cudaLaunchKernel(fn, grid, block, args, smem, s));
    };
    const bool ex = m == Math::exact;
    if (w_update) {
        exchange_reset(s, k, plan.grid, partials, counters);
        const void* fn;
        if (scratch)  // column-major tile scratch (stream_w_kernel)
            fn = world ? (ex ? (const void*)stream_w_kernel<MathExact, true, true> : (const void*)stream_w_kernel<MathFused, true, true>)
                       : (ex ? (const void*)stream_w_kernel<MathExact, true, false> : (const void*)stream_w_kernel<MathFused, true, false>);
        else
            fn = world ? (ex ? (const void*)stream_update_kernel<MathExact, true, true>
                             : (const void*)stream_update_kernel<MathFused, true, true>)
                       : (ex ? (const void*)stream_update_kernel<MathExact, true> : (const void*)stream_update_kernel<MathFused, true>);
        launch(fn, plan.cooperative);
    } else if (scratch) {
        const void* fn = pushing ? (ex ? (const void*)stream_w_kernel<MathExact, false, true>
                                       : (const void*)stream_w_kernel<MathFused, false, true>)
                                 : (ex ? (const void*)stream_w_kernel<MathExact, false, false>
                                       : (const void*)stream_w_kernel<MathFused, false, false>);
        launch(fn, false);
    } else if (ex) {
        stream_update_kernel<MathExact, false><<<grid, block, 0, s>>>(a);
    } else {
        stream_update_kernel<MathFused, false><<<grid, block, 0, s>>>(a);
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return launches;
}

}  // namespace kern
}  // namespace plnmf
