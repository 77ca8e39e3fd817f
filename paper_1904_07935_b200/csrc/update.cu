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
#include "lookahead.cuh"
#include "update_kern.cuh"

namespace plnmf {
namespace upd {
extern template void launch_pl<MathExact, true>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
extern template void launch_pl<MathExact, false>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
extern template void launch_pl<MathFused, true>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
extern template void launch_pl<MathFused, false>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
}  // namespace upd
namespace {
using upd::LookArgs;
using upd::launch_pl;
using upd::kLThreads;

int sm_count(int device) {
    int n = 0;
    PLNMF_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

// look-ahead threads of a CTA with `rows` rows (the kernel's warp split)
int pl_nupd(int64_t rows, bool normalize) {
    const int row_warps = (int)std::min<int64_t>(8, std::max<int64_t>(1, (rows + 31) / 32));
    return kLThreads - 32 * (row_warps + (normalize ? 1 : 0));
}
// rings of the staged look-ahead GEMM: one per thread that owns items
int64_t pl_kbuf(int64_t rows, int64_t k, int64_t tile, bool normalize) {
    const int64_t items = rows * ((std::min<int64_t>(tile, k) + 15) / 16);
    return std::min<int64_t>(items, pl_nupd(rows, normalize));
}
size_t pl_smem(int64_t rows, int64_t k, int64_t tile, bool stage_ops, bool sqn_smem, int kc, int kst = 2,
               bool normalize = false) {
    const int64_t tq = (tile + 7) & ~int64_t(7);
    const int64_t ldt = (tile + 1) | 1;  // the kernel's odd shared-memory row stride
    const int64_t prods = (normalize && tile <= 32) ? rows * ldt : 0;  // W chain products (exact path)
    const int64_t rings = kc > 0 ? kst * pl_kbuf(rows, k, tile, normalize) * (kc + 2) : 0;
    return sizeof(double) * (size_t)((stage_ops ? 4 : 2) * rows * ldt + (sqn_smem ? k * tq : 0) +
                                     tile * tile + 48 + 1 + rings + prods);
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
    WorldXch xch;  // WORLD: the column norms span the ranks of a sharded engine (peer.cuh)
};

template <class M, bool WORLD = false>
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
            const double nrm =
                WORLD ? __dsqrt_rn(world_sum(grid_exchange_sum(blk, kk, gridDim.x, a.partials, a.counters), kk, a.xch))
                      : grid_exchange(blk, kk, gridDim.x, a.partials, a.counters);
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


}  // namespace

namespace kern {

int64_t exchange_partials_doubles(int64_t k, int g) { return xch_partials(k, g); }
int64_t exchange_counters(int64_t k) { return xch_counters(k); }

namespace {
// developer-build knobs only (common.cuh: kDebugKnobs); always false in production
bool knob(const char* name) { return kDebugKnobs && std::getenv(name) != nullptr; }
int knob_int(const char* name) { return knob(name) ? std::atoi(std::getenv(name)) : 0; }
}  // namespace

PhaseBPlan plan_tiled_update(int64_t n, int64_t k, int64_t tile, bool normalize, int device, bool force_streaming) {
    PhaseBPlan plan;
    int max_smem = 0;
    PLNMF_CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    const int sms = sm_count(device);
    int64_t rpc = n > 0 ? (n + sms - 1) / sms : 1;  // one SM's share of rows
    if (force_streaming) return plan_stream_update(n, k, tile, normalize, device);
    // shared-memory variants, most staged first
    const bool variants[3][2] = {{true, true}, {false, true}, {false, false}};
    // the staged look-ahead GEMM wants >= 8-wide operand chunks; an unstaged
    // look-ahead is the last resort of each variant
    auto pick = [&](int64_t rows) -> int {
        for (int v = 0; v < 3; ++v)
            if (pl_smem(rows, k, tile, variants[v][0], variants[v][1], kPrivKC, 2, normalize) <= (size_t)max_smem) return v;
        for (int v = 0; v < 3; ++v)
            if (pl_smem(rows, k, tile, variants[v][0], variants[v][1], 0, 2, normalize) <= (size_t)max_smem) return v;
        return -1;
    };
    int v = -1;
    if (normalize) {
        // persistent + grid-synchronised: exactly one resident CTA per SM with
        // one SM's rows (one row per chain thread); otherwise the streaming path
        v = rpc <= 8 * 32 ? pick(rpc) : -1;
        // neither the operands nor the coefficient panel staged (plan 2): at large K the look-ahead
        // re-reads the panel from global for every row and the streaming kernel wins (measured,
        // tools/tile_plans.py: TDT2 K=480, T=20-32: 8.0-10.0 ms vs 5.2-5.9 ms per W update; at
        // 20News K=240, T=24 the look-ahead still wins, 1.57 vs 1.71 ms)
        if (v == 2 && k > 320) v = -1;
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
    plan.kc = 0;
    plan.kst = 0;
    {
        // the staged GEMM runs items (row x 16 columns) round-robin over the look-ahead threads
        const int nupd = pl_nupd(rpc, normalize);
        const int64_t items = rpc * ((std::min<int64_t>(tile, k) + 15) / 16);
        if (!knob("PLNMF_NO_STAGED_GEMM") && plan.sqn_smem && items <= 4 * (int64_t)nupd)
            for (int st : {3, 2})
                if (pl_smem(rpc, k, tile, plan.stage_ops, plan.sqn_smem, kPrivKC, st, normalize) <= (size_t)max_smem) {
                    plan.kc = kPrivKC;
                    plan.kst = st;
                    plan.kbuf = (int)pl_kbuf(rpc, k, tile, normalize);
                    break;
                }
    }
    plan.smem = pl_smem(rpc, k, tile, plan.stage_ops, plan.sqn_smem, plan.kc, plan.kst, normalize);
    if (!normalize && tile <= 16 && !knob("PLNMF_NO_RESIDENT")) {
        // H: keep the CTA's rows resident in shared memory when they fit (no
        // staging, no oldB), up to 4 rows per look-ahead thread of a column
        const int64_t tq = (tile + 7) & ~int64_t(7);
        const size_t smem = sizeof(double) * (size_t)(2 * rpc * ((tile + 1) | 1) + k * tq + tile * tile + 48 + 1 +
                                                      rpc * (k + 2));
        if (smem <= (size_t)max_smem && rpc <= 4 * (pl_nupd(rpc, false) / 16)) {
            plan.resident = 1;
            plan.stage_ops = false;
            plan.sqn_smem = true;
            plan.kc = 0;
            plan.kst = 0;
            plan.kbuf = 0;
            plan.smem = smem;
        }
    }
    return plan;
}

int64_t qpanel_doubles(int64_t k, int64_t tile) {
    const int64_t tq = (tile + 7) & ~int64_t(7);
    return ((k + tile - 1) / tile) * k * tq;
}

int tiled_update(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t n, int64_t k, int64_t tile,
                 double eps, bool w_update, const double* old_m, double* out, const double* coeff,
                 const double* add, double* norms, double* partials, unsigned* counters, double* totals,
                 long long* prof, double* qpanel, double* stream_scratch, const FusedPush* push,
                 void* tensor_ws) {
    if (n <= 0 || k <= 0) return 0;
    if (plan.streaming)
        return stream_update(s, m, plan, n, k, tile, eps, w_update, old_m, out, coeff, add, norms, partials,
                             counters, nullptr, stream_scratch, push, tensor_ws);
    if (push && push->world > 1) throw std::logic_error("tiled_update: a fused push needs the streaming plan");
    LookArgs a{n, (int)k, (int)tile, eps, w_update ? 1 : 0, (int)plan.rows_per_cta, old_m, out, coeff, add,
               norms, partials, counters, totals, prof, knob("PLNMF_NO_OVERLAP") ? 0 : knob("PLNMF_SKIP_LOOKAHEAD") ? 2 : 1,
               nullptr, qpanel, plan.stage_ops ? 1 : 0, plan.sqn_smem ? 1 : 0, plan.kc, plan.kst, plan.kbuf,
               knob_int("PLNMF_DBG"), plan.resident, (int)k + 2};
    const bool panel = !plan.sqn_smem || !w_update;  // the W kernel stages its panels from coeff
    if (panel) {
        const int tq = (int)((tile + 7) & ~int64_t(7));
        qpanel_kernel<<<(unsigned)std::min<int64_t>(1024, (qpanel_doubles(k, tile) + 255) / 256), 256, 0, s>>>(
            (int)k, (int)tile, tq, coeff, qpanel);
        PLNMF_CUDA_CHECK(cudaGetLastError());
    }
    static unsigned long long* trace_buf = nullptr;  // developer builds only (one process, one device)
    if (w_update && knob("PLNMF_TRACE_EXCHANGE")) {
        if (!trace_buf) PLNMF_CUDA_CHECK(cudaMalloc(&trace_buf, sizeof(unsigned long long) * kTraceSlots * 1024 * 512));
        a.trace = trace_buf;
        PLNMF_CUDA_CHECK(cudaMemsetAsync(trace_buf, 0, sizeof(unsigned long long) * kTraceSlots * 1024 * 512, s));
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
    if (kDebugKnobs && a.trace) {
        const int g = plan.grid;
        std::vector<unsigned long long> h((size_t)kTraceSlots * k * g);
        PLNMF_CUDA_CHECK(cudaMemcpyAsync(h.data(), a.trace, sizeof(unsigned long long) * h.size(),
                                         cudaMemcpyDeviceToHost, s));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(s));
        // SM-clock durations per CTA (clocks are per SM: only same-CTA differences are meaningful).
        // Stamps: 0 arrival, 1 counter complete, 2 partials read (exchange warp); 3 exchange warp
        // past the norm barrier; 4 chain warp 0 past the norm barrier, 5 its next value done,
        // 6 its square reduced and parked; 7 exchange warp has the CTA partial.
        const int S = kTraceSlots;
        auto span = [&](bool boundary, int a0, int a1, bool prev) {
            double sum = 0;
            int64_t n = 0;
            for (int c = 0; c < g; ++c)
                for (int64_t t = prev ? 1 : 0; t < k; ++t) {
                    if (((t % tile) == 0) != boundary) continue;
                    const unsigned long long* x = &h[(size_t)(t * g + c) * S];
                    const unsigned long long* xp = prev ? &h[(size_t)((t - 1) * g + c) * S] : x;
                    if (!xp[a0] || !x[a1]) continue;
                    sum += double((long long)(x[a1] - xp[a0]));
                    ++n;
                }
            return n ? sum / n : 0.0;
        };
        for (int bnd = 0; bnd < 2; ++bnd)
            std::fprintf(stderr,
                         "[plnmf] exchange trace, %s columns (SM cycles, mean over CTAs): arrive->complete %.0f, "
                         "->read %.0f, ->xwarp past barrier %.0f, read->chain past barrier %.0f, ->value %.0f | "
                         "prev value->square parked %.0f, ->xwarp has partial %.0f, ->arrive %.0f\n",
                         bnd ? "tile-first" : "in-tile", span(bnd, 0, 1, false), span(bnd, 1, 2, false),
                         span(bnd, 2, 3, false), span(bnd, 2, 4, false), span(bnd, 4, 5, false), span(bnd, 5, 6, true),
                         span(bnd, 6, 7, false), span(bnd, 7, 0, false));
        // tile boundaries: stamps 9..13 on each tile's last column (chain warp 0; the exact
        // W path publishes without a stamp of its own, so the first span includes the publish)
        double bs[5] = {0, 0, 0, 0, 0};
        int64_t nb = 0;
        for (int c = 0; c < g; ++c)
            for (int64_t t = tile - 1; t + 1 < k; t += tile) {
                const unsigned long long* x = &h[(size_t)(t * g + c) * S];
                const unsigned long long ev[6] = {x[5], x[9], x[10], x[11], x[12], x[13]};
                bool ok = true;
                for (int i = 0; i < 6; ++i) ok = ok && ev[i] != 0;
                if (!ok) continue;
                for (int i = 0; i < 5; ++i) bs[i] += double((long long)(ev[i + 1] - ev[i]));
                ++nb;
            }
        if (nb)
            std::fprintf(stderr, "[plnmf] tile boundary (SM cycles): last value->published %.0f, ->past __syncthreads %.0f, "
                         "->phase-3 done %.0f, ->coeff block + sync %.0f, ->first value %.0f\n",
                         bs[0] / nb, bs[1] / nb, bs[2] / nb, bs[3] / nb, bs[4] / nb);
    }
    return panel ? 2 : 1;  // (qpanel_kernel +) pl_update_kernel
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
                       unsigned* counters, double* totals, const WorldXch* xch) {
    if (v <= 0 || k <= 0) return 0;
    exchange_reset(s, k, plan.grid, partials, counters);
    const bool world = xch && xch->world > 1;
    RefWArgs a{v, (int)k, eps, plan.rows_per_cta, w, p, q, norms, partials, counters, totals,
               world ? *xch : WorldXch{}};
    void* args[] = {&a};
    const bool ex = m == Math::exact;
    const void* fn = world ? (ex ? (const void*)ref_update_w_kernel<MathExact, true>
                                 : (const void*)ref_update_w_kernel<MathFused, true>)
                           : (ex ? (const void*)ref_update_w_kernel<MathExact> : (const void*)ref_update_w_kernel<MathFused>);
    if (plan.cooperative)
        PLNMF_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, dim3((unsigned)plan.grid), dim3(kRefWThreads), args, 0, s));
    else  // ranks sharing one GPU: a share of the SMs, co-resident with the other ranks' kernels
        PLNMF_CUDA_CHECK(cudaLaunchKernel(fn, dim3((unsigned)plan.grid), dim3(kRefWThreads), args, 0, s));
    return 1;
}

}  // namespace kern
}  // namespace plnmf

