// The engine: device-resident A (CSR + CSR of A^T, or dense), factors and
// workspace, the iteration loop of proj/src/solver.cpp:53-115, the step API of
// proj/include/plnmf/hals.hpp / tiled.hpp, and the C-ABI over it.
//
// One engine = one device + two streams (the main stream runs the chain; the
// side stream runs the Gram product concurrently with the SpMM that reads the
// same factor).  All host<->device traffic happens at the boundary
// (create / set / get); the loop itself only reads back the 3-double error
// report when the objective is evaluated.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "engine.hpp"

using plnmf::Math;
namespace kern = plnmf::kern;

namespace plnmf {
namespace eng {

void release(plnmf_gpu_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    if (e->s) cudaStreamSynchronize(e->s);
    if (e->s2) cudaStreamSynchronize(e->s2);
    if (e->shard) shard::close_peers(e);
    for (void* ptr : e->allocs) cudaFree(ptr);
    if (e->host_scalars) cudaFreeHost(e->host_scalars);
    for (cudaEvent_t ev : e->events) cudaEventDestroy(ev);
    if (e->fork) cudaEventDestroy(e->fork);
    if (e->join_r) cudaEventDestroy(e->join_r);
    if (e->join_pw) cudaEventDestroy(e->join_pw);
    if (e->err_done) cudaEventDestroy(e->err_done);
    if (e->join) cudaEventDestroy(e->join);
    if (e->s) cudaStreamDestroy(e->s);
    if (e->s2) cudaStreamDestroy(e->s2);
    delete e;
}

void check_engine(const plnmf_gpu_engine* e) {
    if (!e) throw std::invalid_argument("plnmf_gpu: null engine");
    PLNMF_CUDA_CHECK(cudaSetDevice(e->device));
}

void setup_common(plnmf_gpu_engine* e, int device, int64_t rank) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw DeviceError("plnmf_gpu: no CUDA device available (the engine has no CPU fallback)");
    if (device < 0 || device >= ndev) throw std::invalid_argument("plnmf_gpu: device index out of range");
    if (rank < 1) throw std::invalid_argument("SolverConfig: rank must be >= 1");
    e->device = device;
    e->k = rank;
    PLNMF_CUDA_CHECK(cudaSetDevice(device));
    PLNMF_CUDA_CHECK(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, device));
    PLNMF_CUDA_CHECK(cudaStreamCreateWithFlags(&e->s, cudaStreamNonBlocking));
    PLNMF_CUDA_CHECK(cudaStreamCreateWithFlags(&e->s2, cudaStreamNonBlocking));
    PLNMF_CUDA_CHECK(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
    PLNMF_CUDA_CHECK(cudaEventCreateWithFlags(&e->join, cudaEventDisableTiming));
    PLNMF_CUDA_CHECK(cudaEventCreateWithFlags(&e->join_r, cudaEventDisableTiming));
    PLNMF_CUDA_CHECK(cudaEventCreateWithFlags(&e->join_pw, cudaEventDisableTiming));
    PLNMF_CUDA_CHECK(cudaEventCreateWithFlags(&e->err_done, cudaEventDisableTiming));
}

// The workspace (UpdateWorkspace, proj/include/plnmf/workspace.hpp:15-55).  A
// sharded engine's factor buffers are slices of its peer window (set up by
// shard_engine.cu before this call).
void alloc_workspace(plnmf_gpu_engine* e) {
    const int64_t v = e->v, d = e->d, k = e->k;
    if (!e->shard) {
        e->w = dalloc<double>(e, v * k);
        e->w_new = dalloc<double>(e, v * k);
        e->ht = dalloc<double>(e, d * k);
        e->h_new = dalloc<double>(e, d * k);
    }
    e->p = dalloc<double>(e, v * k);
    e->r = dalloc<double>(e, d * k);
    e->r_next = dalloc<double>(e, d * k);
    e->q = dalloc<double>(e, k * k);
    e->sm = dalloc<double>(e, k * k);
    e->norms = dalloc<double>(e, k);
    e->gram_scratch = dalloc<double>(e, kern::gram_scratch_doubles(std::max(v, d), k));
    e->n_partials = kern::exchange_partials_doubles(k, 2 * e->sms);
    e->partials = dalloc<double>(e, e->n_partials);
    e->dot_partials = dalloc<double>(e, kern::kDotBlocks);
    e->dot_partials2 = dalloc<double>(e, kern::kDotBlocks);
    e->scalars = dalloc<double>(e, 8);
    e->staging = dalloc<double>(e, std::max(std::max(v, d), k) * k);  // factors and K x K products
    e->counters = dalloc<unsigned>(e, kern::exchange_counters(k));
    e->totals = dalloc<double>(e, k);
    if (e->sparse) {  // column-blocked SpMM cursors (operands far larger than L2)
        e->cursor_p = dalloc<int64_t>(e, v);
        e->cursor_r = dalloc<int64_t>(e, d);
    }
    PLNMF_CUDA_CHECK(cudaMallocHost(&e->host_scalars, sizeof(double) * 8));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->norms, 0, sizeof(double) * k, e->s));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->p, 0, sizeof(double) * v * k, e->s));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->r, 0, sizeof(double) * d * k, e->s));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->q, 0, sizeof(double) * k * k, e->s));
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->sm, 0, sizeof(double) * k * k, e->s));
    if (!e->shard) {
        PLNMF_CUDA_CHECK(cudaMemsetAsync(e->w, 0, sizeof(double) * v * k, e->s));
        PLNMF_CUDA_CHECK(cudaMemsetAsync(e->ht, 0, sizeof(double) * d * k, e->s));
    }
}

}  // namespace eng
}  // namespace plnmf

namespace {

using plnmf::DeviceError;
using plnmf::dalloc;
using plnmf::guarded;
using namespace plnmf::eng;

// ---- Math::tensor dense products (ozaki.cu) ----------------------------------------------
void ensure_tensor(plnmf_gpu_engine* e) {
    if (e->dig_ap) return;
    const int nt = kern::ozaki_nt(e->k);
    e->dig_ap = dalloc<uint8_t>(e, kern::ozaki_digit_bytes(e->v, e->d, 128));
    e->dig_ar = dalloc<uint8_t>(e, kern::ozaki_digit_bytes(e->d, e->v, 128));
    e->dig_b = dalloc<uint8_t>(e, std::max(kern::ozaki_digit_bytes(e->k, e->d, nt), kern::ozaki_digit_bytes(e->k, e->v, nt)));
    e->sc_ap = dalloc<double>(e, e->v);
    e->sc_ar = dalloc<double>(e, e->d);
    e->sc_b = dalloc<double>(e, e->k);
    e->oz_part = dalloc<double>(e, std::max(kern::ozaki_partial_doubles(e->v, e->k, e->d),
                                            kern::ozaki_partial_doubles(e->d, e->k, e->v)));
    e->launches += kern::ozaki_slice(e->s, e->v, e->d, e->a_dense, e->d, false, 128, e->sc_ap, e->dig_ap);
    e->launches += kern::ozaki_slice(e->s, e->d, e->v, e->a_dense, e->d, true, 128, e->sc_ar, e->dig_ar);
}

// P = A Ht: left = A (V x D), right^T = Ht (D x K) -> right rows = Ht's columns
void tensor_a_ht(plnmf_gpu_engine* e) {
    ensure_tensor(e);
    const int nt = kern::ozaki_nt(e->k);
    e->launches += kern::ozaki_slice(e->s, e->k, e->d, e->ht, e->k, true, nt, e->sc_b, e->dig_b);
    e->launches += kern::ozaki_gemm(e->s, e->v, e->k, e->d, e->dig_ap, e->sc_ap, e->dig_b, e->sc_b, e->oz_part, e->p);
}

// R = A^T W: left = A^T (D x V), right rows = W's columns
void tensor_at_w(plnmf_gpu_engine* e) {
    ensure_tensor(e);
    const int nt = kern::ozaki_nt(e->k);
    e->launches += kern::ozaki_slice(e->s, e->k, e->v, e->w, e->k, true, nt, e->sc_b, e->dig_b);
    e->launches += kern::ozaki_gemm(e->s, e->d, e->k, e->v, e->dig_ar, e->sc_ar, e->dig_b, e->sc_b, e->oz_part, e->r);
}

// Math::tensor workspace of the streaming updates' phase A (kern::tensor_phase_a), or null
void* tensor_phase_a_ws(plnmf_gpu_engine* e, const kern::PhaseBPlan& plan) {
    if (!e->tensor || !plan.streaming) return nullptr;
    const int64_t bytes = kern::tensor_phase_a_bytes(std::max(e->v, e->d), e->k);
    if (bytes > e->tensor_ws_bytes) {
        e->tensor_ws = dalloc<char>(e, bytes);
        e->tensor_ws_bytes = bytes;
    }
    return e->tensor_ws;
}

// ---- products ------------------------------------------------------------------------
// rows of the gathered operand of R = A^T W / P = A Ht (a shard's padded full factor)
int64_t operand_rows_w(const plnmf_gpu_engine* e) { return e->shard ? e->world * e->vcap : e->v; }
int64_t operand_rows_h(const plnmf_gpu_engine* e) { return e->shard ? e->world * e->dcap : e->d; }

// R = A^T W then S = W^T W, one after the other on the engine stream (S is
// skipped when the last error evaluation already left gram(W) in S: same W,
// same deterministic kernel, same bits — the reference recomputes it,
// proj/src/solver.cpp:34 vs proj/src/hals.cpp:31).  With an error evaluation
// every iteration both come from evaluate_error_launch (the Gram first, then
// R ahead on s2 in the registers the Gram leaves, see precompute_w).
void precompute_h(plnmf_gpu_engine* e) {
    if (e->r_valid) {  // R was computed ahead, next to the last error evaluation
        PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s, e->join_r, 0));
        std::swap(e->r, e->r_next);
        e->r_valid = false;
    } else if (e->sparse && !e->shard && !e->s_valid) {  // S first, R beside it (as in precompute_w)
        PLNMF_CUDA_CHECK(cudaEventRecord(e->fork, e->s));
        PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s2, e->fork, 0));
        e->launches += kern::gram(e->s, e->math, e->v, e->k, e->w, e->sm, e->gram_scratch, e->sms);
        e->launches += kern::spmm_csr(e->s2, e->math, e->d, e->trp, e->tci, e->tval, e->w, e->k, e->r, e->nnz_t,
                                      operand_rows_w(e), e->cursor_r, e->spmm_block, true);
        PLNMF_CUDA_CHECK(cudaEventRecord(e->join, e->s2));
        PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s, e->join, 0));
        e->s_valid = true;
        return;
    } else if (e->sparse) {
        const double* w = e->w;
        if (e->shard) {  // every rank's W rows have arrived in this rank's window
            plnmf::shard::wait(e, plnmf::kChanW);
            w = plnmf::shard::w_full(e);
        }
        e->launches += kern::spmm_csr(e->s, e->math, e->d, e->trp, e->tci, e->tval, w, e->k, e->r, e->nnz_t,
                                      operand_rows_w(e), e->cursor_r, e->spmm_block);
    } else if (e->tensor) {
        tensor_at_w(e);
    } else {
        e->launches += kern::dense_at_w(e->s, e->math, e->v, e->d, e->k, e->a_dense, e->w, e->r);
    }
    if (e->s_valid) return;
    e->launches += kern::gram(e->s, e->math, e->v, e->k, e->w, e->sm, e->gram_scratch, e->sms);
    if (e->shard) plnmf::shard::reduce_kxk(e, plnmf::kChanS, e->sm);  // S = sum of the ranks' partials
    e->s_valid = true;
}

// P = A Ht and Q = Ht^T Ht (the Gram scratch is shared with S).
void precompute_w(plnmf_gpu_engine* e) {
    if (e->sparse && !e->shard) {
        // Q first: its one wave of CTAs leaves each SM a quarter of its
        // registers, where the 64-register SpMM runs alongside (P || Q 188 us vs
        // P; Q 232 us at C2).  Launched the other way round, the SpMM's CTAs take
        // every register and the two serialise.
        PLNMF_CUDA_CHECK(cudaEventRecord(e->fork, e->s));
        PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s2, e->fork, 0));
        e->launches += kern::gram(e->s, e->math, e->d, e->k, e->ht, e->q, e->gram_scratch, e->sms);
        e->launches += kern::spmm_csr(e->s2, e->math, e->v, e->rp, e->ci, e->val, e->ht, e->k, e->p, e->nnz,
                                      operand_rows_h(e), e->cursor_p, e->spmm_block, true);
        PLNMF_CUDA_CHECK(cudaEventRecord(e->join, e->s2));
        PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s, e->join, 0));
        return;
    }
    if (e->sparse) {
        const double* ht = e->ht;
        if (e->shard) {
            plnmf::shard::wait(e, plnmf::kChanHt);
            ht = plnmf::shard::ht_full(e);
        }
        e->launches += kern::spmm_csr(e->s, e->math, e->v, e->rp, e->ci, e->val, ht, e->k, e->p, e->nnz,
                                      operand_rows_h(e), e->cursor_p, e->spmm_block);
    } else if (e->tensor) {
        tensor_a_ht(e);
    } else {
        e->launches += kern::dense_a_ht(e->s, e->math, e->v, e->d, e->k, e->a_dense, e->ht, e->p);
    }
    e->launches += kern::gram(e->s, e->math, e->d, e->k, e->ht, e->q, e->gram_scratch, e->sms);
    if (e->shard) plnmf::shard::reduce_kxk(e, plnmf::kChanQ, e->q);
}

void ensure_plans(plnmf_gpu_engine* e, int64_t tile) {
    if (e->plan_tile == tile) return;
    if (e->shard) {
        // the sharded W update is the streaming kernel with the cross-rank norm exchange
        e->plan_w = kern::plan_stream_update(e->v, e->k, tile, true, e->device);
        if (e->sm_cap > 0 && e->sm_cap < e->plan_w.grid) {  // ranks sharing one GPU
            e->plan_w.grid = e->sm_cap;
            e->plan_w.cooperative = false;
            e->plan_w.rows_per_cta = e->v > 0 ? (e->v + e->sm_cap - 1) / e->sm_cap : 1;
        }
    } else {
        e->plan_w = kern::plan_tiled_update(e->v, e->k, tile, true, e->device, e->force_streaming);
    }
    e->plan_h = kern::plan_tiled_update(e->d, e->k, tile, false, e->device, e->force_streaming);
    if (e->plan_w.streaming || e->plan_h.streaming) {  // column-major tile scratch (stream_w_kernel)
        const int64_t xn = std::max(e->plan_w.streaming ? kern::stream_w_scratch_doubles(e->plan_w, tile) : 0,
                                    e->plan_h.streaming ? kern::stream_w_scratch_doubles(e->plan_h, tile) : 0);
        if (xn > e->wscratch_n) {
            e->wscratch = dalloc<double>(e, xn);
            e->wscratch_n = xn;
        }
    }
    const int64_t qn = kern::qpanel_doubles(e->k, tile);
    if (qn > e->qpanel_n) {
        e->qpanel = dalloc<double>(e, qn);
        e->qpanel_n = qn;
    }
    if (kern::exchange_partials_doubles(e->k, e->plan_w.grid) > e->n_partials)
        throw std::logic_error("plnmf_gpu: grid-norm partial buffer too small");
    e->plan_tile = tile;
}

// MAC counts exactly as the reference instruments them
// (hals.cpp:70,105; tiled.cpp:49,62,152-153,172).
uint64_t tiled_macs(int64_t n, int64_t k, int64_t tile, bool w) {
    uint64_t m = w ? (uint64_t)n * k : 0;
    for (int64_t b = 0; b < k; b += tile) {
        const int64_t e = std::min(k, b + tile), width = e - b;
        if (b > 0) m += (uint64_t)n * width * b;         // phase 1 for this tile
        m += (uint64_t)n * width * width;                 // phase 2
        if (w) m += 2ull * n * width;                     // normalisation
        m += (uint64_t)n * width * (k - e);               // phase 3
    }
    return m;
}

void check_tile(const plnmf_config& cfg, int64_t k) {
    if (cfg.tile_size < 1 || cfg.tile_size > k)
        throw std::invalid_argument("iterate: tiled algorithm needs tile_size in [1, rank]");
}

long long* prof_buffer(plnmf_gpu_engine* e, int grid) {
    if (!plnmf::kDebugKnobs || !std::getenv("PLNMF_PROFILE")) return nullptr;
    if (!e->prof || e->prof_n < 24 * (int64_t)grid) {
        e->prof_n = 24 * (int64_t)grid;
        e->prof = dalloc<long long>(e, e->prof_n);
    }
    PLNMF_CUDA_CHECK(cudaMemsetAsync(e->prof, 0, sizeof(long long) * e->prof_n, e->s));
    return e->prof;
}

void prof_report(plnmf_gpu_engine* e, const char* what, int grid) {
    std::vector<long long> h((size_t)24 * grid);
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(h.data(), e->prof, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, e->s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    const char* names[8] = {"prologue", "chain", "grid", "wait", "boundary", "lookahead/pre", "div", "dot"};
    for (int view = 0; view < 3; ++view) {
        std::fprintf(stderr, "[plnmf] %s (%d CTAs) %s view, Mcycles mean/max:", what, grid,
                     view == 0 ? "look-ahead" : view == 1 ? "chain" : "exchange-warp");
        for (int sct = 0; sct < 8; ++sct) {
            double sum = 0, mx = 0;
            for (int c = 0; c < grid; ++c) {
                const double x = (double)h[(size_t)c * 24 + view * 8 + sct];
                sum += x;
                mx = std::max(mx, x);
            }
            std::fprintf(stderr, " %s %.3f/%.3f", names[sct], sum / grid / 1e6, mx / 1e6);
        }
        std::fprintf(stderr, "\n");
    }
}

void update_h(plnmf_gpu_engine* e, const plnmf_config& cfg, plnmf_algorithm alg) {
    bool h_fused = false;
    if (alg == PLNMF_ALGORITHM_TILED) {
        check_tile(cfg, e->k);
        ensure_plans(e, cfg.tile_size);
        long long* prof = prof_buffer(e, e->plan_h.grid);
        // sharded: the Ht all-gather fused into the streaming update (each finished tile to every rank)
        h_fused = e->shard && e->world > 1 && e->plan_h.streaming && kern::stream_fuses_push(e->k, cfg.tile_size);
        plnmf::FusedPush fp;
        if (h_fused) fp = plnmf::shard::fused_push(e, plnmf::kChanHt, e->h_new);
        e->launches += kern::tiled_update(e->s, e->math, e->plan_h, e->d, e->k, cfg.tile_size, cfg.epsilon, false,
                                          e->ht, e->h_new, e->sm, e->r, nullptr, nullptr, nullptr, nullptr, prof,
                                          e->qpanel, e->wscratch, h_fused ? &fp : nullptr,
                                          tensor_phase_a_ws(e, e->plan_h));
        if (prof) prof_report(e, "H update", e->plan_h.grid);
        std::swap(e->ht, e->h_new);  // ht.swap(ws.h_new), tiled.cpp:213
        e->update_macs += tiled_macs(e->d, e->k, cfg.tile_size, false);
    } else {
        e->launches += kern::reference_update_h(e->s, e->math, e->d, e->k, cfg.epsilon, e->ht, e->r, e->sm);
        e->update_macs += (uint64_t)e->d * e->k * e->k;
    }
    if (e->shard && !h_fused) plnmf::shard::push_factor(e, plnmf::kChanHt);  // this rank's new Ht rows to every rank
}

// The W update with the reference's norm order (Math::reference_order): column
// stepped, one launch per piece.  Tiled: phase A (init + phase 1), then per
// column the phase-2 values (the fast path's per-element order), the norm from
// ref_threads chunk partials (tiled.cpp:103-142), the normalisation, and per tile
// phase 3.  Fast-hals: per column the values and one serial norm (hals.cpp:87-103).
void update_w_reference_order(plnmf_gpu_engine* e, const plnmf_config& cfg, plnmf_algorithm alg) {
    if (!e->col_ss) e->col_ss = dalloc<double>(e, 1);
    if (!e->col_partials) e->col_partials = dalloc<double>(e, 512);
    const int64_t v = e->v, k = e->k;
    if (alg == PLNMF_ALGORITHM_TILED) {
        check_tile(cfg, k);
        const int64_t T = cfg.tile_size;
        e->launches += kern::stream_phase_a(e->s, Math::exact, v, k, T, true, e->w, e->q, e->w_new);
        for (int64_t b = 0; b < k; b += T) {
            const int64_t en = std::min(k, b + T);
            for (int64_t t = b; t < en; ++t) {
                e->launches += kern::shard_col_step(e->s, Math::exact, v, k, b, en, t, cfg.epsilon, e->w, e->w_new,
                                                    e->q, e->p, e->col_partials, nullptr);
                e->launches += kern::ordered_ss(e->s, v, k, t, e->ref_threads, e->w_new, e->col_ss);
                e->launches += kern::shard_normalize(e->s, v, k, t, cfg.epsilon, 1, e->col_ss, e->w_new, e->norms);
            }
            e->launches += kern::shard_phase3(e->s, Math::exact, v, k, b, en, e->w_new, e->q);
        }
        std::swap(e->w, e->w_new);  // w.swap(ws.w_new), tiled.cpp:192
        e->update_macs += tiled_macs(v, k, T, true);
    } else {
        for (int64_t kk = 0; kk < k; ++kk) {
            e->launches += kern::ref_w_values(e->s, v, k, kk, cfg.epsilon, e->w, e->p, e->q);
            e->launches += kern::ordered_ss(e->s, v, k, kk, 1, e->w, e->col_ss);
            e->launches += kern::shard_normalize(e->s, v, k, kk, cfg.epsilon, 1, e->col_ss, e->w, e->norms);
        }
        e->update_macs += (uint64_t)v * k * (k + 3);
    }
    e->s_valid = false;
    e->r_valid = false;
}

// The sharded W update: the streaming kernel on the local
// rows, every column's norm exchanged with the other ranks inside the kernel
// (peer.cuh), then the new rows pushed into every rank's window.
void update_w_shard(plnmf_gpu_engine* e, const plnmf_config& cfg, plnmf_algorithm alg) {
    if (alg != PLNMF_ALGORITHM_TILED) {
        // update_w_reference (hals.cpp:77-108) on the local rows, in place, every column's norm
        // exchanged with the other ranks inside the persistent kernel; then the rows to every rank
        if (!e->have_ref_w) {
            e->plan_ref_w = kern::plan_reference_w(e->v, e->device);
            if (e->sm_cap > 0 && e->sm_cap < e->plan_ref_w.grid) {  // ranks sharing one GPU
                e->plan_ref_w.grid = e->sm_cap;
                e->plan_ref_w.cooperative = false;
                e->plan_ref_w.rows_per_cta = e->v > 0 ? (e->v + e->sm_cap - 1) / e->sm_cap : 1;
            }
            e->have_ref_w = true;
        }
        const plnmf::WorldXch x = plnmf::shard::next_exchange(e);
        e->launches += kern::reference_update_w(e->s, e->math, e->plan_ref_w, e->v, e->k, cfg.epsilon, e->w, e->p,
                                                e->q, e->norms, e->partials, e->counters, e->totals, &x);
        e->update_macs += (uint64_t)e->v * e->k * (e->k + 3);
        plnmf::shard::push_factor(e, plnmf::kChanW);
        e->s_valid = false;
        e->r_valid = false;
        return;
    }
    check_tile(cfg, e->k);
    ensure_plans(e, cfg.tile_size);
    const plnmf::WorldXch x = plnmf::shard::next_exchange(e);
    // the W all-gather fused into the update kernel: each finished tile goes to every rank's
    // window while the later tiles compute (a separate push kernel when the kernel cannot)
    const bool fuse = e->world > 1 && kern::stream_fuses_push(e->k, cfg.tile_size);
    plnmf::FusedPush fp;
    if (fuse) fp = plnmf::shard::fused_push(e, plnmf::kChanW, e->w_new);
    e->launches += kern::stream_update(e->s, e->math, e->plan_w, e->v, e->k, cfg.tile_size, cfg.epsilon, true, e->w,
                                       e->w_new, e->q, e->p, e->norms, e->partials, e->counters, &x, e->wscratch,
                                       fuse ? &fp : nullptr);
    std::swap(e->w, e->w_new);  // w.swap(ws.w_new), tiled.cpp:192
    e->update_macs += tiled_macs(e->v, e->k, cfg.tile_size, true);
    if (!fuse) plnmf::shard::push_factor(e, plnmf::kChanW);
    e->s_valid = false;
    e->r_valid = false;
}

void update_w(plnmf_gpu_engine* e, const plnmf_config& cfg, plnmf_algorithm alg) {
    if (e->shard) return update_w_shard(e, cfg, alg);
    if (e->ref_order) return update_w_reference_order(e, cfg, alg);
    if (alg == PLNMF_ALGORITHM_TILED) {
        check_tile(cfg, e->k);
        ensure_plans(e, cfg.tile_size);
        long long* prof = prof_buffer(e, e->plan_w.grid);
        e->launches += kern::tiled_update(e->s, e->math, e->plan_w, e->v, e->k, cfg.tile_size, cfg.epsilon, true,
                                          e->w, e->w_new, e->q, e->p, e->norms, e->partials, e->counters, e->totals,
                                          prof, e->qpanel, e->wscratch, nullptr, tensor_phase_a_ws(e, e->plan_w));
        if (prof) prof_report(e, "W update", e->plan_w.grid);
        std::swap(e->w, e->w_new);  // w.swap(ws.w_new), tiled.cpp:192
        e->update_macs += tiled_macs(e->v, e->k, cfg.tile_size, true);
    } else {
        if (!e->have_ref_w) {
            e->plan_ref_w = kern::plan_reference_w(e->v, e->device);
            if (kern::exchange_partials_doubles(e->k, e->plan_ref_w.grid) > e->n_partials)
                throw std::logic_error("plnmf_gpu: grid-norm partial buffer too small");
            e->have_ref_w = true;
        }
        e->launches += kern::reference_update_w(e->s, e->math, e->plan_ref_w, e->v, e->k, cfg.epsilon, e->w, e->p,
                                                e->q, e->norms, e->partials, e->counters, e->totals);
        e->update_macs += (uint64_t)e->v * e->k * (e->k + 3);
    }
    e->s_valid = false;
    e->r_valid = false;
}

struct ErrorReport {
    double frob = 0, rel = 0;
    bool cancellation = false;
};

ErrorReport direct_error(plnmf_gpu_engine* e) {
    if (e->a2 == 0.0) throw plnmf::DomainError("relative_error_direct: zero input matrix");
    const int64_t np = kern::direct_residual_partials(e->v, e->shard ? e->world * e->dcap : e->d);
    if (np > e->n_direct_partials) {
        e->direct_partials = dalloc<double>(e, np);
        e->n_direct_partials = np;
    }
    if (e->shard) {  // this rank's rows of A - W Ht^T against the gathered Ht, summed over ranks
        plnmf::shard::wait(e, plnmf::kChanHt);
        e->launches += kern::direct_residual(e->s, e->math, e->v, e->world * e->dcap, e->k, e->rp, e->ci, e->val,
                                             nullptr, e->w, plnmf::shard::ht_full(e), e->direct_partials, np,
                                             e->scalars + 5);
        plnmf::shard::reduce_scalar(e, e->scalars + 5);
    } else {
        e->launches += kern::direct_residual(e->s, e->math, e->v, e->d, e->k, e->rp, e->ci, e->val, e->a_dense, e->w,
                                             e->ht, e->direct_partials, np, e->scalars + 5);
    }
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(e->host_scalars + 5, e->scalars + 5, sizeof(double), cudaMemcpyDeviceToHost, e->s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    if (e->shard) plnmf::shard::check_error(e);
    ErrorReport rep;
    rep.frob = e->host_scalars[5];
    rep.rel = std::sqrt(rep.frob / e->a2);
    return rep;
}

// evaluate_error, proj/src/solver.cpp:32-39
// ahead_r: also start the next iteration's R = A^T W on the side stream, beside
// gram(W) and then the error reductions and the host round trip (round 2, the
// 64-register SpMM: e2e 702 -> 704 it/s against R started after the Gram; with
// the earlier 80-register SpMM beside the Gram was slower, 1.87 vs 1.83 ms).
// evaluate_error in two halves: launch (the kernels and the asynchronous readback of the
// 3-double report, completion recorded in `done`) and finish (read it after `done`; the
// direct fallback below 1e-6).  iterate() queues work between the two.
void evaluate_error_launch(plnmf_gpu_engine* e, bool ahead_r, cudaEvent_t done);
ErrorReport evaluate_error_finish(plnmf_gpu_engine* e, cudaEvent_t done);

ErrorReport evaluate_error(plnmf_gpu_engine* e, bool ahead_r = false) {
    cudaEvent_t done = e->err_done;
    evaluate_error_launch(e, ahead_r, done);
    return evaluate_error_finish(e, done);
}

void evaluate_error_launch(plnmf_gpu_engine* e, bool ahead_r, cudaEvent_t done) {
    if (e->a2 == 0.0) throw plnmf::DomainError("relative_error_gram: zero input norm");
    if (!(e->a2 == e->a2)) throw std::invalid_argument("sharded engine: ||A||^2 not set (plnmf_gpu_shard_set_norm_sq)");
    // R ahead: forked before the Gram so that it runs beside it (the Gram's CTAs
    // are dispatched first; the 64-register SpMM takes the registers its wave
    // leaves, as in precompute_w), then beside the error dots
    if (ahead_r) {
        PLNMF_CUDA_CHECK(cudaEventRecord(e->fork, e->s));
        PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s2, e->fork, 0));
    }
    e->launches += kern::gram(e->s, e->math, e->v, e->k, e->w, e->sm, e->gram_scratch, e->sms);
    if (e->shard) plnmf::shard::reduce_kxk(e, plnmf::kChanS, e->sm);
    e->s_valid = true;
    // <P, W> reads only P and W: with R ahead it runs on s2 as well, after the SpMM and beside
    // the Gram, off the engine stream's critical path (its own partials buffer)
    const bool pw_side = ahead_r && !e->ref_order && !e->shard;
    if (ahead_r) {
        e->launches += kern::spmm_csr(e->s2, e->math, e->d, e->trp, e->tci, e->tval, e->w, e->k, e->r_next, e->nnz_t,
                                      operand_rows_w(e), e->cursor_r, e->spmm_block, true);
        PLNMF_CUDA_CHECK(cudaEventRecord(e->join_r, e->s2));
        e->r_valid = true;
        if (pw_side) {
            e->launches += kern::dot(e->s2, e->math, e->v * e->k, e->p, e->w, e->dot_partials2, e->scalars + 0);
            PLNMF_CUDA_CHECK(cudaEventRecord(e->join_pw, e->s2));
        }
    }
    if (e->ref_order) {  // the reference's serial sums (metrics.cpp:104-115)
        e->launches += kern::serial_dot_colmajor(e->s, e->v, e->k, e->p, e->w, e->scalars + 0);
        e->launches += kern::serial_dot_colmajor(e->s, e->k, e->k, e->sm, e->q, e->scalars + 1);
    } else {
        if (!pw_side) {
            e->launches += kern::dot(e->s, e->math, e->v * e->k, e->p, e->w, e->dot_partials, e->scalars + 0);
            if (e->shard) plnmf::shard::reduce_scalar(e, e->scalars + 0);  // <P, W> over all ranks' rows
        }
        e->launches += kern::dot(e->s, e->math, e->k * e->k, e->sm, e->q, e->dot_partials, e->scalars + 1);
        if (pw_side) PLNMF_CUDA_CHECK(cudaStreamWaitEvent(e->s, e->join_pw, 0));
    }
    e->launches += kern::error_finalize(e->s, e->a2, e->scalars + 0, e->scalars + 1, e->scalars + 2);
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(e->host_scalars + 2, e->scalars + 2, 3 * sizeof(double), cudaMemcpyDeviceToHost, e->s));
    PLNMF_CUDA_CHECK(cudaEventRecord(done, e->s));
}

ErrorReport evaluate_error_finish(plnmf_gpu_engine* e, cudaEvent_t done) {
    PLNMF_CUDA_CHECK(cudaEventSynchronize(done));
    if (e->shard) plnmf::shard::check_error(e);
    ErrorReport rep;
    rep.frob = e->host_scalars[2];
    rep.rel = e->host_scalars[3];
    rep.cancellation = e->host_scalars[4] != 0.0;
    if (rep.rel < 1e-6) rep = direct_error(e);
    return rep;
}

void upload_factor(plnmf_gpu_engine* e, const double* host_colmajor, int64_t rows, double* dst) {
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(e->staging, host_colmajor, sizeof(double) * rows * e->k, cudaMemcpyHostToDevice, e->s));
    e->launches += kern::colmajor_to_rowmajor(e->s, rows, e->k, e->staging, dst);
}

void download_rowmajor(plnmf_gpu_engine* e, const double* src, int64_t rows, int64_t cols, double* host_colmajor) {
    e->launches += kern::rowmajor_to_colmajor(e->s, rows, cols, src, e->staging);
    PLNMF_CUDA_CHECK(cudaMemcpyAsync(host_colmajor, e->staging, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, e->s));
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
}

void set_factors(plnmf_gpu_engine* e, const double* w, const double* ht) {
    if (!w || !ht) throw std::invalid_argument("set_factors: null factor");
    upload_factor(e, w, e->v, e->w);
    upload_factor(e, ht, e->d, e->ht);
    if (e->shard) {  // a sharded engine's local rows go to every rank's window
        plnmf::shard::push_factor(e, plnmf::kChanW);
        plnmf::shard::push_factor(e, plnmf::kChanHt);
    }
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    e->s_valid = false;
    e->r_valid = false;
}

void get_factors(plnmf_gpu_engine* e, double* w, double* ht) {
    if (w) download_rowmajor(e, e->w, e->v, e->k, w);
    if (ht) download_rowmajor(e, e->ht, e->d, e->k, ht);
}

cudaEvent_t event_at(plnmf_gpu_engine* e, size_t i) {
    while (e->events.size() <= i) {
        cudaEvent_t ev;
        PLNMF_CUDA_CHECK(cudaEventCreate(&ev));
        e->events.push_back(ev);
    }
    return e->events[i];
}

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    PLNMF_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
}

void add_times(plnmf_phase_times& t, const plnmf_phase_times& o) {
    t.precompute_h += o.precompute_h; t.update_h += o.update_h; t.precompute_w += o.precompute_w;
    t.update_w += o.update_w; t.phase1 += o.phase1; t.phase2 += o.phase2; t.phase3 += o.phase3;
    t.normalize += o.normalize; t.error_eval += o.error_eval;
}

// iterate, proj/src/solver.cpp:53-115.  Phase buckets (PhaseTimes) come from
// CUDA events around each step: precompute_h / precompute_w always; for the
// reference algorithm update_h / update_w (W's normalisation is fused into
// its kernel, so `normalize` stays 0); for the tiled algorithm the whole
// update (init, phases 1-3, normalisation) is one fused look-ahead kernel per
// factor and is reported in phase2 (phase1 / phase3 / normalize stay 0).
// error_eval is host wall time of the evaluation, as in the reference.
void iterate(plnmf_gpu_engine* e, const plnmf_config& cfg, plnmf_algorithm alg, plnmf_trace* trace) {
    plnmf::validate_config(cfg);
    if (cfg.rank != e->k) throw std::invalid_argument("iterate: factor dimensions do not match input and rank");
    if (alg == PLNMF_ALGORITHM_TILED) check_tile(cfg, e->k);
    if (trace && trace->records && trace->capacity < cfg.max_iters)
        throw std::invalid_argument("iterate: trace capacity is smaller than max_iters");
    using clock = std::chrono::steady_clock;
    const uint64_t macs0 = e->update_macs;
    const auto t0 = clock::now();
    auto since = [](clock::time_point a) { return std::chrono::duration<double>(clock::now() - a).count(); };
    plnmf_phase_times totals{};
    const bool tiled = alg == PLNMF_ALGORITHM_TILED;

    // initial error of the given factors (solver.cpp:75-76)
    cudaEvent_t ev[8];
    for (int i = 0; i < 8; ++i) ev[i] = event_at(e, (size_t)i);
    PLNMF_CUDA_CHECK(cudaEventRecord(ev[0], e->s));
    precompute_w(e);
    PLNMF_CUDA_CHECK(cudaEventRecord(ev[1], e->s));
    PLNMF_CUDA_CHECK(cudaEventSynchronize(ev[1]));
    totals.precompute_w += elapsed_s(ev[0], ev[1]);
    auto te = clock::now();
    const double initial = evaluate_error(e).rel;
    totals.error_eval += since(te);
    double prev = initial;
    int64_t n_rec = 0;

    // Speculation (tiled updates, single engine): while the host waits for an error report,
    // the next iteration's precompute_h and update_h are already queued behind it, so the
    // GPU does not idle through the readback and the stop-rule check.  update_h writes the
    // other Ht buffer, so stopping undoes it by swapping the buffers back; everything else it
    // touches (R consumed, S unchanged) stays valid for the final factors.
    const bool can_spec = tiled && !e->shard;
    bool spec = false;  // this iteration's precompute_h + update_h were queued by the previous one
    int set = 0;        // event set of this iteration (the speculative half records into the other)
    auto evs = [&](int st, int i) { return event_at(e, (size_t)(8 + 8 * st + i)); };
    auto queue_h_half = [&](int st) {
        PLNMF_CUDA_CHECK(cudaEventRecord(evs(st, 0), e->s));
        precompute_h(e);
        PLNMF_CUDA_CHECK(cudaEventRecord(evs(st, 1), e->s));
        update_h(e, cfg, alg);
        PLNMF_CUDA_CHECK(cudaEventRecord(evs(st, 2), e->s));
    };
    auto undo_h_half = [&] {
        std::swap(e->ht, e->h_new);  // back to the Ht the final W was computed from
        e->update_macs -= tiled_macs(e->d, e->k, cfg.tile_size, false);
        e->r_valid = false;
    };

    for (int64_t it = 1; it <= cfg.max_iters; ++it) {
        if (!spec) queue_h_half(set);
        spec = false;
        precompute_w(e);
        PLNMF_CUDA_CHECK(cudaEventRecord(evs(set, 3), e->s));
        update_w(e, cfg, alg);
        PLNMF_CUDA_CHECK(cudaEventRecord(evs(set, 4), e->s));
        const bool eval = it % cfg.error_every == 0;
        plnmf_phase_times ph{};
        auto phase_times = [&] {
            ph.precompute_h = elapsed_s(evs(set, 0), evs(set, 1));
            ph.precompute_w = elapsed_s(evs(set, 2), evs(set, 3));
            if (tiled) {
                // one fused look-ahead kernel per update (init, phases 1-3, normalisation)
                ph.phase2 = elapsed_s(evs(set, 1), evs(set, 2)) + elapsed_s(evs(set, 3), evs(set, 4));
            } else {
                ph.update_h = elapsed_s(evs(set, 1), evs(set, 2));
                ph.update_w = elapsed_s(evs(set, 3), evs(set, 4));
            }
        };
        if (eval) {
            // next iteration's R = A^T W computed ahead (unused if the loop stops)
            evaluate_error_launch(e, e->sparse && !e->shard && it < cfg.max_iters, e->err_done);
            PLNMF_CUDA_CHECK(cudaEventRecord(evs(set, 5), e->s));
            if (can_spec && it < cfg.max_iters) {
                queue_h_half(set ^ 1);
                spec = true;
            }
            PLNMF_CUDA_CHECK(cudaEventSynchronize(evs(set, 5)));
            ErrorReport rep;
            {
                ErrorReport r0;
                r0.frob = e->host_scalars[2];
                r0.rel = e->host_scalars[3];
                r0.cancellation = e->host_scalars[4] != 0.0;
                if (e->shard) plnmf::shard::check_error(e);
                if (r0.rel < 1e-6) {  // the direct fallback reads Ht: not with the speculative one
                    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
                    if (spec) undo_h_half();
                    spec = false;
                    r0 = direct_error(e);
                }
                rep = r0;
            }
            phase_times();
            // the evaluation's own time (from the end of the W update to its readback)
            ph.error_eval = elapsed_s(evs(set, 4), evs(set, 5));
            add_times(totals, ph);
            if (!std::isfinite(rep.rel)) {
                if (spec) {
                    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
                    undo_h_half();
                }
                throw plnmf::NonFinite("iterate: objective became non-finite at iteration " + std::to_string(it));
            }
            if (trace && trace->records) {
                plnmf_trace_record& rec = trace->records[n_rec];
                rec.iteration = it;
                rec.rel_error = rep.rel;
                rec.elapsed_s = since(t0);
                rec.phases = ph;
            }
            ++n_rec;
            if (prev > 0.0 && std::fabs(prev - rep.rel) / prev < cfg.rel_tol) {
                prev = rep.rel;
                if (spec) {
                    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
                    undo_h_half();
                    spec = false;
                }
                break;
            }
            prev = rep.rel;
        } else {
            PLNMF_CUDA_CHECK(cudaEventSynchronize(evs(set, 4)));
            phase_times();
            add_times(totals, ph);
        }
        if (spec) set ^= 1;
    }
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    if (trace) {
        trace->initial_error = initial;
        trace->n_records = n_rec;
        trace->totals = totals;
        trace->total_seconds = since(t0);
        trace->update_macs = e->update_macs - macs0;
    }
}

double* product_ptr(plnmf_gpu_engine* e, plnmf_product which, int64_t& rows, int64_t& cols) {
    switch (which) {
        case PLNMF_PRODUCT_P: rows = e->v; cols = e->k; return e->p;
        case PLNMF_PRODUCT_Q: rows = e->k; cols = e->k; return e->q;
        case PLNMF_PRODUCT_R: rows = e->d; cols = e->k; return e->r;
        case PLNMF_PRODUCT_S: rows = e->k; cols = e->k; return e->sm;
        case PLNMF_PRODUCT_COLUMN_NORMS: rows = e->k; cols = 1; return e->norms;
    }
    throw std::invalid_argument("plnmf_gpu: unknown product");
}

void validate_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci, const double* val) {
    // CsrMatrix::validate, proj/src/csr_matrix.cpp:8-28 (same messages)
    if (rows < 0 || cols < 0) throw std::invalid_argument("CsrMatrix: negative dimension");
    if (!rp) throw std::invalid_argument("CsrMatrix: row_ptr length must be rows+1");
    if (rp[0] != 0 || rp[rows] != nnz) throw std::invalid_argument("CsrMatrix: row_ptr must start at 0 and end at nnz");
    if (nnz > 0 && (!ci || !val)) throw std::invalid_argument("CsrMatrix: col_idx and values lengths differ");
    for (int64_t r = 0; r < rows; ++r) {
        if (rp[r] > rp[r + 1]) throw std::invalid_argument("CsrMatrix: row_ptr must be non-decreasing");
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
            if (ci[e] < 0 || ci[e] >= cols) throw std::invalid_argument("CsrMatrix: column index out of range");
            if (e > rp[r] && ci[e] <= ci[e - 1])
                throw std::invalid_argument("CsrMatrix: column indices must be strictly increasing per row");
            if (!std::isfinite(val[e]) || val[e] < 0.0)
                throw std::invalid_argument("CsrMatrix: values must be finite and non-negative");
        }
    }
}

template <class T>
void adopt(plnmf_gpu_engine* e, T* ptr, int64_t n) {
    e->allocs.push_back(ptr);
    e->bytes += (int64_t)(sizeof(T) * (size_t)std::max<int64_t>(1, n));
}

// A sparse engine on a CSR that already lives on the device (device generator,
// Matrix Market assembly): takes ownership of the arrays, sums ||A||^2 serially
// in the reference's order (input_matrix.cpp:15-20) from the device values
// (streamed to the host in chunks; also InputMatrix's finiteness check), builds
// A^T on the device and the workspace.
void finish_device_csr(plnmf_gpu_engine* e, int64_t rows, int64_t cols, int64_t nnz, int64_t* rp, int32_t* ci,
                       double* val) {
    adopt(e, rp, rows + 1);
    adopt(e, ci, nnz);
    adopt(e, val, nnz);
    if (cols > INT32_MAX || rows > INT32_MAX)
        throw std::invalid_argument("plnmf_gpu_create: dimensions exceed int32 column indexing");
    e->v = rows;
    e->d = cols;
    e->nnz = nnz;
    e->nnz_t = nnz;
    e->sparse = true;
    e->rp = rp;
    e->ci = ci;
    e->val = val;
    {
        constexpr int64_t kChunk = 1 << 23;
        double* host = nullptr;
        PLNMF_CUDA_CHECK(cudaMallocHost(&host, sizeof(double) * (size_t)std::min<int64_t>(kChunk, std::max<int64_t>(1, nnz))));
        double n2 = 0.0;
        bool finite = true;
        try {
            for (int64_t b = 0; b < nnz; b += kChunk) {
                const int64_t m = std::min(kChunk, nnz - b);
                PLNMF_CUDA_CHECK(cudaMemcpyAsync(host, val + b, sizeof(double) * m, cudaMemcpyDeviceToHost, e->s));
                PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
                for (int64_t i = 0; i < m; ++i) {
                    finite = finite && std::isfinite(host[i]) && host[i] >= 0.0;
                    n2 += host[i] * host[i];
                }
            }
        } catch (...) {
            cudaFreeHost(host);
            throw;
        }
        PLNMF_CUDA_CHECK(cudaFreeHost(host));
        if (!finite) throw std::invalid_argument("CsrMatrix: values must be finite and non-negative");
        e->a2 = n2;
    }
    e->trp = dalloc<int64_t>(e, cols + 1);
    e->tci = dalloc<int32_t>(e, nnz);
    e->tval = dalloc<double>(e, nnz);
    e->launches += kern::csr_transpose(e->s, rows, cols, nnz, e->rp, e->ci, e->val, e->trp, e->tci, e->tval);
    alloc_workspace(e);
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
}

}  // namespace

// =============================================================================== C-ABI
extern "C" {

int32_t plnmf_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

plnmf_status plnmf_gpu_device_name(int32_t device, char* buf, int32_t len) {
    return guarded([&] {
        if (!buf || len < 1) throw std::invalid_argument("plnmf_gpu_device_name: bad buffer");
        cudaDeviceProp prop{};
        PLNMF_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        std::snprintf(buf, (size_t)len, "%s", prop.name);
    });
}

plnmf_status plnmf_gpu_create_csr(int32_t device, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                                  const int64_t* col_idx, const double* values, int64_t rank,
                                  plnmf_gpu_engine** out) {
    plnmf_gpu_engine* e = nullptr;
    const plnmf_status st = guarded([&] {
        if (!out) throw std::invalid_argument("plnmf_gpu_create_csr: null output");
        validate_csr(rows, cols, nnz, row_ptr, col_idx, values);
        if (cols > INT32_MAX || rows > INT32_MAX)
            throw std::invalid_argument("plnmf_gpu_create_csr: dimensions exceed int32 column indexing");
        e = new plnmf_gpu_engine();
        setup_common(e, device, rank);
        e->v = rows;
        e->d = cols;
        e->nnz = nnz;
        e->nnz_t = nnz;
        e->sparse = true;
        double n2 = 0.0;  // InputMatrix ctor, proj/src/input_matrix.cpp:15-20 (serial)
        for (int64_t i = 0; i < nnz; ++i) n2 += values[i] * values[i];
        e->a2 = n2;
        std::vector<int32_t> ci32(nnz > 0 ? nnz : 1);
        for (int64_t i = 0; i < nnz; ++i) ci32[i] = (int32_t)col_idx[i];
        e->rp = dalloc<int64_t>(e, rows + 1);
        e->ci = dalloc<int32_t>(e, nnz);
        e->val = dalloc<double>(e, nnz);
        e->trp = dalloc<int64_t>(e, cols + 1);
        e->tci = dalloc<int32_t>(e, nnz);
        e->tval = dalloc<double>(e, nnz);
        PLNMF_CUDA_CHECK(cudaMemcpy(e->rp, row_ptr, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice));
        if (nnz > 0) {
            PLNMF_CUDA_CHECK(cudaMemcpy(e->ci, ci32.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
            PLNMF_CUDA_CHECK(cudaMemcpy(e->val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice));
        }
        e->launches += kern::csr_transpose(e->s, rows, cols, nnz, e->rp, e->ci, e->val, e->trp, e->tci, e->tval);
        alloc_workspace(e);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        *out = e;
    });
    if (st != PLNMF_OK) release(e);
    return st;
}

plnmf_status plnmf_gpu_create_dense(int32_t device, int64_t rows, int64_t cols, const double* a, int64_t rank,
                                    plnmf_gpu_engine** out) {
    plnmf_gpu_engine* e = nullptr;
    const plnmf_status st = guarded([&] {
        if (!out || !a) throw std::invalid_argument("plnmf_gpu_create_dense: null argument");
        if (rows < 0 || cols < 0) throw std::invalid_argument("DenseMatrix: negative dimension");
        e = new plnmf_gpu_engine();
        setup_common(e, device, rank);
        e->v = rows;
        e->d = cols;
        e->sparse = false;
        double n2 = 0.0;  // proj/src/input_matrix.cpp:5-13
        int64_t nz = 0;
        for (int64_t i = 0; i < rows * cols; ++i) {
            n2 += a[i] * a[i];
            if (a[i] != 0.0) ++nz;
        }
        e->a2 = n2;
        e->nnz = nz;
        e->a_dense = dalloc<double>(e, rows * cols);
        double* tmp = nullptr;
        PLNMF_CUDA_CHECK(cudaMalloc(&tmp, sizeof(double) * (size_t)std::max<int64_t>(1, rows * cols)));
        PLNMF_CUDA_CHECK(cudaMemcpy(tmp, a, sizeof(double) * rows * cols, cudaMemcpyHostToDevice));
        e->launches += kern::colmajor_to_rowmajor(e->s, rows, cols, tmp, e->a_dense);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        PLNMF_CUDA_CHECK(cudaFree(tmp));
        alloc_workspace(e);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        *out = e;
    });
    if (st != PLNMF_OK) release(e);
    return st;
}

plnmf_status plnmf_gpu_create_synthetic(int32_t device, int64_t rows, int64_t cols, double density, uint64_t seed,
                                        int64_t rank, plnmf_gpu_engine** out) {
    plnmf_gpu_engine* e = nullptr;
    const plnmf_status st = guarded([&] {
        if (!out) throw std::invalid_argument("plnmf_gpu_create_synthetic: null output");
        e = new plnmf_gpu_engine();
        setup_common(e, device, rank);
        int64_t* rp = nullptr;
        int32_t* ci = nullptr;
        double* val = nullptr;
        const int64_t nnz = kern::synth_csr_device(e->s, rows, cols, density, seed, &rp, &ci, &val);
        e->launches += 2;
        finish_device_csr(e, rows, cols, nnz, rp, ci, val);
        *out = e;
    });
    if (st != PLNMF_OK) release(e);
    return st;
}

plnmf_status plnmf_gpu_create_mm(int32_t device, const plnmf_mm* m, int64_t rank, plnmf_gpu_engine** out) {
    if (m && !plnmf::mm_coordinate(m)) {  // "array real general": a dense InputMatrix
        if (!out) return guarded([] { throw std::invalid_argument("plnmf_gpu_create_mm: null output"); });
        return plnmf_gpu_create_dense(device, plnmf::mm_nrows(m), plnmf::mm_ncols(m), plnmf::mm_values(m).data(),
                                      rank, out);
    }
    plnmf_gpu_engine* e = nullptr;
    const plnmf_status st = guarded([&] {
        if (!m || !out) throw std::invalid_argument("plnmf_gpu_create_mm: null argument");
        e = new plnmf_gpu_engine();
        setup_common(e, device, rank);
        int64_t* rp = nullptr;
        int32_t* ci = nullptr;
        double* val = nullptr;
        const auto& v = plnmf::mm_values(m);
        const int64_t nnz = kern::coo_to_csr_device(e->s, plnmf::mm_nrows(m), plnmf::mm_ncols(m), (int64_t)v.size(),
                                                    plnmf::mm_rows(m).data(), plnmf::mm_cols(m).data(), v.data(),
                                                    &rp, &ci, &val);
        e->launches += 5;
        finish_device_csr(e, plnmf::mm_nrows(m), plnmf::mm_ncols(m), nnz, rp, ci, val);
        *out = e;
    });
    if (st != PLNMF_OK) release(e);
    return st;
}

plnmf_status plnmf_gpu_get_csr(plnmf_gpu_engine* e, int64_t* row_ptr, int64_t* col_idx, double* values) {
    return guarded([&] {
        check_engine(e);
        if (!e->sparse || e->shard) throw std::invalid_argument("plnmf_gpu_get_csr: not a sparse single engine");
        if (row_ptr)
            PLNMF_CUDA_CHECK(cudaMemcpyAsync(row_ptr, e->rp, sizeof(int64_t) * (e->v + 1), cudaMemcpyDeviceToHost, e->s));
        std::vector<int32_t> ci32(col_idx ? std::max<int64_t>(1, e->nnz) : 0);
        if (col_idx && e->nnz > 0)
            PLNMF_CUDA_CHECK(cudaMemcpyAsync(ci32.data(), e->ci, sizeof(int32_t) * e->nnz, cudaMemcpyDeviceToHost, e->s));
        if (values && e->nnz > 0)
            PLNMF_CUDA_CHECK(cudaMemcpyAsync(values, e->val, sizeof(double) * e->nnz, cudaMemcpyDeviceToHost, e->s));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        if (col_idx)
            for (int64_t i = 0; i < e->nnz; ++i) col_idx[i] = ci32[i];
    });
}

plnmf_status plnmf_gpu_get_csr_rows(plnmf_gpu_engine* e, int32_t transposed, const int64_t* rows, int64_t n,
                                    int64_t* row_ptr_out, int64_t* col_idx, double* values) {
    return guarded([&] {
        check_engine(e);
        if (!e->sparse) throw std::invalid_argument("plnmf_gpu_get_csr_rows: not a sparse engine");
        const int64_t* rp = transposed ? e->trp : e->rp;
        const int32_t* ci = transposed ? e->tci : e->ci;
        const double* val = transposed ? e->tval : e->val;
        const int64_t nrows = transposed ? e->d : e->v;
        if (n < 0 || (n > 0 && (!rows || !row_ptr_out))) throw std::invalid_argument("plnmf_gpu_get_csr_rows: bad argument");
        row_ptr_out[0] = 0;
        std::vector<int64_t> lo(n), hi(n);
        for (int64_t i = 0; i < n; ++i) {
            if (rows[i] < 0 || rows[i] >= nrows) throw std::invalid_argument("plnmf_gpu_get_csr_rows: row out of range");
            int64_t b[2];
            PLNMF_CUDA_CHECK(cudaMemcpy(b, rp + rows[i], sizeof(b), cudaMemcpyDeviceToHost));
            lo[i] = b[0];
            hi[i] = b[1];
            row_ptr_out[i + 1] = row_ptr_out[i] + (b[1] - b[0]);
        }
        if (!col_idx && !values) return;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t cnt = hi[i] - lo[i];
            if (cnt == 0) continue;
            if (col_idx) {
                std::vector<int32_t> c32(cnt);
                PLNMF_CUDA_CHECK(cudaMemcpy(c32.data(), ci + lo[i], sizeof(int32_t) * cnt, cudaMemcpyDeviceToHost));
                for (int64_t j = 0; j < cnt; ++j) col_idx[row_ptr_out[i] + j] = c32[j];
            }
            if (values)
                PLNMF_CUDA_CHECK(cudaMemcpy(values + row_ptr_out[i], val + lo[i], sizeof(double) * cnt,
                                            cudaMemcpyDeviceToHost));
        }
    });
}

plnmf_status plnmf_gpu_get_rows(plnmf_gpu_engine* e, plnmf_buffer which, const int64_t* rows, int64_t n,
                                double* out) {
    return guarded([&] {
        check_engine(e);
        if (n < 0 || (n > 0 && (!rows || !out))) throw std::invalid_argument("plnmf_gpu_get_rows: bad argument");
        const double* src = nullptr;
        int64_t nr = 0;
        switch (which) {
            case PLNMF_BUF_W: src = e->w; nr = e->v; break;
            case PLNMF_BUF_HT: src = e->ht; nr = e->d; break;
            case PLNMF_BUF_P: src = e->p; nr = e->v; break;
            case PLNMF_BUF_R: src = e->r; nr = e->d; break;
            default: throw std::invalid_argument("plnmf_gpu_get_rows: W, HT, P or R expected");
        }
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        for (int64_t i = 0; i < n; ++i) {
            if (rows[i] < 0 || rows[i] >= nr) throw std::invalid_argument("plnmf_gpu_get_rows: row out of range");
            PLNMF_CUDA_CHECK(cudaMemcpyAsync(out + i * e->k, src + rows[i] * e->k, sizeof(double) * e->k,
                                             cudaMemcpyDeviceToHost, e->s));
        }
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    });
}

plnmf_status plnmf_gpu_destroy(plnmf_gpu_engine* e) {
    return guarded([&] { release(e); });
}

plnmf_status plnmf_gpu_input_info(const plnmf_gpu_engine* e, int64_t* rows, int64_t* cols, int64_t* nnz, double* norm_sq) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("plnmf_gpu: null engine");
        if (rows) *rows = e->v;
        if (cols) *cols = e->d;
        if (nnz) *nnz = e->nnz;
        if (norm_sq) *norm_sq = e->a2;
    });
}

plnmf_status plnmf_gpu_set_math(plnmf_gpu_engine* e, plnmf_math math) {
    return guarded([&] {
        check_engine(e);
        if (math != PLNMF_MATH_EXACT && math != PLNMF_MATH_FUSED && math != PLNMF_MATH_REFERENCE_ORDER &&
            math != PLNMF_MATH_TENSOR)
            throw std::invalid_argument("plnmf_gpu_set_math: unknown mode");
        if (e->shard && (math == PLNMF_MATH_REFERENCE_ORDER || math == PLNMF_MATH_TENSOR))
            throw std::invalid_argument("plnmf_gpu_set_math: a sharded engine runs Math::exact or Math::fused");
        e->math = math == PLNMF_MATH_FUSED ? Math::fused : Math::exact;
        e->ref_order = math == PLNMF_MATH_REFERENCE_ORDER;
        // Math::tensor: the dense-A products (dense inputs) and phase A of streaming tiled
        // updates (any input) on the tensor cores
        e->tensor = math == PLNMF_MATH_TENSOR;
        e->s_valid = false;
        e->r_valid = false;
    });
}

plnmf_status plnmf_gpu_force_streaming(plnmf_gpu_engine* e, int32_t on) {
    return guarded([&] {
        check_engine(e);
        e->force_streaming = on != 0;
        e->plan_tile = -1;  // re-plan on the next tiled update
    });
}

plnmf_status plnmf_gpu_force_spmm_blocks(plnmf_gpu_engine* e, int64_t operand_rows) {
    return guarded([&] {
        check_engine(e);
        if (operand_rows < 0) throw std::invalid_argument("plnmf_gpu_force_spmm_blocks: negative block");
        e->spmm_block = operand_rows;
    });
}

plnmf_status plnmf_gpu_set_reference_threads(plnmf_gpu_engine* e, int32_t nthreads) {
    return guarded([&] {
        check_engine(e);
        if (nthreads < 1 || nthreads > 1024)
            throw std::invalid_argument("plnmf_gpu_set_reference_threads: thread count must be in [1, 1024]");
        e->ref_threads = nthreads;
    });
}

plnmf_status plnmf_gpu_set_factors(plnmf_gpu_engine* e, const double* w, const double* ht) {
    return guarded([&] { check_engine(e); set_factors(e, w, ht); });
}

plnmf_status plnmf_gpu_get_factors(plnmf_gpu_engine* e, double* w, double* ht) {
    return guarded([&] { check_engine(e); get_factors(e, w, ht); });
}

plnmf_status plnmf_gpu_init_factors(plnmf_gpu_engine* e, const plnmf_config* cfg) {
    return guarded([&] {
        check_engine(e);
        if (!cfg) throw std::invalid_argument("plnmf_gpu_init_factors: null config");
        if (cfg->rank != e->k) throw std::invalid_argument("init_factors: rank does not match the engine");
        if (e->shard) {  // the whole factors' stream (solver.cpp:43-51), this rank's rows of it
            std::vector<double> w((size_t)(e->vfull * e->k)), ht((size_t)(e->dfull * e->k));
            plnmf::init_factors_host(e->vfull, e->dfull, *cfg, w.data(), ht.data());
            std::vector<double> wl((size_t)(e->v * e->k)), hl((size_t)(e->d * e->k));
            for (int64_t j = 0; j < e->k; ++j) {
                std::memcpy(&wl[(size_t)(j * e->v)], &w[(size_t)(j * e->vfull + e->v_lo)], sizeof(double) * e->v);
                std::memcpy(&hl[(size_t)(j * e->d)], &ht[(size_t)(j * e->dfull + e->d_lo)], sizeof(double) * e->d);
            }
            set_factors(e, wl.data(), hl.data());
            return;
        }
        std::vector<double> w((size_t)(e->v * e->k)), ht((size_t)(e->d * e->k));
        plnmf::init_factors_host(e->v, e->d, *cfg, w.data(), ht.data());
        set_factors(e, w.data(), ht.data());
    });
}

plnmf_status plnmf_gpu_iterate(plnmf_gpu_engine* e, const plnmf_config* cfg, plnmf_algorithm alg, plnmf_trace* trace) {
    return guarded([&] {
        check_engine(e);
        if (!cfg) throw std::invalid_argument("plnmf_gpu_iterate: null config");
        iterate(e, *cfg, alg, trace);
    });
}

plnmf_status plnmf_gpu_iterate_host(plnmf_gpu_engine* e, const plnmf_config* cfg, plnmf_algorithm alg, double* w,
                                    double* ht, plnmf_trace* trace) {
    return guarded([&] {
        check_engine(e);
        if (!cfg) throw std::invalid_argument("plnmf_gpu_iterate_host: null config");
        set_factors(e, w, ht);
        iterate(e, *cfg, alg, trace);
        get_factors(e, w, ht);
    });
}

// step calls finish on the host; a sharded rank also reports a peer that never arrived
static void finish_step(plnmf_gpu_engine* e) {
    PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
    if (e->shard) plnmf::shard::check_error(e);
}

plnmf_status plnmf_gpu_precompute_h_products(plnmf_gpu_engine* e) {
    return guarded([&] { check_engine(e); precompute_h(e); finish_step(e); });
}

plnmf_status plnmf_gpu_precompute_w_products(plnmf_gpu_engine* e) {
    return guarded([&] { check_engine(e); precompute_w(e); finish_step(e); });
}

plnmf_status plnmf_gpu_update_h(plnmf_gpu_engine* e, const plnmf_config* cfg, plnmf_algorithm alg) {
    return guarded([&] {
        check_engine(e);
        if (!cfg) throw std::invalid_argument("plnmf_gpu_update_h: null config");
        update_h(e, *cfg, alg);
        finish_step(e);
    });
}

plnmf_status plnmf_gpu_update_w(plnmf_gpu_engine* e, const plnmf_config* cfg, plnmf_algorithm alg) {
    return guarded([&] {
        check_engine(e);
        if (!cfg) throw std::invalid_argument("plnmf_gpu_update_w: null config");
        update_w(e, *cfg, alg);
        finish_step(e);
    });
}

plnmf_status plnmf_gpu_evaluate_error(plnmf_gpu_engine* e, double* out3) {
    return guarded([&] {
        check_engine(e);
        const ErrorReport r = evaluate_error(e);
        if (out3) {
            out3[0] = r.frob;
            out3[1] = r.rel;
            out3[2] = r.cancellation ? 1.0 : 0.0;
        }
    });
}

plnmf_status plnmf_gpu_relative_error_direct(plnmf_gpu_engine* e, double* out2) {
    return guarded([&] {
        check_engine(e);
        const ErrorReport r = direct_error(e);
        if (out2) {
            out2[0] = r.frob;
            out2[1] = r.rel;
        }
    });
}

plnmf_status plnmf_gpu_get_product(plnmf_gpu_engine* e, plnmf_product which, double* out) {
    return guarded([&] {
        check_engine(e);
        if (!out) throw std::invalid_argument("plnmf_gpu_get_product: null output");
        int64_t rows, cols;
        double* src = product_ptr(e, which, rows, cols);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        if (cols == 1) {
            PLNMF_CUDA_CHECK(cudaMemcpy(out, src, sizeof(double) * rows, cudaMemcpyDeviceToHost));
        } else {
            download_rowmajor(e, src, rows, cols, out);
        }
    });
}

plnmf_status plnmf_gpu_set_product(plnmf_gpu_engine* e, plnmf_product which, const double* in) {
    return guarded([&] {
        check_engine(e);
        if (!in) throw std::invalid_argument("plnmf_gpu_set_product: null input");
        int64_t rows, cols;
        double* dst = product_ptr(e, which, rows, cols);
        if (cols == 1) {  // on the engine stream: a pending normalisation must not overwrite it
            PLNMF_CUDA_CHECK(cudaMemcpyAsync(dst, in, sizeof(double) * rows, cudaMemcpyHostToDevice, e->s));
            PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        } else {
            PLNMF_CUDA_CHECK(cudaMemcpyAsync(e->staging, in, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, e->s));
            e->launches += kern::colmajor_to_rowmajor(e->s, rows, cols, e->staging, dst);
            PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        }
        if (which == PLNMF_PRODUCT_S) e->s_valid = false;
    e->r_valid = false;
    });
}

// One FAST-HALS iteration in the reference's order (solver.cpp:79-92).  (A
// CUDA-graph replay of whole iterations was measured slower, 1.73 vs 1.65 ms,
// and removed: the GPU is never idle between these launches.)
void one_iteration(plnmf_gpu_engine* e, const plnmf_config& cfg, plnmf_algorithm alg) {
    precompute_h(e);
    update_h(e, cfg, alg);
    precompute_w(e);
    update_w(e, cfg, alg);
}

plnmf_status plnmf_gpu_run_iterations(plnmf_gpu_engine* e, const plnmf_config* cfg, plnmf_algorithm alg, int64_t n,
                                      double* device_ms) {
    return guarded([&] {
        check_engine(e);
        if (!cfg) throw std::invalid_argument("plnmf_gpu_run_iterations: null config");
        plnmf::validate_config(*cfg);
        if (cfg->rank != e->k) throw std::invalid_argument("iterate: factor dimensions do not match input and rank");
        cudaEvent_t a = event_at(e, 0), b = event_at(e, 1);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        // per-phase events on the engine stream (the stream every step's kernels are
        // launched on; the Gram side stream joins it inside precompute_*), 5 per iteration
        for (int64_t i = 0; i < 5 * n + 2; ++i) event_at(e, (size_t)i);
        PLNMF_CUDA_CHECK(cudaEventRecord(a, e->s));
        for (int64_t i = 0; i < n; ++i) {
            cudaEvent_t* ev = &e->events[(size_t)(2 + 5 * i)];
            PLNMF_CUDA_CHECK(cudaEventRecord(ev[0], e->s));
            precompute_h(e);
            PLNMF_CUDA_CHECK(cudaEventRecord(ev[1], e->s));
            update_h(e, *cfg, alg);
            PLNMF_CUDA_CHECK(cudaEventRecord(ev[2], e->s));
            precompute_w(e);
            PLNMF_CUDA_CHECK(cudaEventRecord(ev[3], e->s));
            update_w(e, *cfg, alg);
            PLNMF_CUDA_CHECK(cudaEventRecord(ev[4], e->s));
        }
        PLNMF_CUDA_CHECK(cudaEventRecord(b, e->s));
        PLNMF_CUDA_CHECK(cudaEventSynchronize(b));
        if (e->shard) plnmf::shard::check_error(e);
        if (device_ms) *device_ms = elapsed_s(a, b) * 1e3;
        double ph[4] = {0, 0, 0, 0};
        for (int64_t i = 0; i < n; ++i) {
            cudaEvent_t* ev = &e->events[(size_t)(2 + 5 * i)];
            for (int j = 0; j < 4; ++j) ph[j] += elapsed_s(ev[j], ev[j + 1]) * 1e3;
        }
        for (int j = 0; j < 4; ++j) e->last_phase_ms[j] = ph[j];
    });
}

plnmf_status plnmf_gpu_phase_ms(const plnmf_gpu_engine* e, double* out4) {
    return guarded([&] {
        if (!e || !out4) throw std::invalid_argument("plnmf_gpu_phase_ms: null argument");
        for (int j = 0; j < 4; ++j) out4[j] = e->last_phase_ms[j];
    });
}

plnmf_status plnmf_gpu_time_kernel(plnmf_gpu_engine* e, const plnmf_config* cfg, int32_t which, int32_t reps,
                                   double* avg_ms) {
    return guarded([&] {
        check_engine(e);
        if (!cfg || reps < 1) throw std::invalid_argument("plnmf_gpu_time_kernel: bad argument");
        if (e->shard) throw std::invalid_argument("plnmf_gpu_time_kernel: not available on a shard engine");
        cudaEvent_t a = event_at(e, 0), b = event_at(e, 1);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s2));
        auto once = [&] {
            switch (which) {
                case 0:
                    if (e->sparse) e->launches += kern::spmm_csr(e->s, e->math, e->v, e->rp, e->ci, e->val, e->ht, e->k, e->p, e->nnz, e->d, e->cursor_p, e->spmm_block);
                    else if (e->tensor) tensor_a_ht(e);
                    else e->launches += kern::dense_a_ht(e->s, e->math, e->v, e->d, e->k, e->a_dense, e->ht, e->p);
                    break;
                case 1:
                    if (e->sparse) e->launches += kern::spmm_csr(e->s, e->math, e->d, e->trp, e->tci, e->tval, e->w, e->k, e->r, e->nnz_t, e->v, e->cursor_r, e->spmm_block);
                    else if (e->tensor) tensor_at_w(e);
                    else e->launches += kern::dense_at_w(e->s, e->math, e->v, e->d, e->k, e->a_dense, e->w, e->r);
                    break;
                case 2: e->launches += kern::gram(e->s, e->math, e->v, e->k, e->w, e->sm, e->gram_scratch, e->sms); break;
                case 5: e->launches += kern::gram(e->s, e->math, e->d, e->k, e->ht, e->q, e->gram_scratch, e->sms); break;
                case 6: precompute_w(e); break;  // Q = gram(Ht) || P = A Ht on two streams
                case 8:  // S = gram(W) || R = A^T W on two streams
                    e->s_valid = false;
                    e->r_valid = false;
                    precompute_h(e);
                    break;
                case 7:  // H-side phase A (init + phase 1 of every tile) into the staging buffer
                    e->launches += kern::stream_phase_a(e->s, e->math, e->d, e->k, cfg->tile_size, false, e->ht, e->sm,
                                                        e->staging);
                    break;
                case 3:  // successive W updates against the same P, Q (mutates W)
                    update_w(e, *cfg, cfg->tile_size > 0 ? PLNMF_ALGORITHM_TILED : PLNMF_ALGORITHM_REFERENCE);
                    break;
                case 4: update_h(e, *cfg, cfg->tile_size > 0 ? PLNMF_ALGORITHM_TILED : PLNMF_ALGORITHM_REFERENCE); break;
                default: throw std::invalid_argument("plnmf_gpu_time_kernel: unknown kernel family");
            }
        };
        once();  // warm
        PLNMF_CUDA_CHECK(cudaEventRecord(a, e->s));
        for (int i = 0; i < reps; ++i) once();
        PLNMF_CUDA_CHECK(cudaEventRecord(b, e->s));
        PLNMF_CUDA_CHECK(cudaEventSynchronize(b));
        if (avg_ms) *avg_ms = elapsed_s(a, b) * 1e3 / reps;
        e->s_valid = false;
    e->r_valid = false;
    });
}

// GPU tile selection: the reference picks T from a cache
// model (best_integer_tile, proj/src/cost_model.cpp:131-142); on the GPU the
// update kernels' cost is set by their shared-memory staging and register-tile
// instantiations (T <= 16 / <= 32), not by a 35 MB cache, so the candidates are
// measured: for each T, one warm-up and one timed H + W tiled update from the
// current factors (products recomputed per T), factors restored afterwards.
plnmf_status plnmf_gpu_best_integer_tile(plnmf_gpu_engine* e, const plnmf_config* cfg, const int32_t* candidates,
                                         int32_t n, int32_t* best, double* update_ms) {
    return guarded([&] {
        check_engine(e);
        if (!cfg || !best || n < 0 || (n > 0 && !candidates))
            throw std::invalid_argument("best_integer_tile: bad argument");
        if (e->shard) throw std::invalid_argument("best_integer_tile: not available on a shard engine");
        plnmf::validate_config(*cfg);
        if (cfg->rank != e->k) throw std::invalid_argument("iterate: factor dimensions do not match input and rank");
        std::vector<int32_t> cand;
        if (n > 0) {
            cand.assign(candidates, candidates + n);
        } else {
            for (int32_t t : {1, 2, 4, 8, 12, 16, 20, 24, 32})
                if (t <= e->k) cand.push_back(t);
        }
        for (int32_t t : cand)
            if (t < 1 || t > e->k) throw std::invalid_argument("best_integer_tile: tile size must be in [1, K]");
        // Snapshot of everything a trial update changes — factors, the workspace
        // products P, Q, R, S, the column norms — restored afterwards together
        // with the MAC counter, so the call leaves the engine as it found it.
        const size_t wb = sizeof(double) * (size_t)(e->v * e->k), hb = sizeof(double) * (size_t)(e->d * e->k);
        const size_t kb = sizeof(double) * (size_t)(e->k * e->k), nb = sizeof(double) * (size_t)e->k;
        struct Snap { double** live; size_t bytes; double* copy; };
        Snap snaps[] = {{&e->w, wb, nullptr}, {&e->ht, hb, nullptr}, {&e->p, wb, nullptr}, {&e->r, hb, nullptr},
                        {&e->q, kb, nullptr}, {&e->sm, kb, nullptr}, {&e->norms, nb, nullptr}};
        const uint64_t macs0 = e->update_macs;
        auto free_snaps = [&] {
            for (Snap& sn : snaps) if (sn.copy) cudaFree(sn.copy);
        };
        auto restore = [&](bool products) {
            for (Snap& sn : snaps) {
                if (!products && sn.live != &e->w && sn.live != &e->ht) continue;
                PLNMF_CUDA_CHECK(cudaMemcpyAsync(*sn.live, sn.copy, sn.bytes, cudaMemcpyDeviceToDevice, e->s));
            }
            e->s_valid = false;
            e->r_valid = false;
        };
        try {
            PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s2));
            for (Snap& sn : snaps) {
                PLNMF_CUDA_CHECK(cudaMalloc(&sn.copy, sn.bytes));
                PLNMF_CUDA_CHECK(cudaMemcpyAsync(sn.copy, *sn.live, sn.bytes, cudaMemcpyDeviceToDevice, e->s));
            }
            cudaEvent_t a0 = event_at(e, 0), a1 = event_at(e, 1), b0 = event_at(e, 2), b1 = event_at(e, 3);
            double best_ms = 0.0;
            for (size_t i = 0; i < cand.size(); ++i) {
                plnmf_config c = *cfg;
                c.tile_size = cand[i];
                double ms = 0.0;
                for (int rep = 0; rep < 2; ++rep) {  // warm-up (plans, coefficient panels), then timed
                    restore(false);
                    precompute_h(e);
                    PLNMF_CUDA_CHECK(cudaEventRecord(a0, e->s));
                    update_h(e, c, PLNMF_ALGORITHM_TILED);
                    PLNMF_CUDA_CHECK(cudaEventRecord(a1, e->s));
                    precompute_w(e);
                    PLNMF_CUDA_CHECK(cudaEventRecord(b0, e->s));
                    update_w(e, c, PLNMF_ALGORITHM_TILED);
                    PLNMF_CUDA_CHECK(cudaEventRecord(b1, e->s));
                    PLNMF_CUDA_CHECK(cudaEventSynchronize(b1));
                    ms = (elapsed_s(a0, a1) + elapsed_s(b0, b1)) * 1e3;
                }
                if (update_ms) update_ms[i] = ms;
                if (i == 0 || ms < best_ms) {
                    best_ms = ms;
                    *best = cand[i];
                }
            }
            restore(true);
            PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
            e->update_macs = macs0;
        } catch (...) {
            free_snaps();
            throw;
        }
        free_snaps();
    });
}

plnmf_status plnmf_gpu_get_stats(const plnmf_gpu_engine* e, plnmf_gpu_stats* out) {
    return guarded([&] {
        if (!e || !out) throw std::invalid_argument("plnmf_gpu_get_stats: null argument");
        out->kernel_launches = e->launches;
        out->persistent_ctas = e->plan_w.grid;
        auto code = [&](const kern::PhaseBPlan& pl) {
            if (e->plan_tile < 0) return -1;
            return pl.streaming ? 3 : pl.stage_ops ? 0 : pl.sqn_smem ? 1 : 2;
        };
        out->w_plan = code(e->plan_w);
        out->h_plan = code(e->plan_h);
        out->sm_count = e->sms;
        out->device_bytes = e->bytes;
    });
}

plnmf_status plnmf_gpu_synchronize(plnmf_gpu_engine* e) {
    return guarded([&] {
        check_engine(e);
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s));
        PLNMF_CUDA_CHECK(cudaStreamSynchronize(e->s2));
        if (e->shard) plnmf::shard::check_error(e);
    });
}

}  // extern "C"
