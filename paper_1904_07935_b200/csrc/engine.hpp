// The engine object shared by engine.cu (single-GPU engine, C-ABI) and
// shard_engine.cu (the sharded multi-GPU engine).
#pragma once

#include <vector>

#include "common.cuh"
#include "host.hpp"
#include "kernels.cuh"
#include "peer.cuh"
#include "plnmf_gpu.h"

struct plnmf_gpu_engine {
    int device = 0;
    cudaStream_t s = nullptr, s2 = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    int64_t v = 0, d = 0, k = 0, nnz = 0;
    int64_t nnz_t = -1;  // nonzeros of the A^T block (sharded engines: of the local column block)
    bool sparse = true;
    double a2 = 0.0;
    plnmf::Math math = plnmf::Math::exact;
    // Math::reference_order (PLNMF_MATH_REFERENCE_ORDER): exact arithmetic plus the
    // reference's own summation order for the W norms and the error dots (refmode.cu)
    bool ref_order = false;
    // Math::tensor (dense A only): A's digit tiles for P = A Ht (rows of A) and for
    // R = A^T W (columns of A), built once; the factor's digits per product
    bool tensor = false;
    uint8_t *dig_ap = nullptr, *dig_ar = nullptr, *dig_b = nullptr;
    double *sc_ap = nullptr, *sc_ar = nullptr, *sc_b = nullptr, *oz_part = nullptr;
    int ref_threads = 1;  // the reference's OpenMP team size for the tiled norm partials
    bool force_streaming = false;
    double last_phase_ms[4] = {0, 0, 0, 0};
  // run_iterations: precompute_h, update_h, precompute_w, update_w  // plnmf_gpu_force_streaming: tiled updates take the streaming plan

    int64_t *rp = nullptr, *trp = nullptr;
    int32_t *ci = nullptr, *tci = nullptr;
    double *val = nullptr, *tval = nullptr, *a_dense = nullptr;
    double *w = nullptr, *ht = nullptr, *w_new = nullptr, *h_new = nullptr;
    double *p = nullptr, *q = nullptr, *r = nullptr, *sm = nullptr, *norms = nullptr;
    double* r_next = nullptr;  // R of the current W computed ahead (iterate), swapped into r when used
    int64_t *cursor_p = nullptr, *cursor_r = nullptr;  // column-blocked SpMM cursors (spmm.cu)
    int64_t spmm_block = 0;  // > 0: column blocks of this many operand rows (verification hook)
    double *gram_scratch = nullptr, *partials = nullptr, *dot_partials = nullptr;
    double *scalars = nullptr;  // [0] pw, [1] sq, [2..4] error report, [5] direct sum
    double *staging = nullptr, *direct_partials = nullptr;
    double* host_scalars = nullptr;  // pinned mirror of scalars
    unsigned* counters = nullptr;  // K, grid-exchange arrival counters
    double* totals = nullptr;      // K, grid-exchange published norms
    int64_t n_partials = 0, n_direct_partials = 0;

    bool s_valid = false;  // sm == gram(w) of the current w
    bool r_valid = false;  // r == A^T w of the current w, computed ahead on s2 (iterate: join_r)
    cudaEvent_t join_r = nullptr;
    double* dot_partials2 = nullptr;  // <P, W> on s2 beside gram(W) (evaluate_error_launch with R ahead)
    cudaEvent_t join_pw = nullptr;
    cudaEvent_t err_done = nullptr;  // an error report's readback has landed (evaluate_error)
    uint64_t launches = 0, update_macs = 0;
    int64_t bytes = 0;
    int sms = 0;
    std::vector<void*> allocs;

    // cached phase-B plans, keyed by tile size
    int64_t plan_tile = -1;
    plnmf::kern::PhaseBPlan plan_w, plan_h, plan_ref_w;
    bool have_ref_w = false;


    std::vector<cudaEvent_t> events;  // per-phase timing pool
    long long* prof = nullptr;        // PLNMF_PROFILE=1: phase-B section cycle counters
    int64_t prof_n = 0;
    double* wscratch = nullptr;       // streaming W update: column-major tile scratch (stream.cu)
    char* tensor_ws = nullptr;        // Math::tensor: phase A of the streaming updates (ozaki.cu)
    int64_t tensor_ws_bytes = 0;
    int64_t wscratch_n = 0;
    double* qpanel = nullptr;         // coeff column panels of the tiled updates
    int64_t qpanel_n = 0;

    // reference-order W update (refmode.cu): column sum of squares and chunk partials
    double *col_ss = nullptr, *col_partials = nullptr;

    // sharded engine (multi-GPU, shard_engine.cu): rank `rank` of `world` owns the W rows
    // [v_lo, v_lo + v) and the Ht rows [d_lo, d_lo + d) of balanced contiguous splits.  W, W_new,
    // Ht, H_new are this rank's slices of the double-buffered full factors in the peer window;
    // the full factors are padded to world * vcap (dcap) rows, rank g's rows at g * vcap.
    bool shard = false;
    int world = 1, rank = 0;
    int64_t vfull = 0, dfull = 0, v_lo = 0, d_lo = 0, vcap = 0, dcap = 0;
    plnmf::kern::PeerLayout lay{};
    char* win = nullptr;                           // this rank's window
    char* peer_win[plnmf::kMaxWorld] = {};         // every rank's window as mapped here
    bool peer_ipc[plnmf::kMaxWorld] = {};          // opened from an IPC handle (closed on destroy)
    bool connected = false;
    int sm_cap = 0;                                // ranks sharing one GPU: CTAs of the persistent W kernel
    unsigned ag_epoch[plnmf::kChannels] = {};
    unsigned xch_epoch = 0;
    unsigned long long peer_timeout_ns = plnmf::kPeerTimeoutNs;
    unsigned* push_done = nullptr;
};

namespace plnmf {

template <class T>
T* dalloc(plnmf_gpu_engine* e, int64_t n) {
    void* ptr = nullptr;
    const size_t bytes = sizeof(T) * (size_t)(n > 0 ? n : 1);
    PLNMF_CUDA_CHECK(cudaMalloc(&ptr, bytes));
    e->allocs.push_back(ptr);
    e->bytes += (int64_t)bytes;
    return static_cast<T*>(ptr);
}

// ---- engine lifetime (engine.cu) ---------------------------------------------------------
namespace eng {
void release(plnmf_gpu_engine* e);
void check_engine(const plnmf_gpu_engine* e);
void setup_common(plnmf_gpu_engine* e, int device, int64_t rank);
void alloc_workspace(plnmf_gpu_engine* e);
}  // namespace eng

// ---- sharded engine hooks (shard_engine.cu) ---------------------------------------------
namespace shard {
double* w_full(const plnmf_gpu_engine* e);   // the full W buffer holding the current W
double* ht_full(const plnmf_gpu_engine* e);
void wait(plnmf_gpu_engine* e, PeerChannel c);           // every rank's push of channel c arrived
void push_factor(plnmf_gpu_engine* e, PeerChannel c);    // this rank's W (Ht) rows into every window
void reduce_kxk(plnmf_gpu_engine* e, PeerChannel c, double* inout);  // rank-ordered sum of K x K partials
void reduce_scalar(plnmf_gpu_engine* e, double* inout);              // rank-ordered sum of one double
WorldXch next_exchange(plnmf_gpu_engine* e);             // norm-exchange arguments of the next W update
// the all-gather of channel c fused into the kernel that writes out_local (this rank's slice)
FusedPush fused_push(plnmf_gpu_engine* e, PeerChannel c, const double* out_local);
void check_error(plnmf_gpu_engine* e);                   // raise a peer timeout recorded on the device
void close_peers(plnmf_gpu_engine* e);
}  // namespace shard
}  // namespace plnmf
