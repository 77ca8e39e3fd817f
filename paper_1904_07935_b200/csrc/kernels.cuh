// Launchers of the engine's sm_100a kernels.  Device layout: every dense
// matrix is ROW-major fp64 (row r contiguous, leading dimension = #cols);
// sparse matrices are CSR with int64 row pointers and int32 column indices.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "host.hpp"
#include "peer.cuh"

namespace plnmf {

struct CudaError : DeviceError {
    cudaError_t code;
    CudaError(cudaError_t c, const char* expr, const char* file, int line)
        : DeviceError(std::string("CUDA error ") + cudaGetErrorString(c) + " at " + file + ":" +
                      std::to_string(line) + " (" + expr + ")"),
          code(c) {}
};

enum class Math : int { exact = 0, fused = 1 };

// Every launcher returns the number of kernels it launched (for the
// engine's launch counter).
namespace kern {

// y := a * x over CSR a (rows x ?), x row-major (? x k), y row-major (rows x k).
// Per element: acc = 0; acc += val[e] * x[col[e]][j] for e ascending —
// proj/src/linalg.cpp:139-154.
// nnz: the matrix's nonzero count (selects the unroll depth; -1 if unknown).
// x_rows, cursor (rows int64 of workspace): an operand much larger than L2 is
// processed in column blocks of spmm_block_rows(k) operand rows (bit-identical).
// lean: a 64-register variant (same order) that fits next to a running Gram.
int spmm_csr(cudaStream_t s, Math m, int64_t rows, const int64_t* rp, const int32_t* ci,
             const double* val, const double* x, int64_t k, double* y, int64_t nnz = -1, int64_t x_rows = -1,
             int64_t* cursor = nullptr, int64_t force_block = 0, bool lean = false);
int64_t spmm_block_rows(int64_t k);

// g := m^T m (k x k) for row-major m (n x k), in the reference's compiled
// order (2048-row blocks, even/odd lanes, proj/src/linalg.cpp:168-204).
// scratch: gram_scratch_doubles(n, k) doubles.
int64_t gram_scratch_doubles(int64_t n, int64_t k);
// sms: the device's SM count (selects the CTA shape; the caller caches it).
int gram(cudaStream_t s, Math m, int64_t n, int64_t k, const double* mat, double* g,
         double* scratch, int sms = 148);

// Dense products for a dense input A (row-major v x d on the device).
// p := A * ht    (proj/src/hals.cpp:43 -> accumulate_nn, linalg.cpp:45-59)
int dense_a_ht(cudaStream_t s, Math m, int64_t v, int64_t d, int64_t k, const double* a,
               const double* ht, double* p);
// r := A^T * w   (proj/src/hals.cpp:29 -> accumulate_tn, linalg.cpp:62-79)
int dense_at_w(cudaStream_t s, Math m, int64_t v, int64_t d, int64_t k, const double* a,
               const double* w, double* r);

// ---- Math::tensor: Ozaki-split u8 tcgen05 GEMMs for dense A (ozaki.cu) -------------
// Digit tiles of x(r, k) (rows x cols; base[r*ld + k], or base[k*ld + r] when trans)
// with power-of-two row scales, in the GEMM's streaming layout (row tile rt).
int64_t ozaki_digit_bytes(int64_t rows, int64_t cols, int rt);
int ozaki_nt(int64_t n);  // the GEMM's N tile for n output columns
int ozaki_slice(cudaStream_t s, int64_t rows, int64_t cols, const double* base, int64_t ld, bool trans, int rt,
                double* scale, uint8_t* out);
int64_t ozaki_partial_doubles(int64_t m, int64_t n, int64_t kdim);
// out (m x n, row-major) := left (m x kdim) * right^T, both given as digit tiles
// (left: row tile 128, right: row tile ozaki_nt(n)); part: ozaki_partial_doubles.
int ozaki_gemm(cudaStream_t s, int64_t m, int64_t n, int64_t kdim, const uint8_t* a_digits, const double* sa,
               const uint8_t* b_digits, const double* sb, double* part, double* out);

// Math::tensor phase A of the streaming tiled update: init_new_accumulator +
// phase1_left_contributions (tiled.cpp:28-65) for every column at once as
// init - old * U (U: phase 1's coefficients), the product an Ozaki tcgen05 GEMM.
// ws: tensor_phase_a_bytes(n, k) bytes.
int64_t tensor_phase_a_bytes(int64_t n, int64_t k);
int tensor_phase_a(cudaStream_t s, int64_t n, int64_t k, int64_t tile, bool use_diag, const double* old_m,
                   const double* coeff, double* nb, void* ws);

// ---- tiled (PL-NMF) update, proj/src/tiled.cpp:176-214 --------------------------
struct PhaseBPlan {
    int grid = 0;            // CTAs
    int64_t rows_per_cta = 0;
    size_t smem = 0;         // dynamic shared memory bytes
    bool cooperative = false;
    bool streaming = false;  // fallback: tile operands streamed from global (stream.cu)
    bool stage_ops = true;   // look-ahead: tile old/add operands staged in shared memory
    bool sqn_smem = true;    // look-ahead: next tile's coeff panel staged in shared memory
    int kc = 0;              // look-ahead GEMM: operand chunk width staged by cp.async (0: unstaged path)
    int kst = 0;             // look-ahead GEMM: chunk ring depth
    int kbuf = 0;            // look-ahead GEMM: rings (one per item-owning thread)
    int resident = 0;        // H: the CTA's rows stay in shared memory (lookahead_gemm_resident)
};
// Global scratch for the coeff column panels of one tiled update.
int64_t qpanel_doubles(int64_t k, int64_t tile);
// One look-ahead kernel per update: init_new_accumulator (:28-50), phase 1
// (:52-65), and per tile phase 2 (:67-156) + phase 3 (:158-174).  w_update =>
// init scales by the diagonal and every column is L2-normalised with a
// grid-wide exchange (cooperative persistent launch, one CTA per SM).
// force_streaming: take the streaming fallback whatever the shape (verification).
PhaseBPlan plan_tiled_update(int64_t n, int64_t k, int64_t tile, bool normalize, int device,
                             bool force_streaming = false);
// Streaming fallback (stream.cu): phase A + one persistent streaming launch.
PhaseBPlan plan_stream_update(int64_t n, int64_t k, int64_t tile, bool normalize, int device);
// xch (sharded W update, world > 1): every column's sum of squares is also
// exchanged with the other ranks over peer memory (peer.cuh: world_sum).
// scratch (W only, stream_w_scratch_doubles): phase 2 on a column-major copy of each tile.
// push (with xch, world > 1): the finished tiles are also stored into every other rank's
// window and the channel flag released at the end (requires stream_fuses_push(k, tile)).
// tensor_ws (Math::tensor): phase A on the tensor cores (tensor_phase_a).
int stream_update(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t n, int64_t k, int64_t tile,
                  double eps, bool w_update, const double* old_m, double* out, const double* coeff,
                  const double* add, double* norms, double* partials, unsigned* counters,
                  const WorldXch* xch = nullptr, double* scratch = nullptr, const FusedPush* push = nullptr,
                  void* tensor_ws = nullptr);
bool stream_fuses_push(int64_t k, int64_t tile);
int64_t stream_w_scratch_doubles(const PhaseBPlan& plan, int64_t tile);
// init_new_accumulator + phase1_left_contributions into nb (tiled.cpp:28-65).
int stream_phase_a(cudaStream_t s, Math m, int64_t n, int64_t k, int64_t tile, bool use_diag, const double* old_m,
                   const double* coeff, double* nb);
// Column-stepped W update pieces for the sharded engine (shard.cu).
int shard_col_step(cudaStream_t s, Math m, int64_t n, int64_t k, int64_t b, int64_t e, int64_t t, double eps,
                   const double* old_m, double* nb, const double* coeff, const double* add, double* block_partials,
                   double* ss_out);
int shard_normalize(cudaStream_t s, int64_t n, int64_t k, int64_t t, double eps, int world,
                    const double* world_partials, double* nb, double* norms);
int shard_phase3(cudaStream_t s, Math m, int64_t n, int64_t k, int64_t b, int64_t e, double* nb, const double* coeff);
int tiled_update(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t n, int64_t k, int64_t tile,
                 double eps, bool w_update, const double* old_m, double* out, const double* coeff,
                 const double* add, double* norms, double* partials, unsigned* counters, double* totals,
                 long long* prof, double* qpanel, double* stream_scratch = nullptr,
                 const FusedPush* push = nullptr, void* tensor_ws = nullptr);

// Workspace of the grid-wide norm exchange (replicated partials + counters).
int64_t exchange_partials_doubles(int64_t k, int g);
int64_t exchange_counters(int64_t k);

// ---- reference (fast-hals) updaters, proj/src/hals.cpp --------------------------
int reference_update_h(cudaStream_t s, Math m, int64_t d, int64_t k, double eps, double* ht,
                       const double* r, const double* sm);
PhaseBPlan plan_reference_w(int64_t v, int device);
// xch (sharded engine, world > 1): every column norm summed over the ranks (peer.cuh).
int reference_update_w(cudaStream_t s, Math m, const PhaseBPlan& plan, int64_t v, int64_t k,
                       double eps, double* w, const double* p, const double* q, double* norms,
                       double* partials, unsigned* counters, double* totals, const WorldXch* xch = nullptr);

// ---- reference-order reductions (Math::reference_order, refmode.cu) -------------------
// *ss_out := column t's sum of squares of col_src (row-major n x k) in the
// reference's order: nth = 1 serial (hals.cpp:97-100), nth > 1 per-thread
// chunk partials added in thread order (tiled.cpp:103-106,129-142).
int ordered_ss(cudaStream_t s, int64_t n, int64_t k, int64_t t, int nth, const double* col_src, double* ss_out);
// column kk of update_w_reference before its normalisation (hals.cpp:88-96).
int ref_w_values(cudaStream_t s, int64_t v, int64_t k, int64_t kk, double eps, double* w, const double* p,
                 const double* q);
// *out := serial sum of a.*b over the column-major order of row-major rows x cols
// matrices (relative_error_gram, metrics.cpp:104-115).
int serial_dot_colmajor(cudaStream_t s, int64_t rows, int64_t cols, const double* a, const double* b, double* out);

// ---- metrics ---------------------------------------------------------------------
// out := sum_i a[i]*b[i] (n elements), fixed-order two-pass reduction.
constexpr int kDotBlocks = 296;
int dot(cudaStream_t s, Math m, int64_t n, const double* a, const double* b, double* partials,
        double* out);
// out3 := {frob_sq, relative, cancellation} from a2, *pw, *sq (metrics.cpp:115-126)
int error_finalize(cudaStream_t s, double a2, const double* pw, const double* sq, double* out3);
// Direct residual ||A - W Ht^T||_F^2 for CSR A (metrics.cpp:49-75) or dense A.
int direct_residual(cudaStream_t s, Math m, int64_t v, int64_t d, int64_t k, const int64_t* rp,
                    const int32_t* ci, const double* val, const double* a_dense, const double* w,
                    const double* ht, double* partials, int64_t n_partials, double* out);
int64_t direct_residual_partials(int64_t v, int64_t d);

// ---- input construction on the device (ingest.cu) ---------------------------------
// The synthetic CSR of plnmf_synth_csr generated on the device; returns nnz and
// cudaMalloc'ed arrays (the caller owns them).
// row0: global index of the first generated row (a shard's row block).
int64_t synth_csr_device(cudaStream_t s, int64_t rows, int64_t cols, double density, uint64_t seed,
                         int64_t** rp, int32_t** ci, double** val, int64_t row0 = 0);
// CSR of the transpose's row block [c_lo, c_hi) of the synthetic rows x cols
// matrix (the shard's column block of A): rows of the output are columns of A,
// entries in ascending source-row order (transpose() order,
// proj/src/csr_matrix.cpp:30-50), column indices = global source rows.
int64_t synth_transpose_block_device(cudaStream_t s, int64_t rows, int64_t cols, double density, uint64_t seed,
                                     int64_t c_lo, int64_t c_hi, int64_t** rp, int32_t** ci, double** val);
// read_coordinate's assembly (matrix_market.cpp:147-172) of n host COO entries
// (0-based, file order); returns nnz and cudaMalloc'ed CSR arrays.
int64_t coo_to_csr_device(cudaStream_t s, int64_t rows, int64_t cols, int64_t n, const int64_t* r,
                          const int64_t* c, const double* v, int64_t** rp, int32_t** ci, double** val);

// ---- sharded engine: peer-memory collectives (peer.cu) -----------------------------
// Byte offsets of the sections of one rank's window (identical on every rank).
struct PeerLayout {
    int world = 1;
    int64_t vcap = 0, dcap = 0, k = 0;
    size_t off_wfull[2] = {0, 0}, off_hfull[2] = {0, 0};  // double-buffered full factors, world * cap rows
    size_t off_sparts = 0, off_qparts = 0;                // world K x K Gram partials (slot = source rank)
    size_t off_pw = 0;                                    // kMaxWorld scalar partials
    size_t off_xvals = 0, off_xflags = 0;                 // norm exchange slots, xch_slot(t, rep, src)
    size_t off_agflags = 0;                               // all-gather flags [channel][source rank]
    size_t off_error = 0;                                 // timeout word
    size_t total = 0;
};
PeerLayout peer_layout(int world, int64_t vcap, int64_t dcap, int64_t k);
// Store `bytes` of src into dst.p[p] for every rank p (except this rank when
// skip_self), then release flag.p[p] = epoch in every window.  done: a zeroed
// local counter.
int peer_push(cudaStream_t s, const void* src, int64_t bytes, const PeerPtrs& dst, int world, int rank,
              bool skip_self, const PeerPtrs& flag, unsigned epoch, unsigned* done, int sms);
// Block the stream until flags[0..world) == epoch (bounded: sets *error on timeout).
int peer_wait(cudaStream_t s, const unsigned* flags, int world, unsigned epoch, int* error,
              unsigned long long timeout_ns);
// out[i] := parts[0*stride + i] + parts[1*stride + i] + ... in rank order.
int sum_parts(cudaStream_t s, const double* parts, int world, int64_t n, int64_t stride, double* out);
// Global indices of a balanced contiguous split of n over world ranks -> padded
// positions owner * cap + (x - lo(owner)).
int remap_split_index(cudaStream_t s, int32_t* idx, int64_t nnz, int64_t n, int world, int64_t cap);

// ---- layout / structure ------------------------------------------------------------
// dst (rows x cols, row-major) := src (rows x cols, column-major), and back.
int colmajor_to_rowmajor(cudaStream_t s, int64_t rows, int64_t cols, const double* src, double* dst);
int rowmajor_to_colmajor(cudaStream_t s, int64_t rows, int64_t cols, const double* src, double* dst);
// CSR (rows x cols) -> CSR of the transpose, entries of each output row in
// ascending source-row order (proj/src/csr_matrix.cpp:30-50).
int csr_transpose(cudaStream_t s, int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp,
                  const int32_t* ci, const double* val, int64_t* trp, int32_t* tci, double* tval);

}  // namespace kern
}  // namespace plnmf
