/*
 * plnmf_gpu.h — C-ABI of the B200-native FAST-HALS / PL-NMF engine.
 *
 * This is the drop-in boundary for the reference's iteration loop
 * (arxiv/paper_1904_07935, /root/reference/proj).  Every entry point names the
 * reference interface it replaces.  Only plain pointers, sizes and PODs cross
 * it; matrices cross it exactly as the reference stores them: fp64,
 * column-major, element (r, c) at data[r + c*rows]
 * (proj/include/plnmf/dense_matrix.hpp:33-35), CSR with int64 indices
 * (proj/include/plnmf/csr_matrix.hpp:10-21).  Inside the engine the factors
 * live on the GPU row-major; the layout is converted only here.
 *
 * Errors: every call returns a plnmf_status; the message of the last failing
 * call on the calling thread is plnmf_last_error().  The status codes map 1:1
 * onto the reference's exception types:
 *   PLNMF_INVALID_ARGUMENT  std::invalid_argument  (config, shape, tile)
 *   PLNMF_RUNTIME           std::runtime_error     (non-finite objective)
 *   PLNMF_DOMAIN            std::domain_error      (||A|| = 0)
 *   PLNMF_CUDA              CUDA failure (no reference counterpart)
 *
 * Threading: one engine = one CUDA device + one stream; an engine is not
 * thread-safe, distinct engines are (proj/tools/plnmf.cpp:104-106).
 */
#ifndef PLNMF_GPU_H
#define PLNMF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLNMF_GPU_ABI_VERSION 1

typedef enum plnmf_status {
    PLNMF_OK = 0,
    PLNMF_INVALID_ARGUMENT = 1,
    PLNMF_RUNTIME = 2,
    PLNMF_DOMAIN = 3,
    PLNMF_CUDA = 4,
    PLNMF_NCCL = 5,
    PLNMF_PARSE = 6  /* plnmf::ParseError (a std::runtime_error), "source:line: what" */
} plnmf_status;

/* proj/include/plnmf/config.hpp:9 — Algorithm{reference, tiled}
 * ("fast-hals" / "pl-nmf" on the CLI, proj/tools/plnmf.cpp:76-80). */
typedef enum plnmf_algorithm { PLNMF_ALGORITHM_REFERENCE = 0, PLNMF_ALGORITHM_TILED = 1 } plnmf_algorithm;

/* Arithmetic of the device kernels. EXACT performs every multiply and add
 * separately, round-to-nearest, in the reference's per-element order (no FMA
 * contraction — the reference Release build has none).  FUSED uses fma() in
 * the same order (one rounding per multiply-add). */
typedef enum plnmf_math {
    PLNMF_MATH_EXACT = 0,
    PLNMF_MATH_FUSED = 1,
    /* Verification mode: EXACT arithmetic plus the
     * reference's own summation order for the two reductions the fast path
     * forms as fixed trees — the W column norms (serial over the rows for
     * fast-hals, proj/src/hals.cpp:97-100; per-OpenMP-thread chunk partials
     * combined in thread order for pl-nmf, proj/src/tiled.cpp:103-142, with
     * the team size set by plnmf_gpu_set_reference_threads) and the
     * Gram-identity dots <P,W>, <S,Q> (serial, proj/src/metrics.cpp:104-115).
     * With it, iterate() trajectories are bit-identical to the reference's.
     * Column-stepped and slow (serial chains): not the production path. */
    PLNMF_MATH_REFERENCE_ORDER = 2,
    /* EXACT, except that (a) a DENSE input's products P = A Ht and R = A^T W
     * (hals.cpp:29,43) and (b) the inter-tile phase A of a streaming tiled
     * update — init_new_accumulator + phase1_left_contributions for every column
     * at once (tiled.cpp:28-65), as init - old * U — run on the tensor cores:
     * each fp64 operand row is scaled by a power of two and cut into six 8-bit
     * digits, the 21 digit products that matter are exact u8 x u8 tcgen05.mma
     * GEMMs with int32 accumulators in TMEM, combined in fp64 (the Ozaki scheme;
     * csrc/ozaki.cu).  Error bounded by n 2^-46 times the operand scales; not the
     * reference's summation order. */
    PLNMF_MATH_TENSOR = 3
} plnmf_math;

/* proj/include/plnmf/config.hpp:11-22 — SolverConfig, field for field. */
typedef struct plnmf_config {
    int64_t rank;        /* K, >= 1 */
    double epsilon;      /* clamp floor, > 0 (default 1e-16) */
    int64_t max_iters;   /* >= 0 (default 100) */
    double rel_tol;      /* >= 0 (default 1e-6) */
    uint64_t seed;       /* default 0 */
    int64_t error_every; /* >= 1 (default 1) */
    int32_t deterministic; /* accepted, as in the reference (never read by its kernels);
                              the device kernels are run-to-run deterministic regardless */
    int64_t tile_size;   /* 0 = unresolved; the tiled path needs [1, rank] */
} plnmf_config;

/* proj/include/plnmf/workspace.hpp:15-28 — PhaseTimes (seconds). */
typedef struct plnmf_phase_times {
    double precompute_h, update_h, precompute_w, update_w;
    double phase1, phase2, phase3, normalize, error_eval;
} plnmf_phase_times;

/* proj/include/plnmf/solver.hpp:12-17 — TraceRecord. */
typedef struct plnmf_trace_record {
    int64_t iteration;
    double rel_error;
    double elapsed_s;
    plnmf_phase_times phases;
} plnmf_trace_record;

/* proj/include/plnmf/solver.hpp:19-25 — ConvergenceTrace.  The caller owns
 * `records` (capacity >= max_iters); n_records is filled in. */
typedef struct plnmf_trace {
    double initial_error;
    double total_seconds;
    uint64_t update_macs;
    plnmf_phase_times totals;
    int64_t n_records;
    int64_t capacity;
    plnmf_trace_record* records;
} plnmf_trace;

/* Workspace products (proj/include/plnmf/workspace.hpp:39-55). */
typedef enum plnmf_product {
    PLNMF_PRODUCT_P = 0,  /* A * Ht     V x K */
    PLNMF_PRODUCT_Q = 1,  /* Ht^T * Ht  K x K */
    PLNMF_PRODUCT_R = 2,  /* A^T * W    D x K */
    PLNMF_PRODUCT_S = 3,  /* W^T * W    K x K */
    PLNMF_PRODUCT_COLUMN_NORMS = 4 /* K, last W-update pre-normalisation norms */
} plnmf_product;

typedef struct plnmf_gpu_engine plnmf_gpu_engine;

/* Engine counters (instrumentation; no reference counterpart). */
typedef struct plnmf_gpu_stats {
    uint64_t kernel_launches;  /* engine kernels launched since create / reset */
    int32_t persistent_ctas;   /* CTAs of the grid-synchronised W update */
    int32_t sm_count;
    int64_t device_bytes;      /* device memory held by the engine */
    /* plan of the last tiled W / H update: 0 persistent look-ahead with the tile's
     * operands and the coefficient panel staged in shared memory, 1 panel staged
     * only, 2 neither staged, 3 streaming (stream.cu); -1 none yet */
    int32_t w_plan, h_plan;
} plnmf_gpu_stats;

/* ---- host-side helpers (no GPU needed) --------------------------------------- */
const char* plnmf_last_error(void);
int32_t plnmf_gpu_abi_version(void);
/* SolverConfig defaults (config.hpp:11-22) and SolverConfig::validate (config.cpp:7-15). */
void plnmf_config_default(plnmf_config* cfg);
plnmf_status plnmf_config_validate(const plnmf_config* cfg);
/* plan_tiles (proj/src/tiling.cpp:8-18); begins/ends may be NULL to query gamma. */
plnmf_status plnmf_plan_tiles(int64_t k, int64_t tile_size, int64_t* begins, int64_t* ends,
                              int64_t* gamma);
/* init_factors (proj/src/solver.cpp:43-51): mt19937_64, bit-identical to the reference. */
plnmf_status plnmf_init_factors(int64_t v, int64_t d, const plnmf_config* cfg, double* w_colmajor,
                                double* ht_colmajor);
/* Synthetic non-negative CSR: row r has Bernoulli(density) cells
 * at distinct sorted columns (geometric gaps from a counter-based splitmix64
 * stream keyed by (seed, r)), values U(0.1, 2.0) rounded to fp32.  Two calls:
 * with col_idx == NULL fills row_ptr (rows+1) and *nnz; then fills col_idx/values. */
plnmf_status plnmf_synth_csr(int64_t rows, int64_t cols, double density, uint64_t seed,
                             int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* nnz);

/* ---- Matrix Market input (proj/src/matrix_market.cpp) ---------------
 * plnmf_mm_read parses like read_matrix_market (same banner rules — coordinate
 * real/pattern general or array real general —, comment/blank-line skipping,
 * checks, messages and line numbers; failures return PLNMF_PARSE with
 * "path:line: what").  The parsed entries stay on the host in file order;
 * plnmf_gpu_create_mm assembles the CSR on the device (rows bucketed, each row
 * sorted by column keeping file order, duplicates summed in file order,
 * matrix_market.cpp:147-172) or uploads the dense array. */
typedef struct plnmf_mm plnmf_mm;
plnmf_status plnmf_mm_read(const char* path, plnmf_mm** out);
/* The same parser on an in-memory text (the istream overload, matrix_market.hpp:29). */
plnmf_status plnmf_mm_read_string(const char* text, const char* source_name, plnmf_mm** out);
/* entries = declared coordinate entries (before duplicate summation) or rows*cols. */
plnmf_status plnmf_mm_info(const plnmf_mm* m, int64_t* rows, int64_t* cols, int64_t* entries, int32_t* sparse);
plnmf_status plnmf_mm_free(plnmf_mm* m);

/* ---- engine -------------------------------------------------------------------- */
int32_t plnmf_gpu_device_count(void);
/* The device's name (cudaDeviceProp::name), NUL-terminated, truncated to len. */
plnmf_status plnmf_gpu_device_name(int32_t device, char* buf, int32_t len);

/* Uploads A (InputMatrix, proj/include/plnmf/input_matrix.hpp:11-34): validates
 * like CsrMatrix::validate (proj/src/csr_matrix.cpp:8-28), caches ||A||_F^2 in the
 * reference's serial order (proj/src/input_matrix.cpp:15-20), and builds A^T on
 * the device once (the reference caches transpose(A) in ws.at, proj/src/hals.cpp:26). */
plnmf_status plnmf_gpu_create_csr(int32_t device, int64_t rows, int64_t cols, int64_t nnz,
                                  const int64_t* row_ptr, const int64_t* col_idx,
                                  const double* values, int64_t rank, plnmf_gpu_engine** out);
plnmf_status plnmf_gpu_create_dense(int32_t device, int64_t rows, int64_t cols,
                                    const double* a_colmajor, int64_t rank,
                                    plnmf_gpu_engine** out);
/* An engine on a parsed Matrix Market file (InputMatrix(read_matrix_market(path))). */
plnmf_status plnmf_gpu_create_mm(int32_t device, const plnmf_mm* m, int64_t rank, plnmf_gpu_engine** out);
/* An engine on the SURVEY.md 8(d) synthetic CSR generated ON THE DEVICE (the
 * stream of plnmf_synth_csr; the large config's ~1e9 nonzeros never touch the
 * host).  ||A||^2 is still summed serially in the reference's order
 * (input_matrix.cpp:15-20) from the device values. */
plnmf_status plnmf_gpu_create_synthetic(int32_t device, int64_t rows, int64_t cols, double density, uint64_t seed,
                                        int64_t rank, plnmf_gpu_engine** out);
/* The device CSR of a sparse engine's A (row_ptr rows+1, col_idx/values nnz). */
plnmf_status plnmf_gpu_get_csr(plnmf_gpu_engine* e, int64_t* row_ptr, int64_t* col_idx, double* values);
/* Rows of a sparse engine's A (transposed = 0) or of its device-built A^T
 * (transposed = 1): for the n row indices, row_ptr_out (n+1, offsets into the
 * outputs) and, when col_idx/values are non-NULL, the entries. */
plnmf_status plnmf_gpu_get_csr_rows(plnmf_gpu_engine* e, int32_t transposed, const int64_t* rows, int64_t n,
                                    int64_t* row_ptr_out, int64_t* col_idx, double* values);
plnmf_status plnmf_gpu_destroy(plnmf_gpu_engine* e);
/* InputMatrix::norm_sq / nnz / rows / cols (input_matrix.hpp:17-28). */
plnmf_status plnmf_gpu_input_info(const plnmf_gpu_engine* e, int64_t* rows, int64_t* cols,
                                  int64_t* nnz, double* norm_sq);
plnmf_status plnmf_gpu_set_math(plnmf_gpu_engine* e, plnmf_math math);
/* PLNMF_MATH_REFERENCE_ORDER only: the reference's OpenMP team size
 * (omp_get_max_threads(), `--threads`, proj/tools/plnmf.cpp:104-106), which
 * fixes its tiled norm partials (tiled.cpp:97-99).  Default 1. */
plnmf_status plnmf_gpu_set_reference_threads(plnmf_gpu_engine* e, int32_t nthreads);
/* Verification hook: on != 0 makes every tiled update take the streaming
 * plan (stream.cu) that the planner otherwise picks only for shapes whose
 * per-SM rows do not fit the persistent kernel (C5), so its parity can be
 * tested on small inputs.  Results are those of the same T either way. */
plnmf_status plnmf_gpu_force_streaming(plnmf_gpu_engine* e, int32_t on);
/* Verification hook: the SpMMs take the column-blocked path (spmm.cu) with blocks of
 * `operand_rows` operand rows whenever the operand is larger (0: automatic — blocks of
 * ~48 MB for operands over ~96 MB).  Results are bit-identical either way. */
plnmf_status plnmf_gpu_force_spmm_blocks(plnmf_gpu_engine* e, int64_t operand_rows);

/* FactorPair in/out (proj/include/plnmf/workspace.hpp:32-35). */
plnmf_status plnmf_gpu_set_factors(plnmf_gpu_engine* e, const double* w_colmajor,
                                   const double* ht_colmajor);
plnmf_status plnmf_gpu_get_factors(plnmf_gpu_engine* e, double* w_colmajor, double* ht_colmajor);
/* init_factors on the host (bit-identical) followed by set_factors. */
plnmf_status plnmf_gpu_init_factors(plnmf_gpu_engine* e, const plnmf_config* cfg);

/* iterate (proj/src/solver.cpp:53-115): same loop, cadence, stop rule, trace and
 * exceptions, on the device-resident factors.  trace may be NULL. */
plnmf_status plnmf_gpu_iterate(plnmf_gpu_engine* e, const plnmf_config* cfg,
                               plnmf_algorithm algorithm, plnmf_trace* trace);

/* One-call drop-in for iterate() on HOST factors: uploads W/Ht, iterates,
 * downloads them back in place (what `Algorithm::gpu` in solver.cpp binds to). */
plnmf_status plnmf_gpu_iterate_host(plnmf_gpu_engine* e, const plnmf_config* cfg,
                                    plnmf_algorithm algorithm, double* w_colmajor,
                                    double* ht_colmajor, plnmf_trace* trace);

/* ---- step API (proj/include/plnmf/hals.hpp:11-21, tiled.hpp:37-40) ----------- */
plnmf_status plnmf_gpu_precompute_h_products(plnmf_gpu_engine* e); /* R = A^T W, S = W^T W */
plnmf_status plnmf_gpu_precompute_w_products(plnmf_gpu_engine* e); /* P = A Ht,  Q = Ht^T Ht */
plnmf_status plnmf_gpu_update_h(plnmf_gpu_engine* e, const plnmf_config* cfg,
                                plnmf_algorithm algorithm);
plnmf_status plnmf_gpu_update_w(plnmf_gpu_engine* e, const plnmf_config* cfg,
                                plnmf_algorithm algorithm);
/* evaluate_error (proj/src/solver.cpp:32-39): S = gram(W), Gram identity
 * (metrics.cpp:94-127), direct fallback below 1e-6 (metrics.cpp:79-92).
 * out3 = {frobenius_sq, relative, cancellation}. */
plnmf_status plnmf_gpu_evaluate_error(plnmf_gpu_engine* e, double* out3);
/* relative_error_direct (proj/src/metrics.cpp:79-92); out2 = {frobenius_sq, relative}. */
plnmf_status plnmf_gpu_relative_error_direct(plnmf_gpu_engine* e, double* out2);
plnmf_status plnmf_gpu_get_product(plnmf_gpu_engine* e, plnmf_product which, double* out_colmajor);
plnmf_status plnmf_gpu_set_product(plnmf_gpu_engine* e, plnmf_product which,
                                   const double* in_colmajor);

/* ---- sharded engine (multi-GPU) ------------------------------------
 * One engine per GPU (one process per GPU, or several engines in one process).
 * Rank g of `world` (<= 8) owns the W rows [v_lo, v_hi) and the Ht rows
 * [d_lo, d_hi) of balanced contiguous splits (the first n % world ranks get one
 * row more): A's CSR row block A[v_lo:v_hi, :] and the CSR of A^T's row block
 * A^T[d_lo:d_hi, :] (global indices; entries of each A^T row in ascending source
 * row, the order of transpose(), proj/src/csr_matrix.cpp:30-50).  After the ranks
 * are connected, the ordinary step/loop calls (plnmf_gpu_iterate,
 * plnmf_gpu_run_iterations, plnmf_gpu_precompute_*, plnmf_gpu_update_*,
 * plnmf_gpu_evaluate_error, plnmf_gpu_{set,get,init}_factors) run the sharded
 * iteration; every rank must make the same calls in the same order (they
 * exchange data with each other on the device, over NVLink peer memory).
 * Factors and products crossing the boundary are the rank's local rows;
 * init_factors gives each rank its rows of the whole factors' stream
 * (proj/src/solver.cpp:43-51).  Both algorithms (the W update's column norms are
 * exchanged between the ranks inside its kernel); Math::exact or fused. */
typedef enum plnmf_buffer {
    PLNMF_BUF_W = 0,  /* local W rows, row-major (v_hi-v_lo) x K */
    PLNMF_BUF_HT = 1, /* local Ht rows, row-major (d_hi-d_lo) x K */
    PLNMF_BUF_P = 6,  /* local rows of P */
    PLNMF_BUF_R = 7   /* local rows of R */
} plnmf_buffer;

#define PLNMF_IPC_HANDLE_BYTES 64

/* A rank from host CSR blocks (global indices); a_norm_sq = ||A||_F^2 of the whole matrix. */
plnmf_status plnmf_gpu_create_shard(int32_t device, int32_t world, int32_t shard_rank, int64_t v, int64_t d,
                                    int64_t nnz_rows, const int64_t* rp_rows, const int64_t* ci_rows,
                                    const double* val_rows, int64_t nnz_cols, const int64_t* rp_cols,
                                    const int64_t* ci_cols, const double* val_cols, double a_norm_sq,
                                    int64_t rank, plnmf_gpu_engine** out);
/* A rank of the synthetic matrix of plnmf_synth_csr(v, d, density, seed), its blocks
 * generated on the device (C5: nothing of A exists on the host).  ||A||^2 is then
 * set with plnmf_gpu_shard_set_norm_sq (see plnmf_gpu_shard_norm_sq). */
plnmf_status plnmf_gpu_create_shard_synthetic(int32_t device, int32_t world, int32_t shard_rank, int64_t v,
                                              int64_t d, double density, uint64_t seed, int64_t rank,
                                              plnmf_gpu_engine** out);
plnmf_status plnmf_gpu_shard_info(const plnmf_gpu_engine* e, int32_t* world, int32_t* shard_rank, int64_t* v_lo,
                                  int64_t* v_hi, int64_t* d_lo, int64_t* d_hi);
/* InputMatrix's serial ||A||^2 (proj/src/input_matrix.cpp:15-20) continued from `start`
 * over this rank's rows: chained rank 0 -> world-1 it reproduces the single sum exactly. */
plnmf_status plnmf_gpu_shard_norm_sq(plnmf_gpu_engine* e, double start, double* out);
plnmf_status plnmf_gpu_shard_set_norm_sq(plnmf_gpu_engine* e, double a_norm_sq);
/* Connecting ranks in different processes: every rank exports its window's CUDA IPC
 * handle (PLNMF_IPC_HANDLE_BYTES), the caller all-gathers them (any transport) and
 * passes world handles in rank order. */
plnmf_status plnmf_gpu_shard_ipc_handle(plnmf_gpu_engine* e, void* handle);
plnmf_status plnmf_gpu_shard_connect(plnmf_gpu_engine* e, const void* handles);
/* Connecting the ranks 0..world-1 of one process (any devices with peer access; several
 * ranks may share one device, each then using an equal share of its SMs — that needs
 * CUDA_MODULE_LOADING=EAGER in the process, else PLNMF_INVALID_ARGUMENT).  The ranks use
 * each other's windows directly: destroy them together, after their last call. */
plnmf_status plnmf_gpu_shard_connect_local(plnmf_gpu_engine* const* engines, int32_t world);
/* Failure detection: a device-side wait for another rank gives up after `seconds`
 * (default 20) and the next synchronising call on this rank fails with PLNMF_CUDA
 * ("a peer rank did not arrive ..."); the GPU is never left spinning. */
plnmf_status plnmf_gpu_shard_set_timeout(plnmf_gpu_engine* e, double seconds);
/* Rows of an engine buffer: out = n x K row-major, out[i*K + j] = buffer(rows[i], j).
 * For sampled parity checks on inputs too large to download whole (C5). */
plnmf_status plnmf_gpu_get_rows(plnmf_gpu_engine* e, plnmf_buffer which, const int64_t* rows, int64_t n,
                                double* out);

/* ---- timing / instrumentation --------------------------------------------------- */
/* n full iterations (H then W update, no error evaluation, no host sync inside),
 * timed with CUDA events on the engine stream; *device_ms = total. */
plnmf_status plnmf_gpu_run_iterations(plnmf_gpu_engine* e, const plnmf_config* cfg,
                                      plnmf_algorithm algorithm, int64_t n, double* device_ms);
/* Device time of each step of the last plnmf_gpu_run_iterations call, summed over
 * its iterations (CUDA events on the engine stream between the steps):
 * out4 = {precompute_h (R, S), update_h, precompute_w (P, Q), update_w} in ms. */
plnmf_status plnmf_gpu_phase_ms(const plnmf_gpu_engine* e, double* out4);
/* Times `reps` launches of one engine kernel family on the current state:
 * 0 = SpMM A*Ht (P), 1 = SpMM A^T*W (R), 2 = gram(W), 3 = W update, 4 = H update.
 * *avg_ms = mean CUDA-event duration per launch (events on the engine stream). */
plnmf_status plnmf_gpu_time_kernel(plnmf_gpu_engine* e, const plnmf_config* cfg, int32_t which,
                                   int32_t reps, double* avg_ms);
/* GPU tile selection, replacing best_integer_tile's cache model
 * (proj/include/plnmf/cost_model.hpp:65, proj/src/cost_model.cpp:131-142):
 * times one tiled H + W update from the current factors for each candidate
 * T (n == 0: 1, 2, 4, 8, 12, 16, 20, 24, 32 up to K), restores the factors,
 * and returns the fastest T in *best; update_ms[i] (optional, n entries, or 9
 * when n == 0) gets each candidate's time.  Results are parity-neutral: every
 * T reproduces the reference's tiled update for that T. */
plnmf_status plnmf_gpu_best_integer_tile(plnmf_gpu_engine* e, const plnmf_config* cfg, const int32_t* candidates,
                                         int32_t n, int32_t* best, double* update_ms);
plnmf_status plnmf_gpu_get_stats(const plnmf_gpu_engine* e, plnmf_gpu_stats* out);
plnmf_status plnmf_gpu_synchronize(plnmf_gpu_engine* e);

#ifdef __cplusplus
}
#endif
#endif /* PLNMF_GPU_H */
