/* TEST INFRASTRUCTURE ONLY — the CPU restatement of the reference's FAST-HALS /
 * PL-NMF arithmetic (arxiv/paper_1904_07935, /root/reference/proj).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it;
 * the product path (paper_1904_07935_b200/) never does.
 *
 * Every function restates one reference function in the SAME floating-point
 * operation order, so that on identical inputs it is bit-identical to the
 * compiled reference (oracle/_ref) — that equality is itself tested
 * (tests/test_oracle.py).  Layout is the reference's: fp64, column-major,
 * element (r, c) at data[r + c*rows] (proj/include/plnmf/dense_matrix.hpp:33-35);
 * CSR with int64 indices (proj/include/plnmf/csr_matrix.hpp:10-21).
 */
#ifndef PLNMF_ORACLE_H
#define PLNMF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/solver.cpp:20-28,43-51 — mt19937_64(seed); W first, then Ht. */
void ora_init_factors(int64_t v, int64_t d, int64_t k, uint64_t seed, double eps, double* w,
                      double* ht);

/* proj/src/csr_matrix.cpp:30-50 — counting-sort transpose. */
void ora_transpose(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci,
                   const double* val, int64_t* trp, int64_t* tci, double* tval);

/* proj/src/linalg.cpp:139-154 — y := a * x. */
void ora_spmm(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci, const double* val,
              const double* x, int64_t n, double* y);

/* proj/src/linalg.cpp:168-204 — g := m^T m in the compiled 2-lane order. */
void ora_gram(int64_t n, int64_t k, const double* m, double* g);

/* proj/src/hals.cpp:51-72 */
void ora_update_h_reference(int64_t d, int64_t k, double eps, double* ht, const double* r,
                            const double* s);
/* proj/src/hals.cpp:77-108; norms may be NULL */
void ora_update_w_reference(int64_t v, int64_t k, double eps, double* w, const double* p,
                            const double* q, double* norms);

/* proj/src/tiled.cpp:176-214 — the full tiled update of one factor.
 * W: use_diag = normalize = 1, coeff = Q, add = P.  H: 0, 0, S, R.
 * nthreads reproduces the OpenMP team size the reference ran phase 2 with
 * (its norm partials depend on it, proj/src/tiled.cpp:97-99,138-142).
 * mat is updated in place (the reference swaps buffers, :192,213). */
void ora_update_tiled(int64_t n, int64_t k, int64_t tile, double eps, int use_diag, int normalize,
                      int nthreads, double* mat, const double* coeff, const double* add,
                      double* norms);

/* proj/src/metrics.cpp:94-127 — out3 = {frobenius_sq, relative, cancellation} */
void ora_relative_error_gram(double a_norm_sq, int64_t v, int64_t d, int64_t k, const double* w,
                             const double* p, const double* q, const double* s, double* out3);
/* proj/src/metrics.cpp:49-92 (sparse) — out2 = {frobenius_sq, relative} */
void ora_relative_error_direct_csr(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci,
                                   const double* val, double a_norm_sq, int64_t k, const double* w,
                                   const double* ht, double* out2);
/* proj/src/input_matrix.cpp:15-20 */
double ora_norm_sq(int64_t nnz, const double* val);
/* proj/src/metrics.cpp:129-143 */
double ora_factor_deviation(int64_t size, const double* ref, const double* other);

#ifdef __cplusplus
}
#endif
#endif
