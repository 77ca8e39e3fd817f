// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// extern "C" shim over the UNMODIFIED reference library (libplnmf, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Lets
// the Python tests, the golden-fixture generator and bench.py's CPU-baseline
// leg drive the reference's own public API:
//   init_factors / iterate            proj/include/plnmf/solver.hpp:29-36
//   precompute_{h,w}_products         proj/include/plnmf/hals.hpp:11-15
//   update_{h,w}_reference            proj/include/plnmf/hals.hpp:20-21
//   update_{h,w}_tiled + phases       proj/include/plnmf/tiled.hpp:10-40
//   spmm_into / gram_into / transpose proj/include/plnmf/linalg.hpp:13-27,
//                                     proj/include/plnmf/csr_matrix.hpp:23
//   relative_error_{gram,direct}      proj/include/plnmf/metrics.hpp:17-29
// All matrices cross this shim column-major fp64, exactly as the reference
// stores them (proj/include/plnmf/dense_matrix.hpp:33-35).
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "plnmf/config.hpp"
#include "plnmf/cost_model.hpp"
#include "plnmf/hals.hpp"
#include "plnmf/linalg.hpp"
#include "plnmf/matrix_market.hpp"
#include "plnmf/metrics.hpp"
#include "plnmf/solver.hpp"
#include "plnmf/tiled.hpp"
#include "plnmf/tiling.hpp"

using namespace plnmf;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 runtime_error, 3 domain_error, 4 other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

DenseMatrix from_ptr(const double* p, index_t rows, index_t cols) {
    DenseMatrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), p, sizeof(double) * rows * cols);
    return m;
}

void to_ptr(const DenseMatrix& m, double* p) {
    if (m.size()) std::memcpy(p, m.data(), sizeof(double) * m.size());
}

CsrMatrix csr_from(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci,
                   const double* val) {
    CsrMatrix c;
    c.rows = rows;
    c.cols = cols;
    c.row_ptr.assign(rp, rp + rows + 1);
    c.col_idx.assign(ci, ci + nnz);
    c.values.assign(val, val + nnz);
    return c;
}

struct Session {
    std::vector<InputMatrix> a;  // 0 or 1 element (InputMatrix has no default ctor)
    UpdateWorkspace ws;
    Session(index_t v, index_t d, index_t k) : ws(v, d, k) {}
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_max_threads() { return omp_get_max_threads(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }

// ---- input matrices -------------------------------------------------------
void* ref_input_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci,
                    const double* val) {
    InputMatrix* out = nullptr;
    if (guarded([&] { out = new InputMatrix(csr_from(rows, cols, nnz, rp, ci, val)); })) return nullptr;
    return out;
}
void* ref_input_dense(int64_t rows, int64_t cols, const double* colmajor) {
    InputMatrix* out = nullptr;
    if (guarded([&] { out = new InputMatrix(from_ptr(colmajor, rows, cols)); })) return nullptr;
    return out;
}
void ref_input_free(void* a) { delete static_cast<InputMatrix*>(a); }
double ref_input_norm_sq(void* a) { return static_cast<InputMatrix*>(a)->norm_sq(); }
int64_t ref_input_nnz(void* a) { return static_cast<InputMatrix*>(a)->nnz(); }

// Matrix Market: two calls. First (out arrays NULL) returns shape + nnz + kind
// (1 = csr, 0 = dense); second fills the caller's buffers.
int ref_read_mm(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz, int* is_sparse,
                int64_t* rp, int64_t* ci, double* val) {
    return guarded([&] {
        InputMatrix a = read_matrix_market(std::string(path));
        *rows = a.rows();
        *cols = a.cols();
        *is_sparse = a.is_sparse();
        if (a.is_sparse()) {
            const CsrMatrix& c = a.csr();
            *nnz = c.nnz();
            if (rp) {
                std::memcpy(rp, c.row_ptr.data(), sizeof(int64_t) * (c.rows + 1));
                std::memcpy(ci, c.col_idx.data(), sizeof(int64_t) * c.nnz());
                std::memcpy(val, c.values.data(), sizeof(double) * c.nnz());
            }
        } else {
            *nnz = a.rows() * a.cols();
            if (val) to_ptr(a.dense(), val);
        }
    });
}

// ---- kernels --------------------------------------------------------------
int ref_spmm(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci,
             const double* val, const double* x, int64_t n, double* y) {
    return guarded([&] {
        const CsrMatrix a = csr_from(rows, cols, nnz, rp, ci, val);
        const DenseMatrix xm = from_ptr(x, cols, n);
        DenseMatrix ym(rows, n);
        spmm_into(a, xm, ym);
        to_ptr(ym, y);
    });
}

int ref_transpose(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci,
                  const double* val, int64_t* trp, int64_t* tci, double* tval) {
    return guarded([&] {
        const CsrMatrix t = transpose(csr_from(rows, cols, nnz, rp, ci, val));
        std::memcpy(trp, t.row_ptr.data(), sizeof(int64_t) * (cols + 1));
        std::memcpy(tci, t.col_idx.data(), sizeof(int64_t) * nnz);
        std::memcpy(tval, t.values.data(), sizeof(double) * nnz);
    });
}

int ref_gram(int64_t n, int64_t k, const double* m, double* g) {
    return guarded([&] {
        DenseMatrix gm(k, k);
        gram_into(from_ptr(m, n, k), gm);
        to_ptr(gm, g);
    });
}

int ref_gemm(double alpha, const double* a, int64_t ar, int64_t ac, int ta, const double* b,
             int64_t br, int64_t bc, int tb, double beta, double* c, int64_t cr, int64_t cc) {
    return guarded([&] {
        const DenseMatrix am = from_ptr(a, ar, ac), bm = from_ptr(b, br, bc);
        DenseMatrix cm = from_ptr(c, cr, cc);
        gemm(alpha, am.view(), ta, bm.view(), tb, beta, cm.view());
        to_ptr(cm, c);
    });
}

int ref_init_factors(int64_t v, int64_t d, int64_t k, uint64_t seed, double eps, double* w,
                     double* ht) {
    return guarded([&] {
        SolverConfig cfg;
        cfg.rank = k;
        cfg.seed = seed;
        cfg.epsilon = eps;
        const FactorPair f = init_factors(v, d, cfg);
        to_ptr(f.w, w);
        to_ptr(f.ht, ht);
    });
}

int ref_plan_tiles(int64_t k, int64_t t, int64_t* begins, int64_t* ends, int64_t* gamma) {
    return guarded([&] {
        const TilingPlan p = plan_tiles(k, t);
        *gamma = p.gamma();
        if (begins)
            for (index_t i = 0; i < p.gamma(); ++i) {
                begins[i] = p.tiles[i].begin;
                ends[i] = p.tiles[i].end;
            }
    });
}

double ref_model_tile_size(int64_t k, uint64_t cache_bytes) {
    return model_tile_size(k, MachineModel{cache_bytes, 8});
}
int64_t ref_best_integer_tile(int64_t v, int64_t d, int64_t k, uint64_t cache_bytes) {
    return best_integer_tile({v, d, k}, MachineModel{cache_bytes, 8});
}

// ---- sessions: one InputMatrix + one UpdateWorkspace, driven step by step --
void* ref_session_create(void* a, int64_t k) {
    Session* s = nullptr;
    if (guarded([&] {
            InputMatrix* in = static_cast<InputMatrix*>(a);
            s = new Session(in->rows(), in->cols(), k);
            s->a.push_back(*in);
        }))
        return nullptr;
    return s;
}
void ref_session_free(void* s) { delete static_cast<Session*>(s); }

// which: 0 P, 1 Q, 2 R, 3 S, 4 column_norms
static DenseMatrix* ws_mat(Session* s, int which) {
    switch (which) {
        case 0: return &s->ws.p;
        case 1: return &s->ws.q;
        case 2: return &s->ws.r;
        case 3: return &s->ws.s;
        default: return nullptr;
    }
}
int ref_session_get(void* sp, int which, double* out) {
    Session* s = static_cast<Session*>(sp);
    if (which == 4) {
        std::memcpy(out, s->ws.column_norms.data(), sizeof(double) * s->ws.column_norms.size());
        return 0;
    }
    to_ptr(*ws_mat(s, which), out);
    return 0;
}
int ref_session_set(void* sp, int which, const double* in) {
    Session* s = static_cast<Session*>(sp);
    DenseMatrix* m = ws_mat(s, which);
    std::memcpy(m->data(), in, sizeof(double) * m->size());
    return 0;
}
uint64_t ref_session_macs(void* sp) { return static_cast<Session*>(sp)->ws.update_macs; }
void ref_session_phase_times(void* sp, double* out9) {
    const PhaseTimes& p = static_cast<Session*>(sp)->ws.phase_times;
    const double v[9] = {p.precompute_h, p.update_h, p.precompute_w, p.update_w, p.phase1,
                         p.phase2,       p.phase3,   p.normalize,    p.error_eval};
    std::memcpy(out9, v, sizeof(v));
}

int ref_session_precompute_h(void* sp, const double* w, int64_t k) {
    Session* s = static_cast<Session*>(sp);
    return guarded([&] { precompute_h_products(s->a[0], from_ptr(w, s->a[0].rows(), k), s->ws); });
}
int ref_session_precompute_w(void* sp, const double* ht, int64_t k) {
    Session* s = static_cast<Session*>(sp);
    return guarded([&] { precompute_w_products(s->a[0], from_ptr(ht, s->a[0].cols(), k), s->ws); });
}

// In-place factor updates. tile_size 0 = reference updater.
int ref_session_update_h(void* sp, double* ht, int64_t k, double eps, int64_t tile_size) {
    Session* s = static_cast<Session*>(sp);
    return guarded([&] {
        SolverConfig cfg;
        cfg.rank = k;
        cfg.epsilon = eps;
        const index_t d = s->a[0].cols();
        FactorPair f{DenseMatrix(1, k), from_ptr(ht, d, k)};
        if (tile_size > 0)
            update_h_tiled(f, s->ws, plan_tiles(k, tile_size), cfg);
        else
            update_h_reference(f, s->ws, cfg);
        to_ptr(f.ht, ht);
    });
}
int ref_session_update_w(void* sp, double* w, int64_t k, double eps, int64_t tile_size) {
    Session* s = static_cast<Session*>(sp);
    return guarded([&] {
        SolverConfig cfg;
        cfg.rank = k;
        cfg.epsilon = eps;
        const index_t v = s->a[0].rows();
        FactorPair f{from_ptr(w, v, k), DenseMatrix(1, k)};
        if (tile_size > 0)
            update_w_tiled(f, s->ws, plan_tiles(k, tile_size), cfg);
        else
            update_w_reference(f, s->ws, cfg);
        to_ptr(f.w, w);
    });
}

// ---- phases of the tiled update on raw buffers (tests) ---------------------
int ref_init_new_accumulator(const double* old_m, int64_t n, int64_t k, const double* diag,
                             double* buf, int use_diag) {
    return guarded([&] {
        UpdateWorkspace ws(n, n, k);
        DenseMatrix b(n, k);
        init_new_accumulator(from_ptr(old_m, n, k), from_ptr(diag, k, k), b, use_diag, ws);
        to_ptr(b, buf);
    });
}
int ref_phase1(const double* old_m, int64_t n, int64_t k, const double* coeff, int64_t t,
               double* buf) {
    return guarded([&] {
        UpdateWorkspace ws(n, n, k);
        DenseMatrix b = from_ptr(buf, n, k);
        phase1_left_contributions(from_ptr(old_m, n, k), from_ptr(coeff, k, k), plan_tiles(k, t), b, ws);
        to_ptr(b, buf);
    });
}
int ref_phase2(const double* old_m, int64_t n, int64_t k, const double* coeff, const double* add,
               int64_t t, int64_t tile_idx, int normalize, double eps, double* buf, double* norms) {
    return guarded([&] {
        UpdateWorkspace ws(n, n, k);
        SolverConfig cfg;
        cfg.rank = k;
        cfg.epsilon = eps;
        DenseMatrix b = from_ptr(buf, n, k);
        phase2_in_tile(from_ptr(old_m, n, k), b, from_ptr(coeff, k, k), from_ptr(add, n, k),
                       plan_tiles(k, t), tile_idx, normalize, cfg, ws);
        to_ptr(b, buf);
        if (norms) std::memcpy(norms, ws.column_norms.data(), sizeof(double) * k);
    });
}
int ref_phase3(double* buf, int64_t n, int64_t k, const double* coeff, int64_t t, int64_t tile_idx) {
    return guarded([&] {
        UpdateWorkspace ws(n, n, k);
        DenseMatrix b = from_ptr(buf, n, k);
        phase3_right_contributions(b, from_ptr(coeff, k, k), plan_tiles(k, t), tile_idx, ws);
        to_ptr(b, buf);
    });
}

// ---- metrics ----------------------------------------------------------------
int ref_relative_error_gram(double a_norm_sq, const double* w, int64_t v, const double* ht,
                            int64_t d, int64_t k, const double* p, const double* q, const double* s,
                            double* out3) {
    return guarded([&] {
        const ErrorReport r = relative_error_gram(a_norm_sq, from_ptr(w, v, k), from_ptr(ht, d, k),
                                                  from_ptr(p, v, k), from_ptr(q, k, k), from_ptr(s, k, k));
        out3[0] = r.frobenius_sq;
        out3[1] = r.relative;
        out3[2] = r.cancellation;
    });
}
int ref_relative_error_direct(void* a, const double* w, const double* ht, int64_t k, double* out2) {
    return guarded([&] {
        InputMatrix* in = static_cast<InputMatrix*>(a);
        const ErrorReport r =
            relative_error_direct(*in, from_ptr(w, in->rows(), k), from_ptr(ht, in->cols(), k));
        out2[0] = r.frobenius_sq;
        out2[1] = r.relative;
    });
}
double ref_factor_deviation(const double* ref, const double* other, int64_t rows, int64_t cols) {
    return factor_deviation(from_ptr(ref, rows, cols), from_ptr(other, rows, cols));
}

// ---- the whole loop -----------------------------------------------------------
// records: n x 11 doubles {iteration, rel_error, elapsed_s, 8 phase buckets... error_eval}
// (iteration, rel_error, elapsed_s, precompute_h, update_h, precompute_w,
//  update_w, phase1, phase2, phase3, normalize, error_eval) = 12 per record.
int ref_iterate(void* a, double* w, double* ht, int64_t k, double eps, int64_t max_iters,
                double rel_tol, uint64_t seed, int64_t error_every, int64_t tile_size,
                int algorithm, double* initial_error, int64_t* n_records, double* records,
                double* totals10, uint64_t* macs) {
    return guarded([&] {
        InputMatrix* in = static_cast<InputMatrix*>(a);
        SolverConfig cfg;
        cfg.rank = k;
        cfg.epsilon = eps;
        cfg.max_iters = max_iters;
        cfg.rel_tol = rel_tol;
        cfg.seed = seed;
        cfg.error_every = error_every;
        cfg.tile_size = tile_size;
        FactorPair f{from_ptr(w, in->rows(), k), from_ptr(ht, in->cols(), k)};
        const ConvergenceTrace tr =
            iterate(*in, f, cfg, algorithm ? Algorithm::tiled : Algorithm::reference);
        to_ptr(f.w, w);
        to_ptr(f.ht, ht);
        *initial_error = tr.initial_error;
        *n_records = static_cast<int64_t>(tr.records.size());
        for (std::size_t i = 0; i < tr.records.size(); ++i) {
            const TraceRecord& r = tr.records[i];
            const PhaseTimes& p = r.phases;
            const double row[12] = {double(r.iteration), r.rel_error, r.elapsed_s, p.precompute_h,
                                    p.update_h,          p.precompute_w, p.update_w, p.phase1,
                                    p.phase2,            p.phase3,       p.normalize, p.error_eval};
            std::memcpy(records + 12 * i, row, sizeof(row));
        }
        const PhaseTimes& p = tr.totals;
        const double t[10] = {tr.total_seconds, p.precompute_h, p.update_h, p.precompute_w,
                              p.update_w,       p.phase1,       p.phase2,   p.phase3,
                              p.normalize,      p.error_eval};
        std::memcpy(totals10, t, sizeof(t));
        *macs = tr.update_macs;
    });
}

}  // extern "C"
