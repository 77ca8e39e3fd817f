/* TEST INFRASTRUCTURE ONLY — see plnmf_oracle.h.
 *
 * CPU restatement of the reference arithmetic, one function per reference
 * function, each operation in the reference's order.  Compiled with
 * -ffp-contract=off so no a*b+c is fused (the reference's Release build has no
 * FMA either: proj/CMakeLists.txt:7-9 without -march=native).
 */
#include "plnmf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define AT(m, r, c, ld) (m)[(r) + (int64_t)(c) * (ld)]

/* std::max(eps, x) as the reference evaluates it: x only if eps < x. */
static inline double clamp_floor(double eps, double x) { return (eps < x) ? x : eps; }

/* ---- mt19937_64, the engine of proj/src/solver.cpp:46 ---------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* proj/src/solver.cpp:20-28: lo + (1-lo) * ((rng() >> 11) * 2^-53) */
static void fill_uniform(double* p, int64_t n, mt64* rng, double lo) {
    for (int64_t i = 0; i < n; ++i) {
        const double u = (double)(mt64_next(rng) >> 11) * 0x1.0p-53;
        p[i] = lo + (1.0 - lo) * u;
    }
}

void ora_init_factors(int64_t v, int64_t d, int64_t k, uint64_t seed, double eps, double* w,
                      double* ht) {
    mt64 rng;
    mt64_seed(&rng, seed);
    fill_uniform(w, v * k, &rng, eps);  /* solver.cpp:48 — W first */
    fill_uniform(ht, d * k, &rng, eps); /* solver.cpp:49 */
}

/* ---- proj/src/csr_matrix.cpp:30-50 ----------------------------------------- */
void ora_transpose(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp, const int64_t* ci,
                   const double* val, int64_t* trp, int64_t* tci, double* tval) {
    memset(trp, 0, sizeof(int64_t) * (size_t)(cols + 1));
    for (int64_t e = 0; e < nnz; ++e) ++trp[ci[e] + 1];
    for (int64_t c = 0; c < cols; ++c) trp[c + 1] += trp[c];
    int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cols + 1));
    memcpy(cursor, trp, sizeof(int64_t) * (size_t)cols);
    for (int64_t v = 0; v < rows; ++v)
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
            const int64_t pos = cursor[ci[e]]++;
            tci[pos] = v;
            tval[pos] = val[e];
        }
    free(cursor);
}

/* ---- proj/src/linalg.cpp:139-154: acc over e ascending, from 0.0 ------------ */
void ora_spmm(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci, const double* val,
              const double* x, int64_t n, double* y) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t v = 0; v < rows; ++v)
        for (int64_t j = 0; j < n; ++j) {
            const double* xc = x + j * cols;
            double acc = 0.0;
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) acc += val[e] * xc[ci[e]];
            AT(y, v, j, rows) = acc;
        }
}

/* ---- proj/src/linalg.cpp:168-204 -------------------------------------------
 * Upper-triangle pairs, 2048-row blocks, g(k,l) += acc per block, mirrored.
 * The per-block `omp simd reduction(+:acc)` (linalg.cpp:196-197) compiles, in
 * the reference's Release build, to two SSE2 lanes: lane 0 sums the even row
 * offsets of the block, lane 1 the odd ones (unaligned loads, no peeling); an
 * odd trailing row is added into lane 0; the lanes combine as
 * (lane0 + 0.0) + lane1 (objdump of linalg.o, gram_into._omp_fn.0).         */
void ora_gram(int64_t n, int64_t k, const double* m, double* g) {
    const int64_t kRowBlock = 2048;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t a = 0; a < k; ++a)
        for (int64_t b = a; b < k; ++b) {
            const double* ca = m + a * n;
            const double* cb = m + b * n;
            double gab = 0.0;
            for (int64_t v0 = 0; v0 < n; v0 += kRowBlock) {
                const int64_t v1 = (n < v0 + kRowBlock) ? n : v0 + kRowBlock;
                const int64_t len = v1 - v0;
                double lane0 = 0.0, lane1 = 0.0;
                for (int64_t i = 0; i + 1 < len; i += 2) {
                    lane0 = lane0 + ca[v0 + i] * cb[v0 + i];
                    lane1 = lane1 + ca[v0 + i + 1] * cb[v0 + i + 1];
                }
                if (len & 1) lane0 = lane0 + ca[v1 - 1] * cb[v1 - 1];
                const double acc = (lane0 + 0.0) + lane1;
                gab = gab + acc;
            }
            AT(g, a, b, k) = gab;
            AT(g, b, a, k) = gab;
        }
}

/* ---- proj/src/hals.cpp:51-72 ------------------------------------------------ */
void ora_update_h_reference(int64_t d, int64_t k, double eps, double* ht, const double* r,
                            const double* s) {
    for (int64_t kk = 0; kk < k; ++kk)
        for (int64_t row = 0; row < d; ++row) {
            double dot = 0.0;
            for (int64_t j = 0; j < k; ++j) dot += AT(ht, row, j, d) * AT(s, j, kk, k);
            AT(ht, row, kk, d) = clamp_floor(eps, AT(ht, row, kk, d) + AT(r, row, kk, d) - dot);
        }
}

/* ---- proj/src/hals.cpp:77-108 ----------------------------------------------- */
void ora_update_w_reference(int64_t v, int64_t k, double eps, double* w, const double* p,
                            const double* q, double* norms) {
    for (int64_t kk = 0; kk < k; ++kk) {
        const double qkk = AT(q, kk, kk, k);
        double* wc = w + kk * v;
        for (int64_t row = 0; row < v; ++row) {
            double dot = 0.0;
            for (int64_t j = 0; j < k; ++j) dot += AT(w, row, j, v) * AT(q, j, kk, k);
            wc[row] = clamp_floor(eps, wc[row] * qkk + AT(p, row, kk, v) - dot);
        }
        double ss = 0.0;
        for (int64_t row = 0; row < v; ++row) ss += wc[row] * wc[row];
        const double norm = sqrt(ss);
        if (norms) norms[kk] = norm;
        for (int64_t row = 0; row < v; ++row) wc[row] = clamp_floor(eps, wc[row] / norm);
    }
}

/* ---- proj/src/tiled.cpp ------------------------------------------------------ */
void ora_update_tiled(int64_t n, int64_t k, int64_t tile, double eps, int use_diag, int normalize,
                      int nthreads, double* mat, const double* coeff, const double* add,
                      double* norms) {
    double* nb = (double*)malloc(sizeof(double) * (size_t)(n * k));
    double* scratch = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* partials = (double*)calloc((size_t)(nthreads > 0 ? nthreads : 1), sizeof(double));
    const int64_t gamma = (k + tile - 1) / tile; /* tiling.cpp:8-18 */

    /* init_new_accumulator, tiled.cpp:28-50 */
    for (int64_t c = 0; c < k; ++c) {
        const double dkk = AT(coeff, c, c, k);
        for (int64_t i = 0; i < n; ++i)
            AT(nb, i, c, n) = use_diag ? AT(mat, i, c, n) * dkk : AT(mat, i, c, n);
    }
    /* phase1_left_contributions, tiled.cpp:52-65 -> gemm(-1, old[:,b:e), coeff[b:e,0:b), 1, nb[:,0:b))
     * -> accumulate_nn, linalg.cpp:45-59: c(i,j) += (alpha*b(kk,j)) * a(i,kk), kk ascending */
    for (int64_t tau = 1; tau < gamma; ++tau) {
        const int64_t b = tau * tile, e = (b + tile < k) ? b + tile : k;
        for (int64_t j = 0; j < b; ++j)
            for (int64_t kk = b; kk < e; ++kk) {
                const double f = -1.0 * AT(coeff, kk, j, k);
                for (int64_t i = 0; i < n; ++i) AT(nb, i, j, n) += f * AT(mat, i, kk, n);
            }
    }
    for (int64_t tau = 0; tau < gamma; ++tau) {
        const int64_t b = tau * tile, e = (b + tile < k) ? b + tile : k;
        /* phase2_in_tile, tiled.cpp:67-156 */
        for (int64_t t = b; t < e; ++t) {
            const int64_t nth = nthreads > 0 ? nthreads : 1;
            const int64_t chunk = (n + nth - 1) / nth;
            for (int64_t tid = 0; tid < nth; ++tid) {
                const int64_t v0 = (tid * chunk < n) ? tid * chunk : n;
                const int64_t v1 = (v0 + chunk < n) ? v0 + chunk : n;
                for (int64_t v = v0; v < v1; ++v) scratch[v] = 0.0;
                for (int64_t kk = b; kk < t; ++kk) {
                    const double f = AT(coeff, kk, t, k);
                    for (int64_t v = v0; v < v1; ++v) scratch[v] += AT(nb, v, kk, n) * f;
                }
                for (int64_t kk = t; kk < e; ++kk) {
                    const double f = AT(coeff, kk, t, k);
                    for (int64_t v = v0; v < v1; ++v) scratch[v] += AT(mat, v, kk, n) * f;
                }
                double local = 0.0;
                for (int64_t v = v0; v < v1; ++v) {
                    const double val = clamp_floor(eps, AT(nb, v, t, n) + AT(add, v, t, n) - scratch[v]);
                    AT(nb, v, t, n) = val;
                    local += val * val;
                }
                partials[tid] = local;
            }
            if (normalize) {
                double ss = 0.0;
                for (int64_t i = 0; i < nth; ++i) {
                    ss += partials[i];
                    partials[i] = 0.0;
                }
                const double norm = sqrt(ss);
                if (norms) norms[t] = norm;
                for (int64_t v = 0; v < n; ++v) AT(nb, v, t, n) = clamp_floor(eps, AT(nb, v, t, n) / norm);
            }
        }
        /* phase3_right_contributions, tiled.cpp:158-174 */
        for (int64_t j = e; j < k; ++j)
            for (int64_t kk = b; kk < e; ++kk) {
                const double f = -1.0 * AT(coeff, kk, j, k);
                for (int64_t i = 0; i < n; ++i) AT(nb, i, j, n) += f * AT(nb, i, kk, n);
            }
    }
    memcpy(mat, nb, sizeof(double) * (size_t)(n * k)); /* w.swap(ws.w_new), tiled.cpp:192,213 */
    free(nb);
    free(scratch);
    free(partials);
}

/* ---- proj/src/metrics.cpp ------------------------------------------------------ */
void ora_relative_error_gram(double a_norm_sq, int64_t v, int64_t d, int64_t k, const double* w,
                             const double* p, const double* q, const double* s, double* out3) {
    (void)d;
    double pw = 0.0;
    for (int64_t i = 0; i < v * k; ++i) pw += p[i] * w[i];
    double sq = 0.0;
    for (int64_t i = 0; i < k * k; ++i) sq += s[i] * q[i];
    double frob = a_norm_sq - 2.0 * pw + sq;
    double cancel = 0.0;
    if (frob < 0.0) {
        frob = 0.0;
        cancel = 1.0;
    }
    out3[0] = frob;
    out3[1] = sqrt(frob / a_norm_sq);
    out3[2] = cancel;
}

void ora_relative_error_direct_csr(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci,
                                   const double* val, double a_norm_sq, int64_t k, const double* w,
                                   const double* ht, double* out2) {
    double* per_row = (double*)calloc((size_t)(rows > 0 ? rows : 1), sizeof(double));
#pragma omp parallel
    {
        double* wh = (double*)malloc(sizeof(double) * (size_t)(cols > 0 ? cols : 1));
#pragma omp for schedule(dynamic, 32)
        for (int64_t v = 0; v < rows; ++v) {
            for (int64_t dd = 0; dd < cols; ++dd) wh[dd] = 0.0;
            for (int64_t kk = 0; kk < k; ++kk) {
                const double f = AT(w, v, kk, rows);
                const double* hc = ht + kk * cols;
                for (int64_t dd = 0; dd < cols; ++dd) wh[dd] += hc[dd] * f;
            }
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) wh[ci[e]] -= val[e];
            double acc = 0.0;
            for (int64_t dd = 0; dd < cols; ++dd) acc += wh[dd] * wh[dd];
            per_row[v] = acc;
        }
        free(wh);
    }
    double total = 0.0;
    for (int64_t v = 0; v < rows; ++v) total += per_row[v];
    free(per_row);
    out2[0] = total;
    out2[1] = sqrt(total / a_norm_sq);
}

double ora_norm_sq(int64_t nnz, const double* val) {
    double s = 0.0;
    for (int64_t i = 0; i < nnz; ++i) s += val[i] * val[i];
    return s;
}

double ora_factor_deviation(int64_t size, const double* ref, const double* other) {
    double max_diff = 0.0, max_ref = 0.0;
    for (int64_t i = 0; i < size; ++i) {
        const double dd = fabs(ref[i] - other[i]);
        const double rr = fabs(ref[i]);
        max_diff = (max_diff < dd) ? dd : max_diff;
        max_ref = (max_ref < rr) ? rr : max_ref;
    }
    if (max_ref == 0.0) return max_diff == 0.0 ? 0.0 : INFINITY;
    return max_diff / max_ref;
}
