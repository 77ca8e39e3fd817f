/* TEST INFRASTRUCTURE ONLY — the synthetic workload generator of SURVEY.md 8(d)
 * for the reference side: the same counter-based stream as the engine's
 * plnmf_synth_csr (paper_1904_07935_b200/csrc/host.cpp), restated here so the
 * reference arm of bench.py and the CPU tests can build the benchmark input
 * without loading the engine library.  tests/test_oracle.py checks that both
 * produce identical arrays.
 *
 * Row r: splitmix64 stream seeded with seed ^ (0xD1B54A32D192ED03 * (r+1));
 * Bernoulli(density) cells visited by geometric gaps floor(log(u)/log1p(-p)),
 * u uniform on (0, 1]; values U(0.1, 2.0) rounded to fp32.
 * Compiled with -ffp-contract=off, like the engine's host code. */
#include <math.h>
#include <stdint.h>

static inline uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Walks row r; with col_idx == NULL only counts.  Returns the row's count. */
static int64_t synth_row(int64_t r, int64_t cols, double density, uint64_t seed, int64_t* col_idx,
                         double* values) {
    uint64_t s = seed ^ (0xD1B54A32D192ED03ULL * ((uint64_t)r + 1));
    splitmix64(&s);
    if (density <= 0.0) return 0;
    const int dense = density >= 1.0;
    const double inv_log_q = dense ? 0.0 : 1.0 / log1p(-density);
    int64_t c = -1, n = 0;
    for (;;) {
        int64_t gap = 0;
        if (!dense) {
            const double u = ((double)(splitmix64(&s) >> 11) + 1.0) * 0x1.0p-53;
            const double g = floor(log(u) * inv_log_q);
            if (g >= (double)cols) break;
            gap = (int64_t)g;
        }
        c += 1 + gap;
        if (c >= cols) break;
        const double u = (double)(splitmix64(&s) >> 11) * 0x1.0p-53;
        const float value = (float)(0.1 + 1.9 * u);
        if (col_idx) {
            col_idx[n] = c;
            values[n] = (double)value;
        }
        ++n;
    }
    return n;
}

/* Two calls, like plnmf_synth_csr: col_idx == NULL fills row_ptr and *nnz. */
int ora_synth_csr(int64_t rows, int64_t cols, double density, uint64_t seed, int64_t* row_ptr, int64_t* col_idx,
                  double* values, int64_t* nnz) {
    if (rows < 0 || cols < 0 || !(density >= 0.0) || density > 1.0) return 1;
    if (!col_idx) {
        int64_t* counts = row_ptr + 1;
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t r = 0; r < rows; ++r) counts[r] = synth_row(r, cols, density, seed, 0, 0);
        row_ptr[0] = 0;
        for (int64_t r = 0; r < rows; ++r) row_ptr[r + 1] += row_ptr[r];
        *nnz = row_ptr[rows];
        return 0;
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t r = 0; r < rows; ++r) synth_row(r, cols, density, seed, col_idx + row_ptr[r], values + row_ptr[r]);
    return 0;
}
