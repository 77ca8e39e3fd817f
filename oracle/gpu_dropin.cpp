// TEST INFRASTRUCTURE ONLY — compiles INTEGRATION.md's `Algorithm::gpu`
// binding against the UNMODIFIED reference (its headers and objects, built by
// oracle/Makefile from /root/reference/proj/src) and runs the reference's own
// acceptance claims through it (proj/tests/acceptance.cpp:105-233), plus the
// bit-identity of the drop-in in reference-order mode:
//
//   criterion 5  clamp floor and unit-norm invariants on every GPU iterate
//   criterion 6  exact MAC parity between the GPU update paths and the CPU's
//   criterion 7  objective non-increasing over 100 GPU iterations (K = 8, 16,
//                both algorithms) and planted-instance recovery
//   drop-in      iterate_gpu(..., PLNMF_MATH_REFERENCE_ORDER) == iterate()
//                bit for bit (factors and every trace error), fast-hals and
//                pl-nmf, with the reference's OpenMP team size
//
// Output: one PASS/FAIL line per check; the exit code is the failure count
// (tests/test_dropin.py runs it on the GPU box).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "plnmf/cost_model.hpp"
#include "plnmf/hals.hpp"
#include "plnmf/linalg.hpp"
#include "plnmf/metrics.hpp"
#include "plnmf/solver.hpp"
#include "plnmf/tiled.hpp"
#include "plnmf_gpu.h"

namespace plnmf {

// ---- the Algorithm::gpu branch of iterate(), as a function
void gpu_check(plnmf_status s) {
    switch (s) {
        case PLNMF_OK: return;
        case PLNMF_INVALID_ARGUMENT: throw std::invalid_argument(plnmf_last_error());
        case PLNMF_DOMAIN: throw std::domain_error(plnmf_last_error());
        default: throw std::runtime_error(plnmf_last_error());
    }
}

ConvergenceTrace iterate_gpu(const InputMatrix& a, FactorPair& factors, const SolverConfig& config,
                             Algorithm algorithm, plnmf_math math = PLNMF_MATH_EXACT) {
    // the reference's own argument checks first (solver.cpp:54-68), so a bad FactorPair or
    // tile is std::invalid_argument here too, never an out-of-bounds host access
    config.validate();
    const index_t k = config.rank;
    if (factors.w.rows() != a.rows() || factors.w.cols() != k || factors.ht.rows() != a.cols() ||
        factors.ht.cols() != k)
        throw std::invalid_argument("iterate: factor dimensions do not match input and rank");
    if (algorithm == Algorithm::tiled && (config.tile_size < 1 || config.tile_size > k))
        throw std::invalid_argument("iterate: tiled algorithm needs tile_size in [1, rank]");
    const plnmf_config c{config.rank, config.epsilon, config.max_iters, config.rel_tol,
                         config.seed, config.error_every, config.deterministic ? 1 : 0, config.tile_size};
    plnmf_gpu_engine* e = nullptr;  // a long-lived caller would cache this per InputMatrix
    if (a.is_sparse()) {
        const CsrMatrix& m = a.csr();
        gpu_check(plnmf_gpu_create_csr(0, m.rows, m.cols, m.nnz(), m.row_ptr.data(), m.col_idx.data(),
                                       m.values.data(), config.rank, &e));
    } else {
        gpu_check(plnmf_gpu_create_dense(0, a.rows(), a.cols(), a.dense().data(), config.rank, &e));
    }
    plnmf_status st = plnmf_gpu_set_math(e, math);
    if (st == PLNMF_OK && math == PLNMF_MATH_REFERENCE_ORDER)
        st = plnmf_gpu_set_reference_threads(e, omp_get_max_threads());
    std::vector<plnmf_trace_record> recs(std::max<index_t>(config.max_iters, 1));
    plnmf_trace tr{};
    tr.capacity = static_cast<int64_t>(recs.size());
    tr.records = recs.data();
    if (st == PLNMF_OK)
        st = plnmf_gpu_iterate_host(e, &c, algorithm == Algorithm::tiled ? PLNMF_ALGORITHM_TILED
                                                                         : PLNMF_ALGORITHM_REFERENCE,
                                    factors.w.data(), factors.ht.data(), &tr);
    plnmf_gpu_destroy(e);
    gpu_check(st);
    ConvergenceTrace out;
    out.initial_error = tr.initial_error;
    out.total_seconds = tr.total_seconds;
    out.update_macs = tr.update_macs;
    for (int64_t i = 0; i < tr.n_records; ++i) {
        const plnmf_phase_times& p = recs[i].phases;
        out.records.push_back({recs[i].iteration, recs[i].rel_error, recs[i].elapsed_s,
                               {p.precompute_h, p.update_h, p.precompute_w, p.update_w, p.phase1, p.phase2,
                                p.phase3, p.normalize, p.error_eval}});
    }
    const plnmf_phase_times& t = tr.totals;
    out.totals = {t.precompute_h, t.update_h, t.precompute_w, t.update_w, t.phase1, t.phase2, t.phase3,
                  t.normalize, t.error_eval};
    return out;
}

}  // namespace plnmf

using namespace plnmf;

namespace {

int g_failures = 0;

void report(const char* id, const std::string& name, bool pass, const std::string& detail) {
    std::printf("%s  %s: %s  [%s]\n", pass ? "PASS" : "FAIL", id, name.c_str(), detail.c_str());
    if (!pass) ++g_failures;
}

DenseMatrix random_dense(index_t rows, index_t cols, std::uint64_t seed, double lo, double hi) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(lo, hi);
    DenseMatrix m(rows, cols);
    for (index_t j = 0; j < cols; ++j)
        for (index_t i = 0; i < rows; ++i) m(i, j) = dist(rng);
    return m;
}

double min_element(const DenseMatrix& m) { return *std::min_element(m.data(), m.data() + m.size()); }

double max_norm_deviation(const DenseMatrix& w) {
    double worst = 0.0;
    for (index_t k = 0; k < w.cols(); ++k) {
        double s = 0.0;
        for (index_t v = 0; v < w.rows(); ++v) s += w(v, k) * w(v, k);
        worst = std::max(worst, std::abs(std::sqrt(s) - 1.0));
    }
    return worst;
}

bool same_bits(const DenseMatrix& a, const DenseMatrix& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), sizeof(double) * a.size()) == 0;
}

// criterion 5: run iterations one at a time through the drop-in, checking every iterate
void criterion_5() {
    const index_t v = 50, d = 40, k = 16, iters = 10;
    double worst_floor = 1e300, worst_norm = 0.0;
    for (std::uint64_t seed : {0ull, 1ull, 2ull}) {
        SolverConfig cfg;
        cfg.rank = k;
        cfg.seed = seed;
        cfg.max_iters = 1;
        cfg.rel_tol = 0.0;
        const InputMatrix a(random_dense(v, d, seed ^ 0x9e3779b97f4a7c15ull, 0.0, 1.0));
        for (index_t t : {0, 1, 2, 3, 4, 5, 8, 16}) {
            FactorPair f = init_factors(v, d, cfg);
            SolverConfig c = cfg;
            c.tile_size = t;
            for (index_t it = 0; it < iters; ++it) {
                iterate_gpu(a, f, c, t ? Algorithm::tiled : Algorithm::reference);
                worst_floor = std::min({worst_floor, min_element(f.w), min_element(f.ht)});
                worst_norm = std::max(worst_norm, max_norm_deviation(f.w));
            }
        }
    }
    char buf[96];
    std::snprintf(buf, sizeof(buf), "min element %.3e, worst |norm-1| %.3e", worst_floor, worst_norm);
    report("criterion 5", "clamp floor and unit-norm invariants (GPU)", worst_floor >= 1e-16 && worst_norm <= 1e-12, buf);
}

// criterion 6: the GPU counts the reference's MACs exactly, for both update paths
void criterion_6() {
    const index_t v = 30, d = 20, k = 12;
    SolverConfig cfg;
    cfg.rank = k;
    cfg.seed = 3;
    cfg.max_iters = 1;
    cfg.rel_tol = 0.0;
    const InputMatrix a(random_dense(v, d, 77, 0.0, 1.0));
    std::uint64_t ref_macs = 0;
    {
        FactorPair f = init_factors(v, d, cfg);
        ref_macs = iterate(a, f, cfg, Algorithm::reference).update_macs;
    }
    bool pass = ref_macs > 0;
    std::ostringstream detail;
    detail << "CPU reference " << ref_macs << " MACs; GPU";
    for (index_t t : {0, 1, 3, 4, 6, 12}) {
        FactorPair f = init_factors(v, d, cfg);
        SolverConfig c = cfg;
        c.tile_size = t;
        const std::uint64_t m = iterate_gpu(a, f, c, t ? Algorithm::tiled : Algorithm::reference).update_macs;
        detail << ' ' << m;
        if (m != ref_macs) pass = false;
    }
    report("criterion 6", "flop parity between update paths (GPU vs CPU)", pass, detail.str());
}

// criterion 7: objective behaviour through the drop-in
void criterion_7() {
    const MachineModel paper_machine{35ull << 20, 8};
    bool pass = true;
    std::ostringstream detail;
    for (index_t k : {8, 16}) {
        for (Algorithm alg : {Algorithm::reference, Algorithm::tiled}) {
            SolverConfig cfg;
            cfg.rank = k;
            cfg.seed = 17;
            cfg.max_iters = 100;
            cfg.rel_tol = 0.0;
            cfg.tile_size = alg == Algorithm::tiled ? best_integer_tile({100, 80, k}, paper_machine) : 0;
            const InputMatrix a(random_dense(100, 80, 1000 + k, 0.0, 1.0));
            FactorPair f = init_factors(100, 80, cfg);
            const ConvergenceTrace trace = iterate_gpu(a, f, cfg, alg);
            double prev = trace.initial_error;
            for (const TraceRecord& rec : trace.records) {
                if (rec.rel_error > prev + 1e-8) pass = false;
                prev = rec.rel_error;
            }
        }
    }
    {
        const index_t v = 100, d = 80, k = 16;
        const DenseMatrix w_true = random_dense(v, k, 21, 0.1, 1.0);
        const DenseMatrix ht_true = random_dense(d, k, 22, 0.1, 1.0);
        DenseMatrix prod(v, d);
        gemm(1.0, w_true.view(), false, ht_true.view(), true, 0.0, prod.view());
        const InputMatrix a(prod);
        SolverConfig cfg;
        cfg.rank = k;
        cfg.seed = 23;
        cfg.max_iters = 100;
        cfg.rel_tol = 0.0;
        cfg.tile_size = 4;
        FactorPair f = init_factors(v, d, cfg);
        const ConvergenceTrace trace = iterate_gpu(a, f, cfg, Algorithm::tiled);
        const double final_err = trace.records.back().rel_error;
        detail << "planted: initial " << trace.initial_error << " -> final " << final_err;
        if (!(final_err < 0.5 * trace.initial_error)) pass = false;
    }
    report("criterion 7", "objective non-increasing and planted-instance recovery (GPU)", pass, detail.str());
}

// the drop-in in reference-order mode is iterate() itself, bit for bit
void dropin_bitwise() {
    bool pass = true;
    std::ostringstream detail;
    detail << "threads=" << omp_get_max_threads();
    for (index_t t : {0, 1, 5, 16}) {
        SolverConfig cfg;
        cfg.rank = 16;
        cfg.seed = 4;
        cfg.max_iters = 25;
        cfg.rel_tol = 0.0;
        cfg.tile_size = t;
        std::mt19937_64 rng(99);
        std::uniform_real_distribution<double> u(0.1, 2.0);
        std::bernoulli_distribution keep(0.05);
        CsrMatrix m;
        m.rows = 700;
        m.cols = 400;
        m.row_ptr.assign(1, 0);
        for (index_t r = 0; r < m.rows; ++r) {
            for (index_t c = 0; c < m.cols; ++c)
                if (keep(rng)) {
                    m.col_idx.push_back(c);
                    m.values.push_back(u(rng));
                }
            m.row_ptr.push_back(static_cast<index_t>(m.col_idx.size()));
        }
        const InputMatrix a(m);
        const Algorithm alg = t ? Algorithm::tiled : Algorithm::reference;
        FactorPair cpu = init_factors(m.rows, m.cols, cfg);
        FactorPair gpu = cpu;
        const ConvergenceTrace tc = iterate(a, cpu, cfg, alg);
        const ConvergenceTrace tg = iterate_gpu(a, gpu, cfg, alg, PLNMF_MATH_REFERENCE_ORDER);
        bool same = same_bits(cpu.w, gpu.w) && same_bits(cpu.ht, gpu.ht) && tc.records.size() == tg.records.size() &&
                    tc.initial_error == tg.initial_error && tc.update_macs == tg.update_macs;
        for (size_t i = 0; same && i < tc.records.size(); ++i)
            same = tc.records[i].rel_error == tg.records[i].rel_error && tc.records[i].iteration == tg.records[i].iteration;
        detail << (t ? " pl-nmf(T=" + std::to_string(t) + ")" : std::string(" fast-hals")) << (same ? " ==" : " !=");
        pass = pass && same;
    }
    report("drop-in", "iterate_gpu(reference order) == iterate() bit for bit, 25 iterations", pass, detail.str());
}

// argument errors surface as the reference's exception types, before any device work
void dropin_errors() {
    bool pass = true;
    SolverConfig cfg;
    cfg.rank = 4;
    const InputMatrix a(random_dense(10, 8, 1, 0.0, 1.0));
    FactorPair wrong{DenseMatrix(9, 4), DenseMatrix(8, 4)};
    try {
        iterate_gpu(a, wrong, cfg, Algorithm::reference);
        pass = false;
    } catch (const std::invalid_argument&) {
    }
    FactorPair f = init_factors(10, 8, cfg);
    cfg.tile_size = 9;
    try {
        iterate_gpu(a, f, cfg, Algorithm::tiled);
        pass = false;
    } catch (const std::invalid_argument&) {
    }
    cfg.tile_size = 2;
    cfg.max_iters = -1;
    try {
        iterate_gpu(a, f, cfg, Algorithm::tiled);
        pass = false;
    } catch (const std::invalid_argument&) {
    }
    report("drop-in", "shape, tile and config errors are std::invalid_argument", pass, "3 cases");
}

}  // namespace

int main() {
    if (plnmf_gpu_device_count() < 1) {
        std::printf("SKIP  no CUDA device\n");
        return 0;
    }
    criterion_5();
    criterion_6();
    criterion_7();
    dropin_bitwise();
    dropin_errors();
    std::printf("%d failure(s)\n", g_failures);
    return g_failures;
}
