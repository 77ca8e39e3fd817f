// Host-side pieces of the C-ABI that need no GPU: SolverConfig defaults and
// validation, plan_tiles, the bit-identical init_factors, the synthetic CSR
// generator, and the thread-local error channel.
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"
#include "plnmf_gpu.h"

namespace plnmf {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void validate_config(const plnmf_config& c) {
    // proj/src/config.cpp:7-15, same messages
    if (c.rank < 1) throw std::invalid_argument("SolverConfig: rank must be >= 1");
    if (!(c.epsilon > 0.0)) throw std::invalid_argument("SolverConfig: epsilon must be > 0");
    if (c.max_iters < 0) throw std::invalid_argument("SolverConfig: max_iters must be >= 0");
    if (c.rel_tol < 0.0) throw std::invalid_argument("SolverConfig: rel_tol must be >= 0");
    if (c.error_every < 1) throw std::invalid_argument("SolverConfig: error_every must be >= 1");
    if (c.tile_size < 0 || c.tile_size > c.rank)
        throw std::invalid_argument("SolverConfig: tile_size must be in [1, rank] (0 = auto)");
}

void init_factors_host(int64_t v, int64_t d, const plnmf_config& cfg, double* w, double* ht) {
    // proj/src/solver.cpp:20-28,43-51: W first, then Ht, column-major fill
    validate_config(cfg);
    if (v < 1 || d < 1) throw std::invalid_argument("init_factors: dimensions must be >= 1");
    std::mt19937_64 rng(cfg.seed);
    const double lo = cfg.epsilon;
    auto fill = [&](double* p, int64_t n) {
        for (int64_t i = 0; i < n; ++i) {
            const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
            p[i] = lo + (1.0 - lo) * u;  // built with -ffp-contract=off: no FMA
        }
    };
    fill(w, v * cfg.rank);
    fill(ht, d * cfg.rank);
}

// ---- synthetic CSR -------------------------------------------------
namespace {

inline uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// uniform on (0, 1]
inline double open_uniform(uint64_t& s) { return (static_cast<double>(splitmix64(s) >> 11) + 1.0) * 0x1.0p-53; }

// Walks row r's Bernoulli(density) cells by geometric gaps; calls emit(col, value).
template <class F>
void synth_row(int64_t r, int64_t cols, double density, uint64_t seed, F&& emit) {
    uint64_t s = seed ^ (0xD1B54A32D192ED03ULL * (static_cast<uint64_t>(r) + 1));
    splitmix64(s);
    if (density <= 0.0) return;
    const bool dense = density >= 1.0;
    const double inv_log_q = dense ? 0.0 : 1.0 / std::log1p(-density);
    int64_t c = -1;
    for (;;) {
        int64_t gap = 0;
        if (!dense) {
            const double g = std::floor(std::log(open_uniform(s)) * inv_log_q);
            if (g >= static_cast<double>(cols)) break;
            gap = static_cast<int64_t>(g);
        }
        c += 1 + gap;
        if (c >= cols) break;
        const double u = static_cast<double>(splitmix64(s) >> 11) * 0x1.0p-53;
        const float value = static_cast<float>(0.1 + 1.9 * u);  // U(0.1, 2.0), fp32-representable
        emit(c, static_cast<double>(value));
    }
}

template <class F>
void parallel_rows(int64_t rows, F&& f) {
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    if (rows < 4096) nt = 1;
    std::vector<std::thread> pool;
    const int64_t chunk = (rows + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const int64_t a = t * chunk, b = std::min<int64_t>(rows, a + chunk);
        if (a >= b) break;
        pool.emplace_back([a, b, &f] {
            for (int64_t r = a; r < b; ++r) f(r);
        });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

void synth_csr(int64_t rows, int64_t cols, double density, uint64_t seed, int64_t* row_ptr,
               int64_t* col_idx, double* values, int64_t* nnz) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("synth_csr: negative dimension");
    if (!(density >= 0.0) || density > 1.0) throw std::invalid_argument("synth_csr: density must be in [0, 1]");
    if (!col_idx) {
        std::vector<int64_t> counts(rows, 0);
        parallel_rows(rows, [&](int64_t r) {
            int64_t n = 0;
            synth_row(r, cols, density, seed, [&](int64_t, double) { ++n; });
            counts[r] = n;
        });
        row_ptr[0] = 0;
        for (int64_t r = 0; r < rows; ++r) row_ptr[r + 1] = row_ptr[r] + counts[r];
        *nnz = row_ptr[rows];
        return;
    }
    parallel_rows(rows, [&](int64_t r) {
        int64_t e = row_ptr[r];
        synth_row(r, cols, density, seed, [&](int64_t c, double v) {
            col_idx[e] = c;
            values[e] = v;
            ++e;
        });
    });
}

}  // namespace plnmf

// ---- C-ABI: host helpers ---------------------------------------------------------------
using plnmf::guarded;

extern "C" {

const char* plnmf_last_error(void) { return plnmf::g_last_error.c_str(); }
int32_t plnmf_gpu_abi_version(void) { return PLNMF_GPU_ABI_VERSION; }

void plnmf_config_default(plnmf_config* c) {
    // proj/include/plnmf/config.hpp:11-22
    c->rank = 2;
    c->epsilon = 1e-16;
    c->max_iters = 100;
    c->rel_tol = 1e-6;
    c->seed = 0;
    c->error_every = 1;
    c->deterministic = 0;
    c->tile_size = 0;
}

plnmf_status plnmf_config_validate(const plnmf_config* c) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("plnmf_config_validate: null config");
        plnmf::validate_config(*c);
    });
}

plnmf_status plnmf_plan_tiles(int64_t k, int64_t tile, int64_t* begins, int64_t* ends, int64_t* gamma) {
    return guarded([&] {
        // proj/src/tiling.cpp:8-18
        if (k < 1) throw std::invalid_argument("plan_tiles: k must be >= 1");
        if (tile < 1 || tile > k) throw std::invalid_argument("plan_tiles: tile size must be in [1, k]");
        int64_t n = 0;
        for (int64_t b = 0; b < k; b += tile, ++n)
            if (begins) {
                begins[n] = b;
                ends[n] = std::min(k, b + tile);
            }
        if (gamma) *gamma = n;
    });
}

plnmf_status plnmf_init_factors(int64_t v, int64_t d, const plnmf_config* cfg, double* w, double* ht) {
    return guarded([&] {
        if (!cfg || !w || !ht) throw std::invalid_argument("plnmf_init_factors: null argument");
        plnmf::init_factors_host(v, d, *cfg, w, ht);
    });
}

plnmf_status plnmf_synth_csr(int64_t rows, int64_t cols, double density, uint64_t seed,
                             int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* nnz) {
    return guarded([&] {
        if (!row_ptr || (col_idx && !values) || (!col_idx && !nnz))
            throw std::invalid_argument("plnmf_synth_csr: null argument");
        plnmf::synth_csr(rows, cols, density, seed, row_ptr, col_idx, values, nnz);
    });
}

}  // extern "C"
