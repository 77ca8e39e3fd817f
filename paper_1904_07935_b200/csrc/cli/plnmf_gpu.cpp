// plnmf-gpu — the reference CLI's factorize / sweep-tiles / compare / model
// commands (proj/tools/plnmf.cpp:151-336) on the B200 engine, through the
// C-ABI only (include/plnmf_gpu.h).  Same options, the same report schema as
// report_to_json (proj/src/run_report.cpp:40-66) plus a "gpu" object, the
// same compare table and "max factor deviation" line.
//
//   plnmf-gpu factorize   --input A.mtx | --synthetic V,D,density,seed  --k K
//                         [--algorithm fast-hals|pl-nmf] [--tile auto|scan|gpu|N]
//                         [--max-iters N] [--tol x] [--epsilon x] [--seed s]
//                         [--error-every n] [--output path] [--format json|csv-trace]
//                         [--device i] [--math exact|fused|reference-order|tensor] [--threads n]
//   plnmf-gpu sweep-tiles (as factorize) [--grid 1,2,4,...]
//   plnmf-gpu compare     (as factorize): fast-hals and pl-nmf in lockstep on the GPU
//   plnmf-gpu model       --k K [--v V --d D | --input A.mtx]
//
// --tile auto / scan pick T from the reference's data-movement model
// (model_tile_size / best_integer_tile, proj/src/cost_model.cpp:114-142,
// restated below for the CLI only); --tile gpu measures the candidates on the
// device (plnmf_gpu_best_integer_tile).  --math reference-order with
// --threads n reproduces the reference run with n OpenMP threads bit for bit.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "plnmf_gpu.h"

namespace {

struct Options {
    std::string cmd, input, synthetic, algorithm = "pl-nmf", tile = "auto", output, format = "json", grid;
    std::string math = "exact";
    int64_t k = 0, max_iters = 100, error_every = 1, v = 0, d = 0;
    double tol = 1e-6, epsilon = 1e-16;
    uint64_t seed = 0, cache_bytes = 35ull << 20, word_bytes = 8;
    int device = 0, threads = 0;
    bool deterministic = false;
};

void check(plnmf_status s) {
    if (s == PLNMF_OK) return;
    const std::string msg = plnmf_last_error();
    if (s == PLNMF_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (s == PLNMF_DOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

// ---- the reference's movement model, for --tile auto/scan and the report's cost_model fields
struct Model {
    double c;  // cache words
    explicit Model(const Options& o) {
        if (o.word_bytes == 0) throw std::invalid_argument("MachineModel: word_bytes must be > 0");
        c = (double)(o.cache_bytes / o.word_bytes);
        if (c < 1) throw std::invalid_argument("MachineModel: cache must hold at least one word");
    }
    double c2() const { return 2.0 / std::sqrt(c); }
    double fasthals_total(double v, double d, double k) const {  // cost_model.cpp:43-60
        return k * (k * (v + d) * (1.0 + c2()) + 4.0 * v * d / std::sqrt(c) + 6.0 * v + 3.0 * d + 2.0 * k + 1.0);
    }
    double vol(double v, double k, double t) const {  // cost_model.cpp:93-112
        return v * (1.0 / t + c2()) * (k * k - k * t) + k * v * t;
    }
    double tile_size(int64_t k) const {  // cost_model.cpp:114-119
        if ((double)k <= c2()) throw std::domain_error("model_tile_size: K must exceed 2/sqrt(C)");
        return std::sqrt((double)k - c2());
    }
    int64_t best_integer(double v, int64_t k) const {  // cost_model.cpp:129-142
        int64_t best = 1;
        double bv = vol(v, k, 1);
        for (int64_t t = 2; t <= k; ++t) {
            const double x = vol(v, k, t);
            if (x < bv) { bv = x; best = t; }
        }
        return best;
    }
};

struct Input {
    plnmf_gpu_engine* e = nullptr;
    int64_t rows = 0, cols = 0, nnz = 0;
    double norm_sq = 0;
    ~Input() { if (e) plnmf_gpu_destroy(e); }
};

std::unique_ptr<Input> open_input(const Options& o) {
    auto in = std::make_unique<Input>();
    if (!o.synthetic.empty()) {
        std::stringstream ss(o.synthetic);
        std::string f[4];
        for (auto& x : f)
            if (!std::getline(ss, x, ',')) throw std::invalid_argument("--synthetic expects V,D,density,seed");
        check(plnmf_gpu_create_synthetic(o.device, std::stoll(f[0]), std::stoll(f[1]), std::stod(f[2]),
                                         std::stoull(f[3]), o.k, &in->e));
    } else {
        if (o.input.empty()) throw std::invalid_argument("--input (or --synthetic) is required");
        plnmf_mm* m = nullptr;
        check(plnmf_mm_read(o.input.c_str(), &m));
        const plnmf_status st = plnmf_gpu_create_mm(o.device, m, o.k, &in->e);
        plnmf_mm_free(m);
        check(st);
    }
    check(plnmf_gpu_input_info(in->e, &in->rows, &in->cols, &in->nnz, &in->norm_sq));
    if (o.math == "fused") check(plnmf_gpu_set_math(in->e, PLNMF_MATH_FUSED));
    else if (o.math == "reference-order") {
        check(plnmf_gpu_set_math(in->e, PLNMF_MATH_REFERENCE_ORDER));
        check(plnmf_gpu_set_reference_threads(in->e, o.threads > 0 ? o.threads : 1));
    } else if (o.math == "tensor") {
        check(plnmf_gpu_set_math(in->e, PLNMF_MATH_TENSOR));
    } else if (o.math != "exact") {
        throw std::invalid_argument("--math must be exact, fused, reference-order or tensor");
    }
    if (o.k > std::min(in->rows, in->cols))
        std::cerr << "warning: K = " << o.k << " exceeds min(V, D) = " << std::min(in->rows, in->cols) << "\n";
    return in;
}

plnmf_config config_of(const Options& o) {
    plnmf_config c;
    plnmf_config_default(&c);
    c.rank = o.k;
    c.epsilon = o.epsilon;
    c.max_iters = o.max_iters;
    c.rel_tol = o.tol;
    c.seed = o.seed;
    c.error_every = o.error_every;
    c.deterministic = o.deterministic ? 1 : 0;
    return c;
}

plnmf_algorithm algorithm_of(const Options& o) {
    if (o.algorithm == "fast-hals") return PLNMF_ALGORITHM_REFERENCE;
    if (o.algorithm == "pl-nmf") return PLNMF_ALGORITHM_TILED;
    throw std::invalid_argument("--algorithm must be fast-hals or pl-nmf");
}

struct Tile {
    int64_t size = 0;
    std::string provenance = "none";
};

// resolve_tile (proj/tools/plnmf.cpp:82-102) plus "gpu": measured on the device
Tile resolve_tile(const Options& o, const Input& in, plnmf_config cfg) {
    const Model model(o);
    if (o.tile == "auto") {
        const double t = model.tile_size(o.k);
        const int64_t lo = std::clamp<int64_t>((int64_t)std::floor(t), 1, o.k);
        const int64_t hi = std::clamp<int64_t>((int64_t)std::ceil(t), 1, o.k);
        int64_t pick = lo;
        if (hi != lo && model.vol((double)in.rows, o.k, hi) < model.vol((double)in.rows, o.k, lo)) pick = hi;
        return {pick, "model"};
    }
    if (o.tile == "scan") return {model.best_integer((double)in.rows, o.k), "brute-force"};
    if (o.tile == "gpu") {
        std::vector<double> ms(9);
        int32_t best = 0;
        check(plnmf_gpu_init_factors(in.e, &cfg));
        check(plnmf_gpu_best_integer_tile(in.e, &cfg, nullptr, 0, &best, ms.data()));
        return {best, "gpu-measured"};
    }
    int64_t t = 0;
    try {
        t = std::stoll(o.tile);
    } catch (...) {
        throw std::invalid_argument("--tile must be an integer, 'auto', 'scan' or 'gpu'");
    }
    if (t < 1 || t > o.k) throw std::invalid_argument("--tile must lie in [1, K]");
    return {t, "explicit"};
}

// ---- JSON (the schema of report_to_json, run_report.cpp:40-66, plus "gpu")
std::string num(double x) {
    if (!std::isfinite(x)) return "null";
    char b[40];
    std::snprintf(b, sizeof(b), "%.17g", x);
    return b;
}
std::string phases_json(const plnmf_phase_times& p, const std::string& ind) {
    std::ostringstream s;
    s << "{\n" << ind << "  \"error_eval\": " << num(p.error_eval) << ",\n" << ind << "  \"normalize\": "
      << num(p.normalize) << ",\n" << ind << "  \"phase1\": " << num(p.phase1) << ",\n" << ind << "  \"phase2\": "
      << num(p.phase2) << ",\n" << ind << "  \"phase3\": " << num(p.phase3) << ",\n" << ind << "  \"precompute_h\": "
      << num(p.precompute_h) << ",\n" << ind << "  \"precompute_w\": " << num(p.precompute_w) << ",\n" << ind
      << "  \"update_h\": " << num(p.update_h) << ",\n" << ind << "  \"update_w\": " << num(p.update_w) << "\n" << ind
      << "}";
    return s.str();
}

void emit_report(const Options& o, const Input& in, const Tile& tile, const plnmf_trace& tr,
                 const std::vector<plnmf_trace_record>& recs, double wall_s) {
    const Model model(o);
    std::ostringstream j;
    const double cells = (double)in.rows * (double)in.cols;
    char device_name[128] = "";
    check(plnmf_gpu_device_name(o.device, device_name, (int32_t)sizeof(device_name)));
    plnmf_gpu_stats st{};
    check(plnmf_gpu_get_stats(in.e, &st));
    const int64_t n = tr.n_records;
    if (o.format == "csv-trace") {  // write_run_report's csv_trace (run_report.cpp:95-103)
        j << "iteration,rel_error,elapsed_s\n";
        char b[96];
        for (int64_t i = 0; i < n; ++i) {
            std::snprintf(b, sizeof(b), "%lld,%.17g,%.9g\n", (long long)recs[i].iteration, recs[i].rel_error,
                          recs[i].elapsed_s);
            j << b;
        }
    } else if (o.format == "json") {
        j << "{\n  \"algorithm\": \"" << o.algorithm << "\",\n";
        j << "  \"config\": {\n    \"deterministic\": " << (o.deterministic ? "true" : "false")
          << ",\n    \"epsilon\": " << num(o.epsilon) << ",\n    \"error_every\": " << o.error_every
          << ",\n    \"max_iters\": " << o.max_iters << ",\n    \"rel_tol\": " << num(o.tol) << ",\n    \"seed\": "
          << o.seed << ",\n    \"threads\": " << (o.threads > 0 ? o.threads : 1) << "\n  },\n";
        j << "  \"cost_model\": {\n    \"fasthals_total\": "
          << num(model.fasthals_total((double)in.rows, (double)in.cols, (double)o.k));
        if (tile.size > 0) j << ",\n    \"vol_at_tile\": " << num(model.vol((double)in.rows, o.k, tile.size));
        j << "\n  },\n";
        j << "  \"final_rel_error\": " << num(n ? recs[n - 1].rel_error : tr.initial_error) << ",\n";
        const double iters = n ? (double)recs[n - 1].iteration : 0.0;
        j << "  \"gpu\": {\n    \"device\": \"" << device_name << "\",\n    \"sm_count\": " << st.sm_count
          << ",\n    \"math\": \"" << o.math << "\",\n    \"iterations_per_second\": "
          << num(iters > 0 ? iters / (tr.total_seconds - tr.totals.error_eval) : 0.0)
          << ",\n    \"kernel_launches\": " << st.kernel_launches << ",\n    \"device_bytes\": " << st.device_bytes
          << ",\n    \"w_update_plan\": " << st.w_plan << ",\n    \"h_update_plan\": " << st.h_plan
          << ",\n    \"wall_seconds\": " << num(wall_s) << "\n  },\n";
        j << "  \"initial_rel_error\": " << num(tr.initial_error) << ",\n";
        j << "  \"phase_seconds\": " << phases_json(tr.totals, "  ") << ",\n";
        j << "  \"problem\": {\n    \"d\": " << in.cols << ",\n    \"k\": " << o.k << ",\n    \"nnz\": " << in.nnz
          << ",\n    \"sparsity\": " << num(cells == 0.0 ? 0.0 : 1.0 - (double)in.nnz / cells) << ",\n    \"v\": "
          << in.rows << "\n  },\n";
        j << "  \"tile\": {\n    \"provenance\": \"" << tile.provenance << "\",\n    \"size\": " << tile.size
          << "\n  },\n";
        j << "  \"total_seconds\": " << num(tr.total_seconds) << ",\n  \"trace\": [";
        for (int64_t i = 0; i < n; ++i)
            j << (i ? "," : "") << "\n    {\n      \"elapsed_s\": " << num(recs[i].elapsed_s)
              << ",\n      \"iteration\": " << recs[i].iteration << ",\n      \"phases\": "
              << phases_json(recs[i].phases, "      ") << ",\n      \"rel_error\": " << num(recs[i].rel_error)
              << "\n    }";
        j << (n ? "\n  ]\n}\n" : "]\n}\n");
    } else {
        throw std::invalid_argument("--format must be json or csv-trace");
    }
    if (o.output.empty()) {
        std::cout << j.str();
    } else {
        std::ofstream f(o.output);
        if (!f) throw std::runtime_error("write_run_report: cannot open " + o.output);
        f << j.str();
        if (!f) throw std::runtime_error("write_run_report: write failed for " + o.output);
    }
}

int run_factorize(const Options& o) {
    auto in = open_input(o);
    const plnmf_algorithm alg = algorithm_of(o);
    plnmf_config cfg = config_of(o);
    Tile tile;
    if (alg == PLNMF_ALGORITHM_TILED) {
        tile = resolve_tile(o, *in, cfg);
        cfg.tile_size = tile.size;
    }
    std::vector<plnmf_trace_record> recs((size_t)std::max<int64_t>(1, cfg.max_iters));
    plnmf_trace tr{};
    tr.capacity = (int64_t)recs.size();
    tr.records = recs.data();
    const auto t0 = std::chrono::steady_clock::now();
    check(plnmf_gpu_init_factors(in->e, &cfg));
    check(plnmf_gpu_iterate(in->e, &cfg, alg, &tr));
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    emit_report(o, *in, tile, tr, recs, wall);
    return 0;
}

std::vector<int64_t> parse_grid(const Options& o, const Input& in, const plnmf_config& cfg) {
    std::set<int64_t> grid;
    if (!o.grid.empty()) {
        std::stringstream ss(o.grid);
        std::string item;
        while (std::getline(ss, item, ',')) {
            const int64_t t = std::stoll(item);
            if (t < 1 || t > o.k) throw std::invalid_argument("--grid entries must lie in [1, K]");
            grid.insert(t);
        }
    } else {
        for (int64_t t = 1; t <= o.k; t *= 2) grid.insert(t);
        grid.insert(o.k);
        Options a = o;
        a.tile = "auto";
        grid.insert(resolve_tile(a, in, cfg).size);
    }
    return {grid.begin(), grid.end()};
}

// run_sweep_tiles (proj/tools/plnmf.cpp:236-282): iterate() per tile size from the
// same seeded factors, seconds = total - error_eval; the model's predicted movement
// beside it, and the device's own pick
int run_sweep_tiles(const Options& o) {
    if (algorithm_of(o) != PLNMF_ALGORITHM_TILED) throw std::invalid_argument("sweep-tiles requires --algorithm pl-nmf");
    auto in = open_input(o);
    const Model model(o);
    plnmf_config cfg = config_of(o);
    Options a = o;
    a.tile = "auto";
    const int64_t recommended = resolve_tile(a, *in, cfg).size;
    const std::vector<int64_t> grid = parse_grid(o, *in, cfg);
    std::printf("%6s  %12s  %16s  %s\n", "tile", "seconds", "predicted_vol", "");
    std::vector<double> seconds(grid.size()), predicted(grid.size());
    std::vector<plnmf_trace_record> recs((size_t)std::max<int64_t>(1, cfg.max_iters));
    for (size_t i = 0; i < grid.size(); ++i) {
        cfg.tile_size = grid[i];
        plnmf_trace tr{};
        tr.capacity = (int64_t)recs.size();
        tr.records = recs.data();
        check(plnmf_gpu_init_factors(in->e, &cfg));
        check(plnmf_gpu_iterate(in->e, &cfg, PLNMF_ALGORITHM_TILED, &tr));
        seconds[i] = tr.total_seconds - tr.totals.error_eval;
        predicted[i] = model.vol((double)in->rows, o.k, grid[i]);
        std::printf("%6lld  %12.4f  %16.0f  %s\n", (long long)grid[i], seconds[i], predicted[i],
                    grid[i] == recommended ? "<- model" : "");
    }
    const auto measured = std::min_element(seconds.begin(), seconds.end()) - seconds.begin();
    const auto pred = std::min_element(predicted.begin(), predicted.end()) - predicted.begin();
    std::printf("fastest on this GPU: T=%lld\n", (long long)grid[measured]);
    if (std::abs(measured - pred) > 1)
        std::cerr << "warning: measured optimum (T=" << grid[measured]
                  << ") is more than one grid step from the predicted optimum (T=" << grid[pred] << ")\n";
    if (!o.output.empty()) {
        std::ofstream f(o.output);
        if (!f) throw std::runtime_error("cannot open " + o.output);
        f << "tile,seconds,predicted_vol,model_recommended\n";
        for (size_t i = 0; i < grid.size(); ++i)
            f << grid[i] << ',' << seconds[i] << ',' << predicted[i] << ',' << (grid[i] == recommended ? 1 : 0) << '\n';
        if (!f) throw std::runtime_error("write failed for " + o.output);
    }
    return 0;
}

double factor_deviation(const std::vector<double>& ref, const std::vector<double>& other) {
    double md = 0.0, mr = 0.0;  // metrics.cpp:129-143
    for (size_t i = 0; i < ref.size(); ++i) {
        md = std::max(md, std::abs(ref[i] - other[i]));
        mr = std::max(mr, std::abs(ref[i]));
    }
    if (mr == 0.0) return md == 0.0 ? 0.0 : INFINITY;
    return md / mr;
}

// run_compare (proj/tools/plnmf.cpp:284-336): fast-hals and pl-nmf in lockstep from
// shared factors, each on its own GPU engine; errors and factor deviations per iteration
int run_compare(const Options& o) {
    auto ref = open_input(o);
    auto til = open_input(o);
    plnmf_config cfg = config_of(o);
    const Tile tile = resolve_tile(o, *ref, cfg);
    cfg.tile_size = tile.size;
    check(plnmf_gpu_init_factors(ref->e, &cfg));
    check(plnmf_gpu_init_factors(til->e, &cfg));
    auto eval = [&](Input& in) {
        double out3[3];
        check(plnmf_gpu_evaluate_error(in.e, out3));
        return out3[1];
    };
    check(plnmf_gpu_precompute_w_products(ref->e));
    std::printf("initial rel error: %.12e\n", eval(*ref));
    const std::string head = "pl-nmf(T=" + std::to_string(tile.size) + ")";
    std::printf("%6s  %18s  %18s  %12s  %12s\n", "iter", "fast-hals", head.c_str(), "dev(W)", "dev(Ht)");
    const size_t wn = (size_t)(ref->rows * o.k), hn = (size_t)(ref->cols * o.k);
    std::vector<double> w1(wn), h1(hn), w2(wn), h2(hn);
    double max_dev = 0.0;
    for (int64_t it = 1; it <= o.max_iters; ++it) {
        for (auto [in, alg] : {std::pair{ref.get(), PLNMF_ALGORITHM_REFERENCE}, std::pair{til.get(), PLNMF_ALGORITHM_TILED}}) {
            check(plnmf_gpu_precompute_h_products(in->e));
            check(plnmf_gpu_update_h(in->e, &cfg, alg));
            check(plnmf_gpu_precompute_w_products(in->e));
            check(plnmf_gpu_update_w(in->e, &cfg, alg));
        }
        check(plnmf_gpu_get_factors(ref->e, w1.data(), h1.data()));
        check(plnmf_gpu_get_factors(til->e, w2.data(), h2.data()));
        const double dw = factor_deviation(w1, w2), dh = factor_deviation(h1, h2);
        max_dev = std::max({max_dev, dw, dh});
        const double e1 = eval(*ref), e2 = eval(*til);
        std::printf("%6lld  %18.12e  %18.12e  %12.3e  %12.3e\n", (long long)it, e1, e2, dw, dh);
    }
    std::printf("max factor deviation: %.3e\n", max_dev);
    return 0;
}

// run_model (proj/tools/plnmf.cpp:171-213), the tile-size lines
int run_model(const Options& o) {
    int64_t v = o.v, d = o.d;
    if (!o.input.empty()) {
        plnmf_mm* m = nullptr;
        check(plnmf_mm_read(o.input.c_str(), &m));
        plnmf_mm_info(m, &v, &d, nullptr, nullptr);
        plnmf_mm_free(m);
    }
    if (v < 1) throw std::invalid_argument("model: provide --v (or --input)");
    if (o.k < 1) throw std::invalid_argument("model: provide --k");
    const Model model(o);
    std::printf("shape: V=%lld D=%s K=%lld\n", (long long)v, d >= 1 ? std::to_string(d).c_str() : "?",
                (long long)o.k);
    std::printf("analytic tile size: %.2f\n", model.tile_size(o.k));
    const int64_t best = model.best_integer((double)v, o.k);
    std::printf("best integer tile: %lld\n", (long long)best);
    if (d >= 1) std::printf("total movement per iteration: %.6e\n", model.fasthals_total((double)v, (double)d, (double)o.k));
    return 0;
}

Options parse(int argc, char** argv) {
    if (argc < 2) throw std::invalid_argument("usage: plnmf-gpu factorize|sweep-tiles|compare|model [options]");
    Options o;
    o.cmd = argv[1];
    std::map<std::string, std::string*> str = {
        {"--input", &o.input},   {"--synthetic", &o.synthetic}, {"--algorithm", &o.algorithm},
        {"--tile", &o.tile},     {"--output", &o.output},       {"--format", &o.format},
        {"--grid", &o.grid},     {"--math", &o.math}};
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--deterministic") { o.deterministic = true; continue; }
        if (i + 1 >= argc) throw std::invalid_argument("option " + a + " needs a value");
        const std::string val = argv[++i];
        if (str.count(a)) *str[a] = val;
        else if (a == "--k") o.k = std::stoll(val);
        else if (a == "--max-iters") o.max_iters = std::stoll(val);
        else if (a == "--error-every") o.error_every = std::stoll(val);
        else if (a == "--v") o.v = std::stoll(val);
        else if (a == "--d") o.d = std::stoll(val);
        else if (a == "--tol") o.tol = std::stod(val);
        else if (a == "--epsilon") o.epsilon = std::stod(val);
        else if (a == "--seed") o.seed = std::stoull(val);
        else if (a == "--cache-bytes") o.cache_bytes = std::stoull(val);
        else if (a == "--word-bytes") o.word_bytes = std::stoull(val);
        else if (a == "--device") o.device = std::stoi(val);
        else if (a == "--threads") o.threads = std::stoi(val);
        else throw std::invalid_argument("unknown option " + a);
    }
    if (o.k < 1 && o.cmd != "model") throw std::invalid_argument("--k is required");
    return o;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Options o = parse(argc, argv);
        if (o.cmd == "factorize") return run_factorize(o);
        if (o.cmd == "sweep-tiles") return run_sweep_tiles(o);
        if (o.cmd == "compare") return run_compare(o);
        if (o.cmd == "model") return run_model(o);
        throw std::invalid_argument("unknown command " + o.cmd);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
