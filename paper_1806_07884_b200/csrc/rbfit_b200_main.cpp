// rbfit-b200 -- the reference's batch front end (gen-synthetic | fit | eval |
// bench-blocks, proj/tools/rbfit_main.cpp) on the GPU path.
//
// Same subcommands, options, stdout keys and stderr lines as the reference, so
// scripts written against `rbfit` run unchanged: result lines go to stdout in
// the same key-value / TSV form, timings and warnings to stderr, files are the
// reference's formats (rbfit_io.cpp).  The fit, the evaluation and the error
// report run on the GPU through rbfit_b200::fit / evaluate_model /
// error_report.  The GPU path has no column blocks: --ram-budget and
// --block-size are accepted and reported as one block (block-size = M), and
// bench-blocks times one GPU fit per requested size (the system is
// block-invariant, so max_rel_diff compares the repeated GPU assemblies).
// Option parsing is hand-written (CLI11 is not available); usage errors exit
// with CLI11's codes (104 conversion, 105 validation, 106 required, 108
// excludes, 109 extras).
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "rbfit_gpu.hpp"

extern "C" {  // librbg_datagen.so: the reference's generators, bit for bit (data.cpp:76-124)
void dg_halton(std::uint64_t start, std::uint64_t count, int dims, double* out);
void dg_grid_refs(double x0, double y0, double x1, double y1, std::uint64_t nx, std::uint64_t ny, double* out);
void dg_franke(const double* xy, std::uint64_t n, double* out);
}

namespace {

using namespace rbfit_b200;

struct UsageError : std::runtime_error {
    int code;
    UsageError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

std::string fmt(double v) {
    char buf[32];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, res.ptr);
}

std::string fmt_ms(double seconds) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.1f", seconds * 1e3);
    return buf;
}

template <typename T>
T parse_num(const std::string& opt, const std::string& text) {
    T v{};
    const auto res = std::from_chars(text.data(), text.data() + text.size(), v);
    if (res.ec != std::errc() || res.ptr != text.data() + text.size())
        throw UsageError(104, "Could not convert: " + opt + " = " + text);
    return v;
}

// Parsed options of one subcommand: "--name value", "--name=value", flags.
struct Args {
    std::map<std::string, std::string> values;
    std::map<std::string, bool> flags;
    bool has(const std::string& k) const { return values.count(k) != 0; }
    const std::string& get(const std::string& k) const { return values.at(k); }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& options,
           const std::vector<std::string>& flag_names, const std::map<std::string, std::string>& aliases) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string tok = argv[i];
        std::string val;
        bool has_val = false;
        if (const auto eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = tok.substr(eq + 1);
            tok = tok.substr(0, eq);
            has_val = true;
        }
        if (const auto al = aliases.find(tok); al != aliases.end()) tok = al->second;
        if (std::find(flag_names.begin(), flag_names.end(), tok) != flag_names.end()) {
            a.flags[tok] = true;
            continue;
        }
        if (std::find(options.begin(), options.end(), tok) == options.end())
            throw UsageError(109, "The following arguments were not expected: " + std::string(argv[i]));
        if (!has_val) {
            if (i + 1 >= argc) throw UsageError(114, tok + ": 1 required TEXT missing");
            val = argv[++i];
        }
        a.values[tok] = val;
    }
    return a;
}

void require(const Args& a, const std::string& k) {
    if (!a.has(k)) throw UsageError(106, k + " is required");
}

const std::vector<std::string> kFitOptions = {"--in", "--kernel", "--alpha", "--refs-grid", "--refs-file",
                                              "--ram-budget", "--block-size"};

struct Problem {
    PointCloud cloud;
    std::vector<Point2> refs;
    KernelSpec kernel{KernelFamily::wendland_3_1, 1.0};
    FitOptions options;
};

// rbfit_main.cpp:86-125: centred cloud, grid over its bounding box or a
// reference file shifted into the same frame
Problem load_problem(const Args& a) {
    require(a, "--in");
    require(a, "--alpha");
    if (a.has("--refs-grid") && a.has("--refs-file"))
        throw UsageError(108, "--refs-grid excludes --refs-file");
    if (!a.has("--refs-grid") && !a.has("--refs-file"))
        throw std::invalid_argument("one of --refs-grid or --refs-file is required");
    Problem p;
    p.cloud = center_cloud(load_xyz(a.get("--in")));
    if (a.has("--refs-grid")) {
        const std::string& text = a.get("--refs-grid");
        auto count = [&](const std::string& part) {
            std::size_t v = 0;
            const auto res = std::from_chars(part.data(), part.data() + part.size(), v);
            if (res.ec != std::errc() || res.ptr != part.data() + part.size() || v == 0)
                throw std::invalid_argument("--refs-grid: '" + text + "' is not a positive count or NXxNY shape");
            return v;
        };
        std::size_t nx, ny;
        if (const auto sep = text.find_first_of("xX"); sep == std::string::npos) {
            const std::size_t c = count(text);
            nx = static_cast<std::size_t>(std::llround(std::sqrt(static_cast<double>(c))));
            if (nx * nx != c)
                throw std::invalid_argument("grid reference count " + std::to_string(c) +
                                            " is not a perfect square; give per-axis counts instead");
            ny = nx;
        } else {
            nx = count(text.substr(0, sep));
            ny = count(text.substr(sep + 1));
        }
        Point2 lo = p.cloud.points[0], hi = lo;  // bounding_box (geometry.hpp:29-39)
        for (const Point2& q : p.cloud.points) {
            lo.x = std::min(lo.x, q.x);
            lo.y = std::min(lo.y, q.y);
            hi.x = std::max(hi.x, q.x);
            hi.y = std::max(hi.y, q.y);
        }
        p.refs.resize(nx * ny);
        dg_grid_refs(lo.x, lo.y, hi.x, hi.y, nx, ny, &p.refs[0].x);
    } else {
        p.refs = load_ref_points(a.get("--refs-file"));
        for (Point2& r : p.refs) {
            r.x -= p.cloud.offset.x;
            r.y -= p.cloud.offset.y;
        }
    }
    p.options.poly = a.flags.count("--poly") != 0;
    if (a.has("--ram-budget")) p.options.ram_budget_bytes = parse_num<std::size_t>("--ram-budget", a.get("--ram-budget"));
    if (a.has("--block-size")) p.options.block_size = parse_num<std::size_t>("--block-size", a.get("--block-size"));
    const std::string kname = a.has("--kernel") ? a.get("--kernel") : "wendland-3-1";
    p.kernel = KernelSpec(kernel_from_name(kname), parse_num<double>("--alpha", a.get("--alpha")));
    return p;
}

int cmd_gen(const Args& a) {
    require(a, "--out");
    std::size_t n = 1089;
    if (a.has("--count")) {
        const double v = parse_num<double>("--count", a.get("--count"));
        if (!(v > 0) || v != std::floor(v)) throw UsageError(105, "--count: Value " + a.get("--count") + " should be a positive number");
        n = static_cast<std::size_t>(v);
    }
    PointCloud c;
    c.points.resize(n);
    dg_halton(1, n, 2, &c.points[0].x);  // halton_2d skips index 0 (data.cpp:95)
    c.values.resize(n);
    dg_franke(&c.points[0].x, n, c.values.data());
    save_xyz(c, a.get("--out"));
    std::cout << "points " << c.size() << "\n";
    return 0;
}

int cmd_fit(const Args& a) {
    require(a, "--model");
    Problem p = load_problem(a);
    FitReport report;
    const Model model = fit(p.cloud, std::move(p.refs), p.kernel, p.options, &report);
    save_model(model, a.get("--model"));
    const ErrorReport errors = error_report(model, p.cloud, report.design_nnz);
    std::cout << "points " << p.cloud.size() << "\n"
              << "refs " << model.refs.size() << "\n"
              << "kernel " << kernel_name(model.kernel.family()) << "\n"
              << "alpha " << fmt(model.kernel.alpha()) << "\n"
              << "block-size " << report.plan.block_size << "\n"
              << "n-blocks " << report.plan.n_blocks << "\n"
              << "design-nnz " << report.design_nnz << "\n"
              << "density-pct " << fmt(errors.density_pct.value()) << "\n"
              << "mae " << fmt(errors.mean_absolute_error) << "\n"
              << "deviation " << fmt(errors.deviation_of_error) << "\n"
              << "mean-relative-error-pct " << fmt(errors.mean_relative_error_pct) << "\n"
              << "empty-support-refs " << report.empty_support_refs.size() << "\n"
              << "ridge-lambda " << fmt(report.ridge_lambda) << "\n";
    std::cerr << "index: " << fmt_ms(report.index_seconds) << " ms\n"
              << "assembly: " << fmt_ms(report.assembly_seconds) << " ms\n"
              << "gram+solve: " << fmt_ms(report.gram_solve_seconds) << " ms\n"
              << "peak-memory: " << report.peak_bytes << " bytes\n";
    for (const auto& w : report.warnings) std::cerr << "warning: " << w << "\n";
    return 0;
}

int cmd_eval(const Args& a) {
    require(a, "--model");
    require(a, "--in");
    require(a, "--out");
    const Model model = load_model(a.get("--model"));
    const EvalPoints input = load_eval_points(a.get("--in"));
    std::cout << "points " << input.points.size() << "\n";
    if (input.has_values) {
        PointCloud cloud{input.points, input.values, {0.0, 0.0}};
        const ErrorReport errors = error_report(model, cloud);
        std::vector<double> pred(cloud.size());
        for (std::size_t i = 0; i < cloud.size(); ++i) pred[i] = cloud.values[i] + errors.signed_errors[i];
        write_signed_errors(cloud, pred, a.get("--out"));
        std::cout << "mae " << fmt(errors.mean_absolute_error) << "\n"
                  << "deviation " << fmt(errors.deviation_of_error) << "\n"
                  << "mean-relative-error-pct " << fmt(errors.mean_relative_error_pct) << "\n";
    } else {
        const std::vector<double> f = evaluate_model(model, input.points);
        std::string text;
        for (std::size_t i = 0; i < f.size(); ++i)
            text += fmt(input.points[i].x) + ' ' + fmt(input.points[i].y) + ' ' + fmt(f[i]) + '\n';
        std::ofstream out(a.get("--out"));
        if (!out) throw std::runtime_error("cannot open " + a.get("--out") + " for writing");
        out << text;
    }
    return 0;
}

int cmd_bench(const Args& a) {
    require(a, "--block-sizes");
    std::vector<std::size_t> sizes;
    {
        const std::string& t = a.get("--block-sizes");
        std::size_t s = 0;
        while (s <= t.size()) {
            const std::size_t e = std::min(t.find(',', s), t.size());
            sizes.push_back(parse_num<std::size_t>("--block-sizes", t.substr(s, e - s)));
            s = e + 1;
        }
    }
    Problem p = load_problem(a);
    Device dev(p.options.device);
    const auto t0 = std::chrono::steady_clock::now();
    std::cerr << "index: " << fmt_ms(0.0) << " ms\n";
    std::cout << "block_size\tn_blocks\tassembly_ms\tgram_solve_ms\ttotal_ms\tmae\tmax_rel_diff\n";
    std::optional<NormalSystem> first;
    double worst = 0.0;
    for (const std::size_t bs : sizes) {
        BuildStats st;
        const NormalSystem sys = build_normal_system(p.cloud, p.refs, p.kernel, p.options.poly, &st, &dev);
        const auto ts = std::chrono::steady_clock::now();
        SolveDiag diag;
        const Weights w = solve_weights(sys, &diag, &dev);
        const double solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
        Model model{p.kernel, p.refs, w.c, w.poly, p.cloud.offset};
        const ErrorReport er = error_report(model, p.cloud, std::nullopt, &dev);
        double diff = 0.0;
        if (!first) {
            first = sys;
        } else {  // max |delta| / max |value| over values and rhs (acceptance_main.cpp:118-125)
            double dmax = 0.0, vmax = 0.0;
            for (std::size_t e = 0; e < sys.values.size(); ++e) {
                dmax = std::max(dmax, std::abs(sys.values[e] - first->values[e]));
                vmax = std::max(vmax, std::abs(first->values[e]));
            }
            for (std::size_t i = 0; i < sys.rhs.size(); ++i) {
                dmax = std::max(dmax, std::abs(sys.rhs[i] - first->rhs[i]));
                vmax = std::max(vmax, std::abs(first->rhs[i]));
            }
            diff = vmax > 0.0 ? dmax / vmax : 0.0;
        }
        worst = std::max(worst, diff);
        std::cout << bs << '\t' << 1 << '\t' << fmt_ms(st.assembly_seconds) << '\t' << fmt_ms(solve_s) << '\t'
                  << fmt_ms(st.assembly_seconds + solve_s) << '\t' << fmt(er.mean_absolute_error) << '\t'
                  << fmt(diff) << '\n';
    }
    (void)t0;
    if (worst > 1e-10)
        throw std::runtime_error("normal system drifted across block sizes: max relative difference " + fmt(worst));
    return 0;
}

void usage(std::ostream& os) {
    os << "Out-of-core RBF surface fitting with compactly supported kernels (GPU path)\n"
          "Usage: rbfit-b200 SUBCOMMAND [OPTIONS]\n"
          "Subcommands:\n"
          "  gen-synthetic  sample Franke's surface at Halton points (-n/--count N, --out PATH)\n"
          "  fit            fit a model to scattered data (--in, --kernel, --alpha, --refs-grid|--refs-file,\n"
          "                 --poly, --ram-budget, --block-size, --model)\n"
          "  eval           evaluate a fitted model at query points (--model, --in, --out)\n"
          "  bench-blocks   compare block sizes on one fitting problem (fit options + --block-sizes a,b,c)\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage(std::cerr);
        std::cerr << "A subcommand is required\n";
        return 106;
    }
    const std::string sub = argv[1];
    if (sub == "-h" || sub == "--help") {
        usage(std::cout);
        return 0;
    }
    try {
        try {
            if (sub == "gen-synthetic") return cmd_gen(parse(argc, argv, 2, {"--count", "--out"}, {}, {{"-n", "--count"}}));
            if (sub == "fit") {
                auto opts = kFitOptions;
                opts.push_back("--model");
                return cmd_fit(parse(argc, argv, 2, opts, {"--poly"}, {}));
            }
            if (sub == "eval") return cmd_eval(parse(argc, argv, 2, {"--model", "--in", "--out"}, {}, {}));
            if (sub == "bench-blocks") {
                auto opts = kFitOptions;
                opts.push_back("--block-sizes");
                return cmd_bench(parse(argc, argv, 2, opts, {"--poly"}, {}));
            }
            throw UsageError(109, "The following argument was not expected: " + sub);
        } catch (const UsageError& e) {
            std::cerr << e.what() << "\nRun with --help for more information.\n";
            return e.code;
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
