// rbfit_gpu.cpp -- reference-shaped C++ API over the C ABI (see rbfit_gpu.hpp).
#include "rbfit_gpu.hpp"

#include <array>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>

#include "rbg.h"

namespace rbfit_b200 {

namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

[[noreturn]] void raise(rbg_status st, const std::string& msg) {
    switch (st) {
        case RBG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case RBG_DOMAIN_ERROR: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(rbg_status st, rbg_ctx* ctx) {
    if (st != RBG_OK) raise(st, rbg_last_error(ctx));
}

int family_id(KernelFamily f) { return static_cast<int>(f); }

struct NameEntry {
    KernelFamily family;
    std::string_view name;
};
constexpr NameEntry kNames[] = {  // kernel.cpp:13-18 + the wendland-3-2 extension
    {KernelFamily::wendland_3_0, "wendland-3-0"},
    {KernelFamily::wendland_3_1, "wendland-3-1"},
    {KernelFamily::wendland_3_3, "wendland-3-3"},
    {KernelFamily::wendland_3_2, "wendland-3-2"},
};

const double* flat(std::span<const Point2> p) { return reinterpret_cast<const double*>(p.data()); }

// Device context: the caller's or a temporary one.
struct Using {
    std::unique_ptr<Device> own;
    Device* dev;
    explicit Using(Device* d, int index = 0) : dev(d) {
        if (!dev) {
            own = std::make_unique<Device>(index);
            dev = own.get();
        }
    }
    rbg_ctx* ctx() const { return dev->ctx(); }
};

void set_centres(rbg_ctx* ctx, std::span<const Point2> refs, const KernelSpec& kernel) {
    check(rbg_set_centres(ctx, 2, flat(refs), refs.size(), family_id(kernel.family()),
                          kernel.alpha()),
          ctx);
}

}  // namespace

KernelFamily kernel_from_name(std::string_view name) {
    for (const auto& e : kNames)
        if (e.name == name) return e.family;
    std::string msg = "unknown kernel '" + std::string(name) + "'; expected one of:";
    for (const auto& e : kNames) msg += " " + std::string(e.name);
    throw std::invalid_argument(msg);
}

std::string_view kernel_name(KernelFamily family) {
    for (const auto& e : kNames)
        if (e.family == family) return e.name;
    throw std::invalid_argument("unknown kernel family");
}

KernelSpec::KernelSpec(KernelFamily family, double alpha) : family_(family), alpha_(alpha) {
    if (!(alpha > 0.0) || !std::isfinite(alpha))
        throw std::invalid_argument("kernel shape parameter must be positive and finite");
}

double KernelSpec::evaluate(double r) const {
    double out = 0.0;
    const rbg_status st = rbg_kernel_value(family_id(family_), alpha_, r, &out);
    if (st == RBG_DOMAIN_ERROR)
        throw std::domain_error("kernel evaluate: radius must be finite and non-negative");
    if (st != RBG_OK) throw std::invalid_argument("kernel evaluate: bad kernel");
    return out;
}

Device::Device(int device) {
    const rbg_status st = rbg_create(device, &ctx_);
    if (st != RBG_OK)
        raise(st, "cannot create a GPU context on device " + std::to_string(device));
}

Device::~Device() {
    if (ctx_) rbg_destroy(ctx_);
}

void Device::set_stream(void* s) { check(rbg_set_stream(ctx_, s), ctx_); }

double NormalSystem::at(std::size_t i, std::size_t j) const {
    if (i > j) std::swap(i, j);
    const auto b = cols.begin() + static_cast<std::ptrdiff_t>(row_ptr[i]);
    const auto e = cols.begin() + static_cast<std::ptrdiff_t>(row_ptr[i + 1]);
    const auto it = std::lower_bound(b, e, static_cast<std::uint32_t>(j));
    return (it != e && *it == j) ? values[static_cast<std::size_t>(it - cols.begin())] : 0.0;
}

PointIndex::PointIndex(std::vector<Point2> points) : points_(std::move(points)) {
    if (points_.empty()) throw std::invalid_argument("point index requires at least one point");  // kdtree.cpp:11-17
    if (points_.size() > 0xffffffffull) throw std::invalid_argument("point index limited to 2^32-1 points");
    for (std::size_t i = 0; i < points_.size(); ++i)
        if (!std::isfinite(points_[i].x) || !std::isfinite(points_[i].y))
            throw std::invalid_argument("non-finite coordinate at point index " + std::to_string(i));
}

namespace {

// The caller's hook runs the all-reduce on the context's stream (rbfit_gpu.hpp).
void run_allreduce(rbg_ctx* ctx, const AllReduce& allreduce) {
    if (!allreduce) return;
    double* buf = nullptr;
    std::uint64_t count = 0;
    void* stream = nullptr;
    check(rbg_system_device(ctx, &buf, &count), ctx);
    check(rbg_get_stream(ctx, &stream), ctx);
    allreduce(buf, count, stream);
}

void check_plan(const BlockPlan& plan, std::size_t m) {  // solver.cpp:137-144
    if (plan.m_total != m)
        throw std::invalid_argument("build_normal_system: plan was made for a different reference count");
    if (plan.block_size == 0 || plan.block_size > m || plan.n_blocks == 0)
        throw std::invalid_argument("build_normal_system: malformed block plan");
}

NormalSystem build_on_device(std::span<const Point2> pts, std::span<const double> values,
                             std::span<const Point2> refs, const KernelSpec& kernel, bool poly,
                             BuildStats* stats, Device* device, const AllReduce& allreduce, bool validate) {
    Using u(device);
    rbg_ctx* ctx = u.ctx();
    BuildStats local{};
    auto t0 = Clock::now();
    set_centres(ctx, refs, kernel);
    check(rbg_set_poly(ctx, poly ? 1 : 0), ctx);
    local.index_seconds = seconds_since(t0);
    t0 = Clock::now();
    check(rbg_assemble(ctx, flat(pts), values.data(), pts.size(), 0, validate ? 1 : 0), ctx);
    run_allreduce(ctx, allreduce);
    rbg_pattern_info info{};
    check(rbg_get_pattern_info(ctx, &info), ctx);
    const std::size_t m = refs.size();
    NormalSystem sys;
    sys.side = m;
    sys.row_ptr.resize(m + 1);
    sys.cols.resize(info.nnz_upper);
    sys.values.resize(info.nnz_upper);
    sys.rhs.resize(m);
    std::vector<double> hits(m);
    std::uint64_t design_nnz = 0;
    check(rbg_get_system(ctx, sys.values.data(), sys.rhs.data(), hits.data(), &design_nnz), ctx);
    local.assembly_seconds = seconds_since(t0);
    check(rbg_get_pattern(ctx, sys.row_ptr.data(), sys.cols.data()), ctx);
    for (std::size_t j = 0; j < m; ++j)
        if (hits[j] == 0.0) sys.empty_support_refs.push_back(static_cast<std::uint32_t>(j));
    if (poly) {  // solver.cpp:189-207, 238-262: side = m + T
        const std::size_t T = 3;
        sys.poly = true;
        sys.border_atp.resize(T * m);
        sys.border_ptp.resize(T * T);
        sys.border_pth.resize(T);
        check(rbg_get_border(ctx, sys.border_atp.data(), sys.border_ptp.data(), sys.border_pth.data()), ctx);
    }
    local.design_nnz = design_nnz;
    local.peak_bytes = (info.nnz_upper + 2 * m) * sizeof(double);
    if (stats) *stats = local;
    return sys;
}

}  // namespace

NormalSystem build_normal_system(const PointIndex& index, std::span<const double> values,
                                 std::span<const Point2> refs, const KernelSpec& kernel,
                                 const BlockPlan& plan, bool poly, BuildStats* stats, Device* device,
                                 const AllReduce& allreduce) {
    if (values.size() != index.size())  // solver.cpp:133-134
        throw std::invalid_argument("build_normal_system: value count does not match points");
    if (refs.empty()) throw std::invalid_argument("build_normal_system: no reference points");
    check_plan(plan, refs.size());
    // the index already validated its points (kdtree.cpp:14-17)
    return build_on_device(index.points(), values, refs, kernel, poly, stats, device, allreduce, false);
}

NormalSystem build_normal_system(const PointCloud& cloud, std::span<const Point2> refs,
                                 const KernelSpec& kernel, const BlockPlan& plan, bool poly,
                                 BuildStats* stats, Device* device, const AllReduce& allreduce) {
    if (cloud.values.size() != cloud.points.size())
        throw std::invalid_argument("build_normal_system: value count does not match points");
    if (refs.empty()) throw std::invalid_argument("build_normal_system: no reference points");
    check_plan(plan, refs.size());
    return build_on_device(cloud.points, cloud.values, refs, kernel, poly, stats, device, allreduce, true);
}

NormalSystem build_normal_system(const PointCloud& cloud, std::span<const Point2> refs,
                                 const KernelSpec& kernel, bool poly, BuildStats* stats, Device* device,
                                 const AllReduce& allreduce) {
    if (cloud.values.size() != cloud.points.size())  // solver.cpp:135-136
        throw std::invalid_argument("build_normal_system: value count does not match points");
    if (refs.empty()) throw std::invalid_argument("build_normal_system: no reference points");
    return build_on_device(cloud.points, cloud.values, refs, kernel, poly, stats, device, allreduce, true);
}

Weights solve_weights(const NormalSystem& sys, SolveDiag* diag, Device* device) {
    if (sys.side == 0 || sys.rhs.size() != sys.side || sys.row_ptr.size() != sys.side + 1 ||
        sys.values.size() != sys.cols.size())
        throw std::invalid_argument("solve_weights: malformed normal system");
    if (!device)
        throw std::invalid_argument(
            "solve_weights: pass the Device that assembled the system (the pattern lives there)");
    rbg_ctx* ctx = device->ctx();
    rbg_pattern_info info{};
    check(rbg_get_pattern_info(ctx, &info), ctx);
    if (info.m != sys.side || info.nnz_upper != sys.values.size())
        throw std::invalid_argument("solve_weights: system does not match the device's pattern");
    check(rbg_set_poly(ctx, sys.poly ? 1 : 0), ctx);
    check(rbg_set_system(ctx, sys.values.data(), sys.rhs.data(), nullptr), ctx);
    if (sys.poly)
        check(rbg_set_border(ctx, sys.border_atp.data(), sys.border_ptp.data(), sys.border_pth.data()), ctx);
    Weights w;
    w.c.resize(sys.side);
    rbg_solve_diag d{};
    check(rbg_solve(ctx, nullptr, w.c.data(), &d), ctx);
    if (sys.poly) {  // Weights::poly (solver.cpp:327-328)
        std::array<double, 4> a{};
        check(rbg_get_poly_solution(ctx, a.data()), ctx);
        w.poly = std::array<double, 3>{a[0], a[1], a[2]};
    }
    if (diag) *diag = SolveDiag{d.ridge_lambda, d.ridge_shift, d.attempts, d.iterations, d.rel_residual};
    return w;
}

Model fit(const PointCloud& cloud, std::vector<Point2> refs, const KernelSpec& kernel,
          const FitOptions& options, FitReport* report) {
    if (cloud.size() == 0) throw std::invalid_argument("fit: empty point cloud");  // solver.cpp:403-406
    if (cloud.values.size() != cloud.points.size())
        throw std::invalid_argument("fit: cloud value count mismatch");
    if (refs.empty()) throw std::invalid_argument("fit: no reference points");

    FitReport local{};
    if (cloud.size() < refs.size())
        local.warnings.push_back(
            "fewer data points than reference points; the least-squares system is "
            "underdetermined");
    const std::size_t m = refs.size();
    local.plan = BlockPlan{m, m, 1, options.ram_budget_bytes, options.prec_bytes, true};

    Using u(options.engine, options.device);
    rbg_ctx* ctx = u.ctx();
    auto t0 = Clock::now();
    set_centres(ctx, refs, kernel);
    check(rbg_set_poly(ctx, options.poly ? 1 : 0), ctx);
    local.index_seconds = seconds_since(t0);
    t0 = Clock::now();
    check(rbg_assemble(ctx, flat(cloud.points), cloud.values.data(), cloud.size(), 0, 1), ctx);
    run_allreduce(ctx, options.allreduce);
    std::vector<double> hits(m);
    std::uint64_t design_nnz = 0;
    check(rbg_get_system(ctx, nullptr, nullptr, hits.data(), &design_nnz), ctx);
    local.assembly_seconds = seconds_since(t0);
    t0 = Clock::now();
    std::vector<double> c(m);
    rbg_solve_options so{options.tol, options.max_iter, options.solve_method, options.preconditioner};
    rbg_solve_diag d{};
    std::optional<std::array<double, 3>> poly;
    const std::size_t unknowns = m + (options.poly ? 3 : 0);
    // the orthogonal re-pass over the data (solver.cpp:345-397); false: not finite
    const auto repass = [&]() -> bool {
        std::vector<double> w(unknowns);
        int ok = 0;
        check(rbg_least_squares_repass(ctx, flat(cloud.points), cloud.values.data(), cloud.size(), w.data(), &ok),
              ctx);
        if (!ok) return false;
        std::copy(w.begin(), w.begin() + static_cast<std::ptrdiff_t>(m), c.begin());
        if (options.poly) poly = std::array<double, 3>{w[m], w[m + 1], w[m + 2]};
        return true;
    };
    const rbg_status st = rbg_solve(ctx, &so, c.data(), &d);
    if (st == RBG_RUNTIME_ERROR && unknowns <= rbg_repass_max_unknowns()) {
        // solver.cpp:439-451: every ridge rung failed; a rank-deficient design rethrows
        const std::string why = rbg_last_error(ctx);
        if (!repass()) throw std::runtime_error(why);
        d = rbg_solve_diag{};
        local.warnings.push_back(
            "normal equations unsolvable; weights recovered by an orthogonal re-pass over the data");
    } else {
        check(st, ctx);
        if (options.poly) {
            std::array<double, 4> a{};
            check(rbg_get_poly_solution(ctx, a.data()), ctx);
            poly = std::array<double, 3>{a[0], a[1], a[2]};
        }
    }
    if (d.ridge_lambda > 0.0) {  // solver.cpp:452-464
        if (unknowns > rbg_repass_max_unknowns())
            throw std::runtime_error("normal equations numerically singular (ridge lambda " +
                                     std::to_string(d.ridge_lambda) +
                                     "); the orthogonal re-pass (solver.cpp:345-397) is limited to " +
                                     std::to_string(rbg_repass_max_unknowns()) + " unknowns on the GPU path");
        if (repass()) {
            d.ridge_lambda = 0.0;
            d.ridge_shift = 0.0;
            local.warnings.push_back(
                "normal equations numerically singular; weights recovered by an orthogonal re-pass over "
                "the data");
        }
    }
    local.gram_solve_seconds = seconds_since(t0);
    local.design_nnz = design_nnz;
    for (std::size_t j = 0; j < m; ++j)
        if (hits[j] == 0.0) local.empty_support_refs.push_back(static_cast<std::uint32_t>(j));
    local.ridge_lambda = d.ridge_lambda;
    local.ridge_shift = d.ridge_shift;
    local.iterations = d.iterations;
    rbg_pattern_info info{};
    check(rbg_get_pattern_info(ctx, &info), ctx);
    local.peak_bytes = (info.nnz_upper + 2 * m) * sizeof(double);

    Model model{kernel, std::move(refs), std::move(c), poly, cloud.offset};
    if (report) *report = std::move(local);
    return model;
}

std::vector<BenchRow> bench_block_sizes(const PointCloud& cloud, std::vector<Point2> refs,
                                        const KernelSpec& kernel, const FitOptions& options,
                                        std::span<const std::size_t> block_sizes, double* index_seconds) {
    if (block_sizes.empty()) throw std::invalid_argument("bench_block_sizes: no block sizes given");  // solver.cpp:484-487
    if (cloud.size() == 0) throw std::invalid_argument("bench_block_sizes: empty cloud");
    if (refs.empty()) throw std::invalid_argument("bench_block_sizes: no reference points");
    const auto t0 = Clock::now();
    const PointIndex index(cloud.points);
    if (index_seconds) *index_seconds = seconds_since(t0);
    Using u(options.engine, options.device);
    const std::size_t m = refs.size();
    std::vector<BenchRow> rows;
    NormalSystem baseline;
    for (const std::size_t requested : block_sizes) {
        const std::size_t mb = std::clamp<std::size_t>(requested, 1, m);
        const BlockPlan plan{m, mb, (m + mb - 1) / mb, options.ram_budget_bytes, options.prec_bytes, false};
        BuildStats stats{};
        NormalSystem sys = build_normal_system(index, cloud.values, refs, kernel, plan, options.poly, &stats,
                                               u.dev, options.allreduce);
        const auto ts = Clock::now();
        Weights w = solve_weights(sys, nullptr, u.dev);
        const double solve_seconds = seconds_since(ts);
        const Model model{kernel, refs, std::move(w.c), w.poly, cloud.offset};
        const ErrorReport er = error_report(model, cloud, stats.design_nnz, u.dev);
        BenchRow row;
        row.block_size = mb;
        row.n_blocks = plan.n_blocks;
        row.assembly_seconds = stats.assembly_seconds;
        row.gram_solve_seconds = stats.gram_seconds + solve_seconds;
        row.mae = er.mean_absolute_error;
        if (rows.empty()) {
            baseline = std::move(sys);
        } else {
            double worst = 0.0;
            const auto update = [&worst](double a, double b) {
                const double mag = std::max(std::abs(a), std::abs(b));
                if (mag > 0.0) worst = std::max(worst, std::abs(a - b) / mag);
            };
            for (std::size_t i = 0; i < baseline.values.size(); ++i) update(baseline.values[i], sys.values[i]);
            for (std::size_t i = 0; i < baseline.rhs.size(); ++i) update(baseline.rhs[i], sys.rhs[i]);
            row.max_rel_diff = worst;
        }
        rows.push_back(row);
    }
    return rows;
}

std::vector<double> evaluate_model(const Model& model, std::span<const Point2> queries,
                                   Device* device) {
    if (model.refs.empty()) throw std::invalid_argument("model has no reference points");
    if (model.weights.size() != model.refs.size())
        throw std::invalid_argument("model weight count does not match reference count");
    Using u(device);
    set_centres(u.ctx(), model.refs, model.kernel);
    check(rbg_set_model_poly(u.ctx(), model.poly ? model.poly->data() : nullptr), u.ctx());  // model.cpp:65-68
    std::vector<Point2> shifted;
    std::span<const Point2> q = queries;
    if (model.offset.x != 0.0 || model.offset.y != 0.0) {  // model.cpp:192-194
        shifted.resize(queries.size());
        for (std::size_t i = 0; i < queries.size(); ++i)
            shifted[i] = {queries[i].x + -model.offset.x, queries[i].y + -model.offset.y};
        q = shifted;
    }
    std::vector<double> f(q.size());
    check(rbg_evaluate(u.ctx(), model.weights.data(), flat(q), q.size(), f.data()), u.ctx());
    return f;
}

ErrorReport error_report(const Model& model, const PointCloud& cloud,
                         std::optional<std::size_t> design_nnz, Device* device) {
    if (cloud.size() == 0) throw std::invalid_argument("error_report: empty cloud");
    if (cloud.values.size() != cloud.points.size())
        throw std::invalid_argument("error_report: cloud value count mismatch");
    if (model.weights.size() != model.refs.size())
        throw std::invalid_argument("model weight count does not match reference count");
    Using u(device);
    set_centres(u.ctx(), model.refs, model.kernel);
    check(rbg_set_model_poly(u.ctx(), model.poly ? model.poly->data() : nullptr), u.ctx());
    const Point2 delta{cloud.offset.x - model.offset.x, cloud.offset.y - model.offset.y};
    std::vector<Point2> shifted;
    std::span<const Point2> q = cloud.points;
    if (delta.x != 0.0 || delta.y != 0.0) {  // model.cpp:202-204
        shifted.resize(cloud.size());
        for (std::size_t i = 0; i < cloud.size(); ++i)
            shifted[i] = {cloud.points[i].x + delta.x, cloud.points[i].y + delta.y};
        q = shifted;
    }
    ErrorReport rep;
    rep.signed_errors.resize(cloud.size());
    rbg_error_stats st{};
    check(rbg_error_report(u.ctx(), model.weights.data(), flat(q), cloud.values.data(), cloud.size(),
                           &st, rep.signed_errors.data()),
          u.ctx());
    rep.mean_absolute_error = st.mean_absolute_error;
    rep.deviation_of_error = st.deviation_of_error;
    rep.mean_relative_error_pct = st.mean_relative_error_pct;
    rep.rms_error = st.rms_error;
    rep.max_abs_error = st.max_abs_error;
    if (design_nnz)
        rep.density_pct = 100.0 * static_cast<double>(*design_nnz) /
                          (static_cast<double>(cloud.size()) * static_cast<double>(model.refs.size()));
    return rep;
}

}  // namespace rbfit_b200
