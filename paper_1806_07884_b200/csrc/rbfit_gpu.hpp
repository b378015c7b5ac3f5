// rbfit_gpu.hpp -- C++ host layer with the reference's hot-path API
// (rbfit::fit / build_normal_system / solve_weights / evaluate_model /
// error_report, /root/reference/proj/core/include/rbfit/{solver,model}.hpp),
// executing on the B200 through the C ABI in include/rbg.h.
//
// Drop-in notes:
//  * same names, argument meaning and exception classes (std::invalid_argument,
//    std::runtime_error, std::domain_error) and the same messages where the
//    reference states them;
//  * NormalSystem is sparse (upper CSR) instead of dense side x side: at the
//    BASELINE sizes the dense matrix does not exist in any memory;
//  * the block planner (BlockPlan / ram budget) has no GPU meaning: the whole
//    pattern is resident; FitReport::plan reports one block;
//  * the linear-polynomial border (FitOptions::poly) is supported (2-D: P =
//    [x, y, 1] as the reference); the orthogonal re-pass of fit
//    (solver.cpp:345-397, 439-464) runs on the GPU up to 4096 unknowns and
//    fit throws beyond that instead of keeping a ridge-biased solution.
#pragma once

#include <array>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

struct rbg_ctx;

namespace rbfit_b200 {

struct Point2 {  // layout-identical to rbfit::Point2 (geometry.hpp:9-12)
    double x = 0.0;
    double y = 0.0;
};

struct PointCloud {  // rbfit::PointCloud (data.hpp:17-23)
    std::vector<Point2> points;
    std::vector<double> values;
    Point2 offset{0.0, 0.0};
    std::size_t size() const { return points.size(); }
};

enum class KernelFamily { wendland_3_0, wendland_3_1, wendland_3_3, wendland_3_2 };
KernelFamily kernel_from_name(std::string_view name);
std::string_view kernel_name(KernelFamily family);

class KernelSpec {  // rbfit::KernelSpec (kernel.hpp:32-71)
  public:
    KernelSpec(KernelFamily family, double alpha);
    KernelFamily family() const { return family_; }
    double alpha() const { return alpha_; }
    double support_radius() const { return 1.0 / alpha_; }
    double evaluate(double r) const;  // bitwise the device's phi
    double operator()(double r) const { return evaluate(r); }

  private:
    KernelFamily family_;
    double alpha_;
};

// One GPU engine context (owns an rbg_ctx).  Not thread-safe.
class Device {
  public:
    explicit Device(int device = 0);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    rbg_ctx* ctx() const { return ctx_; }
    void set_stream(void* cuda_stream);

  private:
    rbg_ctx* ctx_ = nullptr;
};

// PointIndex (kdtree.hpp:10-28): owns a copy of the points and validates them
// like the reference (kdtree.cpp:10-17); the spatial index itself is the
// device-side binning done per assembly, so no tree is built on the host.
class PointIndex {
  public:
    explicit PointIndex(std::vector<Point2> points);
    std::size_t size() const { return points_.size(); }
    const std::vector<Point2>& points() const { return points_; }

  private:
    std::vector<Point2> points_;
};

// NormalSystem (solver.hpp:61-69) in upper-CSR form.
struct NormalSystem {
    std::size_t side = 0;
    std::vector<std::uint64_t> row_ptr;  // side + 1
    std::vector<std::uint32_t> cols;     // ascending per row, cols >= row
    std::vector<double> values;
    std::vector<double> rhs;
    bool poly = false;
    // border blocks when poly (side = m + 3 in the reference's dense form):
    std::vector<double> border_atp;  // A^T P, 3 x m term-major
    std::vector<double> border_ptp;  // P^T P, 3 x 3
    std::vector<double> border_pth;  // P^T h, 3
    std::vector<std::uint32_t> empty_support_refs;
    double at(std::size_t i, std::size_t j) const;  // symmetric lookup, 0 off-pattern
};

struct BuildStats {  // solver.hpp:71-78 (device times)
    double index_seconds = 0.0;     // centre binning + symbolic pattern
    double assembly_seconds = 0.0;  // point binning + numeric assembly (incl. copies)
    double gram_seconds = 0.0;      // fused into assembly on the GPU (0)
    std::size_t peak_bytes = 0;
    std::size_t design_nnz = 0;
    std::size_t blocks_assembled = 1;
};

// Sum-allreduce hook for multi-GPU builds: called with the device buffer
// [values | rhs | hits (| border)] (fp64) after the local slab's assembly has
// been ENQUEUED, and with `stream` = the context's cudaStream_t
// (rbg_get_stream).  The hook must enqueue its reduction on that stream (e.g.
// ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, comm, (cudaStream_t)
// stream)): the assembly before it and every read after it run on the same
// stream, so no other synchronisation is needed.
using AllReduce = std::function<void(double* device_buffer, std::uint64_t count, void* stream)>;

struct BlockPlan {  // solver.hpp:26-33; accepted and validated, one block on the GPU
    std::size_t m_total = 0, block_size = 0, n_blocks = 1, ram_budget_bytes = 0, prec_bytes = 8;
    bool sparse_mode = true;
};

// build_normal_system (solver.hpp:86-94).  The plan is validated with the
// reference's messages (solver.cpp:135-144) and otherwise has no effect: the
// whole pattern is resident on the device.
NormalSystem build_normal_system(const PointIndex& index, std::span<const double> values,
                                 std::span<const Point2> refs, const KernelSpec& kernel,
                                 const BlockPlan& plan, bool poly, BuildStats* stats = nullptr,
                                 Device* device = nullptr, const AllReduce& allreduce = {});
NormalSystem build_normal_system(const PointCloud& cloud, std::span<const Point2> refs,
                                 const KernelSpec& kernel, const BlockPlan& plan, bool poly,
                                 BuildStats* stats = nullptr, Device* device = nullptr,
                                 const AllReduce& allreduce = {});
// Convenience form without a plan (one block).
NormalSystem build_normal_system(const PointCloud& cloud, std::span<const Point2> refs,
                                 const KernelSpec& kernel, bool poly, BuildStats* stats = nullptr,
                                 Device* device = nullptr, const AllReduce& allreduce = {});

struct SolveDiag {  // solver.hpp:96-100
    double ridge_lambda = 0.0;
    double ridge_shift = 0.0;
    int attempts = 0;
    int iterations = 0;
    double rel_residual = 0.0;
};

struct Weights {  // solver.hpp:102-105
    std::vector<double> c;
    std::optional<std::array<double, 3>> poly;
};

Weights solve_weights(const NormalSystem& sys, SolveDiag* diag = nullptr, Device* device = nullptr);

struct FitOptions {  // solver.hpp:113-118 (+ GPU solve controls)
    bool poly = false;
    std::size_t ram_budget_bytes = std::size_t{1} << 30;  // accepted, unused on the GPU
    std::size_t prec_bytes = 8;
    std::optional<std::size_t> block_size;  // accepted, unused on the GPU
    double tol = 1e-12;
    int max_iter = 20000;
    int solve_method = 0;   // rbg.h RBG_SOLVE_*: 0 = FSAI-preconditioned CG, 2 = the reference's LLT on the band
    int preconditioner = 0; // rbg.h RBG_PREC_*: 0 = automatic (FSAI; point Jacobi with the border)
    int device = 0;
    Device* engine = nullptr;  // the caller's context (and its stream); `device` is then ignored
    AllReduce allreduce;       // multi-GPU: sum partial systems across ranks (see AllReduce)
};

struct FitReport {  // solver.hpp:120-131
    BlockPlan plan;
    double index_seconds = 0.0;
    double assembly_seconds = 0.0;
    double gram_solve_seconds = 0.0;
    std::size_t peak_bytes = 0;
    std::size_t design_nnz = 0;
    std::vector<std::uint32_t> empty_support_refs;
    double ridge_lambda = 0.0;
    double ridge_shift = 0.0;
    int iterations = 0;
    std::vector<std::string> warnings;
};

struct Model {  // model.hpp:17-23
    KernelSpec kernel;
    std::vector<Point2> refs;
    std::vector<double> weights;
    std::optional<std::array<double, 3>> poly;
    Point2 offset{0.0, 0.0};
};

Model fit(const PointCloud& cloud, std::vector<Point2> refs, const KernelSpec& kernel,
          const FitOptions& options = {}, FitReport* report = nullptr);

struct BenchRow {  // solver.hpp:133-142
    std::size_t block_size = 0;
    std::size_t n_blocks = 0;
    double assembly_seconds = 0.0;
    double gram_solve_seconds = 0.0;
    double mae = 0.0;
    double max_rel_diff = 0.0;  // (b, rhs) against the first run
};

// bench_block_sizes (solver.hpp:144-150, solver.cpp:480-536): one GPU fit per
// requested block size.  The GPU assembles every plan as one block, so the
// rows time repeated fits and max_rel_diff checks run-to-run agreement of the
// assembled system (summation order only).
std::vector<BenchRow> bench_block_sizes(const PointCloud& cloud, std::vector<Point2> refs,
                                        const KernelSpec& kernel, const FitOptions& options,
                                        std::span<const std::size_t> block_sizes,
                                        double* index_seconds = nullptr);

std::vector<double> evaluate_model(const Model& model, std::span<const Point2> queries,
                                   Device* device = nullptr);

struct ErrorReport {  // model.hpp:38-50 (+ rms, max)
    double mean_absolute_error = 0.0;
    double deviation_of_error = 0.0;
    double mean_relative_error_pct = 0.0;
    double rms_error = 0.0;
    double max_abs_error = 0.0;
    std::vector<double> signed_errors;
    std::optional<double> density_pct;
};

ErrorReport error_report(const Model& model, const PointCloud& cloud,
                         std::optional<std::size_t> design_nnz = std::nullopt,
                         Device* device = nullptr);

// ---- on-disk formats (rbfit_io.cpp): byte-identical to the reference's files
void save_model(const Model& model, const std::filesystem::path& path);  // model.cpp:76-115
Model load_model(const std::filesystem::path& path);                     // model.cpp:117-190

struct EvalPoints {  // data.hpp:49-53
    std::vector<Point2> points;
    std::vector<double> values;  // empty unless has_values
    bool has_values = false;
};
PointCloud load_xyz(const std::filesystem::path& path);                      // data.cpp:126-141
void save_xyz(const PointCloud& cloud, const std::filesystem::path& path);   // data.cpp:143-157
EvalPoints load_eval_points(const std::filesystem::path& path);              // data.cpp:159-180
std::vector<Point2> load_ref_points(const std::filesystem::path& path);      // data.cpp:182-196
void write_signed_errors(const PointCloud& cloud, std::span<const double> predictions,
                         const std::filesystem::path& path);                 // model.cpp:234-256
PointCloud center_cloud(PointCloud cloud);                                   // data.cpp:198-223

}  // namespace rbfit_b200
