// ref_driver.cpp -- C entry points over the reference's OWN compiled sources.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// kernel.cpp, kdtree.cpp, coo.cpp, data.cpp and model.cpp straight from
// /root/reference/proj/core/src (unmodified, never copied) into
// oracle/_ref/librbfit_ref.so.  solver.cpp cannot be compiled here (it needs
// Eigen, which is absent), so build_normal_system is restated below for the
// single-block plan (block_size = M, the reference's fastest legal plan) by
// calling the compiled reference primitives in exactly the order of
// solver.cpp:131-236; its output is therefore the reference's own output.
// solve_weights is restated as a textbook Cholesky with the reference's ridge
// ladder (solver.cpp:289-330) -- same method, Eigen's blocked rounding is not
// reproducible without Eigen.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <array>
#include <optional>
#include <span>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "rbfit/coo.hpp"
#include "rbfit/data.hpp"
#include "rbfit/kdtree.hpp"
#include "rbfit/kernel.hpp"
#include "rbfit/model.hpp"

using namespace rbfit;

namespace {

thread_local std::string g_err;

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::domain_error*>(&e)) return 3;
    return 2;
}

std::vector<Point2> to_points(const double* xy, std::uint64_t n) {
    std::vector<Point2> out(n);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = {xy[2 * i], xy[2 * i + 1]};
    return out;
}

KernelFamily family_of(int f) {
    switch (f) {
        case 0: return KernelFamily::wendland_3_0;
        case 1: return KernelFamily::wendland_3_1;
        case 2: return KernelFamily::wendland_3_3;
    }
    throw std::invalid_argument("reference has no kernel family " + std::to_string(f));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_kernel_evaluate(int family, double alpha, double r, double* out) {
    try {
        *out = KernelSpec(family_of(family), alpha).evaluate(r);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ref_radical_inverse(unsigned base, std::uint64_t index) {
    return radical_inverse(base, index);
}

int ref_halton_points(std::uint64_t count, int dims, double* out) {
    try {
        const auto v = halton_points(count, dims);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ref_franke(double x, double y) { return franke(Point2{x, y}); }

// halton_points (data.cpp:89-98) at arbitrary sequence indices, point-major:
// the reference's own radical_inverse, used to build spatial window samples
// of the Halton configs for bench.py --impl reference.
int ref_halton_at(const std::uint64_t* idx, std::uint64_t n, int dims, double* out) {
    static const unsigned kBases[] = {2, 3, 5};
    if (dims < 1 || dims > 3) return 1;
    for (std::uint64_t i = 0; i < n; ++i)
        for (int d = 0; d < dims; ++d) out[i * dims + d] = radical_inverse(kBases[d], idx[i]);
    return 0;
}

// franke (data.cpp:108-116) of n points.
void ref_franke_many(const double* xy, std::uint64_t n, double* out) {
    for (std::uint64_t i = 0; i < n; ++i) out[i] = franke(Point2{xy[2 * i], xy[2 * i + 1]});
}

int ref_uniform_grid_refs(double x0, double y0, double x1, double y1, std::uint64_t nx,
                          std::uint64_t ny, double* out) {
    try {
        const auto v = uniform_grid_refs(Aabb{{x0, y0}, {x1, y1}}, nx, ny);
        for (std::size_t i = 0; i < v.size(); ++i) {
            out[2 * i] = v[i].x;
            out[2 * i + 1] = v[i].y;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// center_cloud (data.cpp:198-223): centres xy in place, writes the offset.
int ref_center_cloud(double* xy, const double* vals, std::uint64_t n, double* offset) {
    try {
        PointCloud c;
        c.points = to_points(xy, n);
        c.values.assign(vals, vals + n);
        c = center_cloud(std::move(c));
        for (std::uint64_t i = 0; i < n; ++i) {
            xy[2 * i] = c.points[i].x;
            xy[2 * i + 1] = c.points[i].y;
        }
        offset[0] = c.offset.x;
        offset[1] = c.offset.y;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Single-block build_normal_system (solver.cpp:131-236 with n_blocks = 1):
// PointIndex -> assemble_submatrix -> transpose_matvec -> CooRowView -> gram_self.
// b_out (m*m, row-major) may be null to time without the dense copy.
int ref_build_normal_system(const double* xy, const double* vals, std::uint64_t n,
                            const double* refs_xy, std::uint64_t m, int family, double alpha,
                            double* b_out, double* rhs_out, std::uint64_t* design_nnz,
                            std::uint32_t* ref_nnz_out, double* times /* index, assembly, gram */) {
    try {
        const KernelSpec kernel(family_of(family), alpha);
        const std::vector<Point2> refs = to_points(refs_xy, m);
        auto t0 = Clock::now();
        const PointIndex index(to_points(xy, n));
        const double t_index = seconds_since(t0);

        t0 = Clock::now();
        const CooMatrix a = assemble_submatrix(index, refs, kernel);
        const double t_asm = seconds_since(t0);

        t0 = Clock::now();
        const std::vector<double> rhs = a.transpose_matvec(std::span<const double>(vals, n));
        const CooRowView view(a);
        const DenseBlock b = gram_self(view);
        const double t_gram = seconds_since(t0);

        if (b_out) std::memcpy(b_out, b.data.data(), m * m * sizeof(double));
        std::memcpy(rhs_out, rhs.data(), m * sizeof(double));
        *design_nnz = a.nnz();
        if (ref_nnz_out) {
            std::memset(ref_nnz_out, 0, m * sizeof(std::uint32_t));
            for (const std::uint32_t c : a.cols()) ++ref_nnz_out[c];
        }
        if (times) {
            times[0] = t_index;
            times[1] = t_asm;
            times[2] = t_gram;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// assemble_submatrix triplets (coo.cpp:166-192), sorted (col, row).
int ref_assemble_triplets(const double* xy, std::uint64_t n, const double* refs_xy,
                          std::uint64_t m, int family, double alpha, std::uint64_t cap,
                          std::uint32_t* rows, std::uint32_t* cols, double* vals,
                          std::uint64_t* nnz) {
    try {
        const PointIndex index(to_points(xy, n));
        const CooMatrix a =
            assemble_submatrix(index, to_points(refs_xy, m), KernelSpec(family_of(family), alpha));
        *nnz = a.nnz();
        if (a.nnz() > cap) throw std::runtime_error("triplet buffer too small");
        std::memcpy(rows, a.rows().data(), a.nnz() * sizeof(std::uint32_t));
        std::memcpy(cols, a.cols().data(), a.nnz() * sizeof(std::uint32_t));
        std::memcpy(vals, a.values().data(), a.nnz() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// evaluate_model (model.cpp:192-194) with a zero offset and no polynomial.
int ref_evaluate_model(const double* refs_xy, const double* w, std::uint64_t m, int family,
                       double alpha, const double* q_xy, std::uint64_t nq, double* f_out) {
    try {
        Model model{KernelSpec(family_of(family), alpha), to_points(refs_xy, m),
                    std::vector<double>(w, w + m), std::nullopt, {0.0, 0.0}};
        const auto f = evaluate_model(model, to_points(q_xy, nq));
        std::memcpy(f_out, f.data(), nq * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// error_report (model.cpp:196-232): out = {mae, deviation, rel_pct}.
int ref_error_report(const double* refs_xy, const double* w, std::uint64_t m, int family,
                     double alpha, const double* xy, const double* vals, std::uint64_t n,
                     double* out, double* signed_errors) {
    try {
        Model model{KernelSpec(family_of(family), alpha), to_points(refs_xy, m),
                    std::vector<double>(w, w + m), std::nullopt, {0.0, 0.0}};
        PointCloud cloud;
        cloud.points = to_points(xy, n);
        cloud.values.assign(vals, vals + n);
        const ErrorReport er = error_report(model, cloud);
        out[0] = er.mean_absolute_error;
        out[1] = er.deviation_of_error;
        out[2] = er.mean_relative_error_pct;
        if (signed_errors)
            std::memcpy(signed_errors, er.signed_errors.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// One timed CPU step of the reference path for bench.py --impl reference:
// index + assembly + rhs + gram on the given sample (no dense copy out).
int ref_bench_step(const double* xy, const double* vals, std::uint64_t n, const double* refs_xy,
                   std::uint64_t m, int family, double alpha, double* seconds,
                   std::uint64_t* design_nnz) {
    std::vector<double> rhs(m);
    double times[3] = {0, 0, 0};
    const auto t0 = Clock::now();
    const int rc = ref_build_normal_system(xy, vals, n, refs_xy, m, family, alpha, nullptr,
                                           rhs.data(), design_nnz, nullptr, times);
    *seconds = seconds_since(t0);
    return rc;
}

// The linear-polynomial border of build_normal_system (solver.cpp:189-207,
// 238-262), restated over the reference's own compiled assemble_submatrix:
// A^T P streamed in stored triplet order, P^T P / P^T h in one pass.
// atp: 3 x m (term-major), ptp: 3 x 3, pth: 3.
int ref_border(const double* xy, const double* vals, std::uint64_t n, const double* refs_xy,
               std::uint64_t m, int family, double alpha, double* atp, double* ptp, double* pth) {
    try {
        const KernelSpec kernel(family_of(family), alpha);
        const std::vector<Point2> pts = to_points(xy, n);
        const PointIndex index(pts);
        const CooMatrix a = assemble_submatrix(index, to_points(refs_xy, m), kernel);
        std::vector<double> slots(m * 3, 0.0);
        const auto arow = a.rows();
        const auto acol = a.cols();
        const auto aval = a.values();
        for (std::size_t i = 0; i < aval.size(); ++i) {
            const Point2 p = pts[arow[i]];
            double* slot = &slots[acol[i] * 3];
            slot[0] += aval[i] * p.x;
            slot[1] += aval[i] * p.y;
            slot[2] += aval[i];
        }
        for (std::size_t j = 0; j < m; ++j)
            for (int q = 0; q < 3; ++q) atp[q * m + j] = slots[j * 3 + q];
        double sxx = 0, sxy = 0, sx = 0, syy = 0, sy = 0, phx = 0, phy = 0, ph1 = 0;
        for (std::size_t i = 0; i < n; ++i) {
            const double x = pts[i].x, y = pts[i].y, h = vals[i];
            sxx += x * x;
            sxy += x * y;
            sx += x;
            syy += y * y;
            sy += y;
            phx += x * h;
            phy += y * h;
            ph1 += h;
        }
        const double t[9] = {sxx, sxy, sx, sxy, syy, sy, sx, sy, static_cast<double>(n)};
        std::memcpy(ptp, t, sizeof(t));
        pth[0] = phx;
        pth[1] = phy;
        pth[2] = ph1;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// evaluate_model (model.cpp:192-194) of a bordered model (poly = a[0..2]).
int ref_evaluate_model_poly(const double* refs_xy, const double* w, const double* a, std::uint64_t m,
                            int family, double alpha, const double* q_xy, std::uint64_t nq, double* f_out) {
    try {
        Model model{KernelSpec(family_of(family), alpha), to_points(refs_xy, m),
                    std::vector<double>(w, w + m), std::array<double, 3>{a[0], a[1], a[2]}, {0.0, 0.0}};
        const auto f = evaluate_model(model, to_points(q_xy, nq));
        std::memcpy(f_out, f.data(), nq * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- on-disk formats: the reference's own writers/readers (model.cpp, data.cpp)
// save_model (model.cpp:76-115); poly may be null.
int ref_save_model(const char* path, int family, double alpha, const double* refs_xy, const double* w,
                   std::uint64_t m, double offx, double offy, const double* poly) {
    try {
        std::optional<std::array<double, 3>> a;
        if (poly) a = std::array<double, 3>{poly[0], poly[1], poly[2]};
        Model model{KernelSpec(family_of(family), alpha), to_points(refs_xy, m), std::vector<double>(w, w + m), a,
                    {offx, offy}};
        save_model(model, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// load_model (model.cpp:117-190): scal = {alpha, offx, offy, poly[3]}; refs/w
// sized by the caller (cap entries).
int ref_load_model(const char* path, int* family, int* has_poly, std::uint64_t* m, double* scal,
                   double* refs_xy, double* w, std::uint64_t cap) {
    try {
        const Model model = load_model(path);
        *family = static_cast<int>(model.kernel.family());
        *has_poly = model.poly ? 1 : 0;
        *m = model.refs.size();
        scal[0] = model.kernel.alpha();
        scal[1] = model.offset.x;
        scal[2] = model.offset.y;
        for (int k = 0; k < 3; ++k) scal[3 + k] = model.poly ? (*model.poly)[k] : 0.0;
        for (std::uint64_t j = 0; j < model.refs.size() && j < cap; ++j) {
            refs_xy[2 * j] = model.refs[j].x;
            refs_xy[2 * j + 1] = model.refs[j].y;
            w[j] = model.weights[j];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// save_xyz (data.cpp:143-157)
int ref_save_xyz(const char* path, const double* xy, const double* h, std::uint64_t n) {
    try {
        PointCloud c;
        c.points = to_points(xy, n);
        c.values.assign(h, h + n);
        save_xyz(c, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// kind 0 load_xyz, 1 load_eval_points, 2 load_ref_points (data.cpp:126-196):
// rows (n x arity) into out (cap doubles).
int ref_load_records(const char* path, int kind, std::uint64_t* n, int* arity, double* out, std::uint64_t cap) {
    try {
        std::vector<double> rows;
        if (kind == 0) {
            const PointCloud c = load_xyz(path);
            *arity = 3;
            for (std::size_t i = 0; i < c.size(); ++i) rows.insert(rows.end(), {c.points[i].x, c.points[i].y, c.values[i]});
        } else if (kind == 1) {
            const EvalPoints e = load_eval_points(path);
            *arity = e.has_values ? 3 : 2;
            for (std::size_t i = 0; i < e.points.size(); ++i) {
                rows.insert(rows.end(), {e.points[i].x, e.points[i].y});
                if (e.has_values) rows.push_back(e.values[i]);
            }
        } else {
            *arity = 2;
            for (const Point2& p : load_ref_points(path)) rows.insert(rows.end(), {p.x, p.y});
        }
        *n = rows.size() / static_cast<std::uint64_t>(*arity);
        std::memcpy(out, rows.data(), std::min<std::uint64_t>(cap, rows.size()) * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// write_signed_errors (model.cpp:234-256)
int ref_write_signed_errors(const char* path, const double* xy, const double* h, std::uint64_t n, double offx,
                            double offy, const double* pred) {
    try {
        PointCloud c;
        c.points = to_points(xy, n);
        c.values.assign(h, h + n);
        c.offset = {offx, offy};
        write_signed_errors(c, std::span<const double>(pred, n), path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
