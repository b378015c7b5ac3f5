// rbfit_io.cpp -- on-disk formats of the reference, host side.
//
// The GPU fit writes and reads the same files as the reference, byte for
// byte, so a model fitted here feeds the reference's own `eval` and vice
// versa:
//   * model file "rbfit model 1"      -- save_model / load_model (model.cpp:76-190)
//   * XYZ records "x y h"             -- load_xyz / save_xyz (data.cpp:126-157)
//   * evaluation / reference points   -- load_eval_points, load_ref_points (data.cpp:159-196)
//   * signed-error export             -- write_signed_errors (model.cpp:234-256)
//   * centring                        -- center_cloud (data.cpp:198-223)
// Numbers are written with std::to_chars shortest round-trip formatting and
// parsed with std::from_chars, as the reference does, so every double
// survives a save/load cycle exactly.  Error classes and messages follow the
// reference's.
//
// The extern "C" shims at the end expose the same functions to the Python
// mirror (paper_1806_07884_b200/rbfit_io.py) through ctypes; C declarations
// in include/rbfit_io.h.
#include <array>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <system_error>

#include "rbfit_gpu.hpp"
#include "rbfit_io.h"

namespace rbfit_b200 {

namespace {

constexpr std::string_view kModelMagic = "rbfit model";
constexpr int kModelVersion = 1;

void put_double(std::string& out, double v) {
    char buf[32];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);
    out.append(buf, res.ptr);
}

// data.cpp:16-22: an optional leading '+', then the whole token must parse
bool parse_number(std::string_view tok, double& out) {
    if (!tok.empty() && tok.front() == '+') tok.remove_prefix(1);
    const char* last = tok.data() + tok.size();
    const auto res = std::from_chars(tok.data(), last, out);
    return res.ec == std::errc() && res.ptr == last;
}

bool separator(char c) { return c == ' ' || c == '\t' || c == ',' || c == '\r'; }

constexpr std::size_t kBadRecord = static_cast<std::size_t>(-1);

// data.cpp:27-42: up to four numeric fields; '#' starts a comment
std::size_t record_fields(std::string_view line, std::array<double, 4>& f) {
    std::size_t n = 0, i = 0;
    for (;;) {
        while (i < line.size() && separator(line[i])) ++i;
        if (i == line.size() || line[i] == '#') return n;
        std::size_t j = i;
        while (j < line.size() && !separator(line[j]) && line[j] != '#') ++j;
        if (n == f.size() || !parse_number(line.substr(i, j - i), f[n])) return kBadRecord;
        ++n;
        i = j;
    }
}

[[noreturn]] void record_error(const std::filesystem::path& path, std::size_t line_no, const std::string& what) {
    throw std::runtime_error(path.string() + ":" + std::to_string(line_no) + ": " + what);
}

template <typename Sink>
void read_records(const std::filesystem::path& path, Sink&& sink) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open '" + path.string() + "' for reading");
    std::string line;
    std::array<double, 4> f{};
    for (std::size_t line_no = 1; std::getline(in, line); ++line_no) {
        const std::size_t n = record_fields(line, f);
        if (n == kBadRecord) record_error(path, line_no, "malformed record '" + line + "'");
        if (n) sink(line_no, f, n);
    }
}

void write_text(const std::filesystem::path& path, const std::string& text) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open '" + path.string() + "' for writing");
    out << text;
    if (!out) throw std::runtime_error("write to '" + path.string() + "' failed");
}

}  // namespace

// ------------------------------------------------------------------ model file
void save_model(const Model& model, const std::filesystem::path& path) {
    if (model.refs.empty()) throw std::invalid_argument("model has no reference points");
    if (model.weights.size() != model.refs.size())
        throw std::invalid_argument("model weight count does not match reference count");
    std::string t;
    t.reserve(64 + model.refs.size() * 72);
    t.append(kModelMagic).append(" ").append(std::to_string(kModelVersion)).append("\n");
    t.append("kernel ").append(kernel_name(model.kernel.family())).append("\n");
    t.append("alpha ");
    put_double(t, model.kernel.alpha());
    t.append("\noffset ");
    put_double(t, model.offset.x);
    t.push_back(' ');
    put_double(t, model.offset.y);
    t.append("\npoly ").append(model.poly ? "1" : "0").append("\n");
    if (model.poly) {
        t.append("poly-coeffs ");
        for (int k = 0; k < 3; ++k) {
            if (k) t.push_back(' ');
            put_double(t, (*model.poly)[k]);
        }
        t.push_back('\n');
    }
    t.append("refs ").append(std::to_string(model.refs.size())).append("\n");
    for (std::size_t j = 0; j < model.refs.size(); ++j) {
        put_double(t, model.refs[j].x);
        t.push_back(' ');
        put_double(t, model.refs[j].y);
        t.push_back(' ');
        put_double(t, model.weights[j]);
        t.push_back('\n');
    }
    write_text(path, t);
}

Model load_model(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open '" + path.string() + "' for reading");
    const std::string where = "model file '" + path.string() + "': ";
    auto bad = [&](const std::string& what) { return std::runtime_error(where + what); };
    std::string line;
    if (!std::getline(in, line) || line.compare(0, kModelMagic.size(), kModelMagic) != 0)
        throw bad("not a model file (missing '" + std::string(kModelMagic) + "' header)");
    {
        std::istringstream hs(line.substr(kModelMagic.size()));
        int version = -1;
        if (!(hs >> version)) throw bad("missing format version");
        if (version != kModelVersion) throw bad("unsupported format version " + std::to_string(version));
    }
    auto field = [&](const char* key) {
        if (!std::getline(in, line)) throw bad(std::string("missing '") + key + "' line");
        std::istringstream ls(line);
        std::string k;
        ls >> k;
        if (k != key) throw bad("expected '" + std::string(key) + "', got '" + k + "'");
        return ls;
    };
    auto number = [&](std::istringstream& ls, const char* what) {
        std::string tok;
        if (!(ls >> tok)) throw bad(std::string("missing ") + what);
        double v = 0.0;
        const auto res = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (res.ec != std::errc() || res.ptr != tok.data() + tok.size())
            throw bad(std::string("bad ") + what + " '" + tok + "'");
        return v;
    };

    auto ls = field("kernel");
    std::string kname;
    if (!(ls >> kname)) throw bad("missing kernel name");
    KernelFamily family;
    try {
        family = kernel_from_name(kname);
    } catch (const std::invalid_argument& e) {
        throw bad(e.what());
    }
    ls = field("alpha");
    const double alpha = number(ls, "alpha");
    ls = field("offset");
    Point2 offset;
    offset.x = number(ls, "offset x");
    offset.y = number(ls, "offset y");
    ls = field("poly");
    int flag = -1;
    if (!(ls >> flag) || (flag != 0 && flag != 1)) throw bad("poly flag must be 0 or 1");
    std::optional<std::array<double, 3>> poly;
    if (flag == 1) {
        ls = field("poly-coeffs");
        std::array<double, 3> a{};
        for (double& v : a) v = number(ls, "poly coefficient");
        poly = a;
    }
    ls = field("refs");
    std::size_t m = 0;
    if (!(ls >> m) || m == 0) throw bad("bad reference count");
    Model model{KernelSpec(family, alpha), {}, {}, poly, offset};
    model.refs.reserve(m);
    model.weights.reserve(m);
    for (std::size_t j = 0; j < m; ++j) {
        if (!std::getline(in, line)) throw bad("truncated reference list");
        std::istringstream rs(line);
        Point2 p;
        p.x = number(rs, "reference x");
        p.y = number(rs, "reference y");
        model.refs.push_back(p);
        model.weights.push_back(number(rs, "weight"));
    }
    return model;
}

// ------------------------------------------------------------------ XYZ files
PointCloud load_xyz(const std::filesystem::path& path) {
    PointCloud cloud;
    read_records(path, [&](std::size_t line_no, const std::array<double, 4>& f, std::size_t n) {
        if (n != 3) record_error(path, line_no, "expected 3 fields (x y h), got " + std::to_string(n));
        if (!std::isfinite(f[0]) || !std::isfinite(f[1]) || !std::isfinite(f[2]))
            record_error(path, line_no, "non-finite value");
        cloud.points.push_back({f[0], f[1]});
        cloud.values.push_back(f[2]);
    });
    if (cloud.points.empty()) throw std::runtime_error("'" + path.string() + "' contains no data records");
    return cloud;
}

void save_xyz(const PointCloud& cloud, const std::filesystem::path& path) {
    std::string t;
    t.reserve(cloud.size() * 64);
    for (std::size_t i = 0; i < cloud.size(); ++i) {
        put_double(t, cloud.points[i].x);
        t.push_back(' ');
        put_double(t, cloud.points[i].y);
        t.push_back(' ');
        put_double(t, cloud.values[i]);
        t.push_back('\n');
    }
    write_text(path, t);
}

EvalPoints load_eval_points(const std::filesystem::path& path) {
    EvalPoints pts;
    std::size_t arity = 0;
    read_records(path, [&](std::size_t line_no, const std::array<double, 4>& f, std::size_t n) {
        if (n != 2 && n != 3) record_error(path, line_no, "expected 2 (x y) or 3 (x y h) fields");
        if (arity == 0) {
            arity = n;
            pts.has_values = n == 3;
        } else if (n != arity) {
            record_error(path, line_no, "mixed 2- and 3-field records");
        }
        if (!std::isfinite(f[0]) || !std::isfinite(f[1]) || (n == 3 && !std::isfinite(f[2])))
            record_error(path, line_no, "non-finite value");
        pts.points.push_back({f[0], f[1]});
        if (n == 3) pts.values.push_back(f[2]);
    });
    if (pts.points.empty()) throw std::runtime_error("'" + path.string() + "' contains no data records");
    return pts;
}

std::vector<Point2> load_ref_points(const std::filesystem::path& path) {
    std::vector<Point2> refs;
    read_records(path, [&](std::size_t line_no, const std::array<double, 4>& f, std::size_t n) {
        if (n != 2 && n != 3) record_error(path, line_no, "expected 2 (x y) fields");  // h tolerated
        if (!std::isfinite(f[0]) || !std::isfinite(f[1])) record_error(path, line_no, "non-finite value");
        refs.push_back({f[0], f[1]});
    });
    if (refs.empty()) throw std::runtime_error("'" + path.string() + "' contains no data records");
    return refs;
}

void write_signed_errors(const PointCloud& cloud, std::span<const double> predictions,
                         const std::filesystem::path& path) {
    if (predictions.size() != cloud.size())
        throw std::invalid_argument("write_signed_errors: prediction count mismatch");
    std::string t;
    t.reserve(cloud.size() * 110);
    for (std::size_t i = 0; i < cloud.size(); ++i) {
        put_double(t, cloud.points[i].x + cloud.offset.x);
        t.push_back(' ');
        put_double(t, cloud.points[i].y + cloud.offset.y);
        t.push_back(' ');
        put_double(t, cloud.values[i]);
        t.push_back(' ');
        put_double(t, predictions[i]);
        t.push_back(' ');
        put_double(t, predictions[i] - cloud.values[i]);
        t.push_back('\n');
    }
    write_text(path, t);
}

// data.cpp:198-223: Neumaier-compensated mean, subtracted, recorded in offset
PointCloud center_cloud(PointCloud cloud) {
    if (cloud.points.empty()) throw std::invalid_argument("center_cloud: empty cloud");
    double s[2] = {0.0, 0.0}, c[2] = {0.0, 0.0};
    auto add = [](double& sum, double& comp, double v) {
        const double t = sum + v;
        comp += std::abs(sum) >= std::abs(v) ? (sum - t) + v : (v - t) + sum;
        sum = t;
    };
    for (const Point2& p : cloud.points) {
        add(s[0], c[0], p.x);
        add(s[1], c[1], p.y);
    }
    const double n = static_cast<double>(cloud.points.size());
    const double mx = (s[0] + c[0]) / n, my = (s[1] + c[1]) / n;
    for (Point2& p : cloud.points) {
        p.x -= mx;
        p.y -= my;
    }
    cloud.offset.x += mx;
    cloud.offset.y += my;
    return cloud;
}

}  // namespace rbfit_b200

// ------------------------------------------------------------------ C shims
// Status 0 ok, 1 std::invalid_argument, 2 std::runtime_error (incl. I/O and
// format errors); the message is kept per thread for rbfit_io_last_error().
namespace {
thread_local std::string g_io_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_io_error = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_io_error = e.what();
        return 2;
    }
}

// Loaded results are parked here between the load call and the copy-out call.
thread_local rbfit_b200::Model* g_model = nullptr;
thread_local std::vector<double> g_rows;  // flattened records
thread_local std::size_t g_arity = 0;
}  // namespace

extern "C" {

const char* rbfit_io_last_error() { return g_io_error.c_str(); }

int rbfit_io_save_model(const char* path, int family, double alpha, const double* refs_xy, const double* weights,
                        uint64_t m, const double* offset, const double* poly) {
    return guarded([&] {
        using namespace rbfit_b200;
        Model model{KernelSpec(static_cast<KernelFamily>(family), alpha), {}, {}, std::nullopt,
                    {offset ? offset[0] : 0.0, offset ? offset[1] : 0.0}};
        model.refs.resize(m);
        if (m) std::memcpy(model.refs.data(), refs_xy, m * sizeof(Point2));
        model.weights.assign(weights, weights + m);
        if (poly) model.poly = std::array<double, 3>{poly[0], poly[1], poly[2]};
        save_model(model, path);
    });
}

// Loads into the per-thread slot; header: family, has_poly, m; doubles: alpha,
// offset x/y, poly[3] (zeros without the border).
int rbfit_io_load_model(const char* path, int* family, int* has_poly, uint64_t* m, double* scalars6) {
    return guarded([&] {
        using namespace rbfit_b200;
        Model loaded = load_model(path);
        delete g_model;
        g_model = new Model(std::move(loaded));
        *family = static_cast<int>(g_model->kernel.family());
        *has_poly = g_model->poly ? 1 : 0;
        *m = g_model->refs.size();
        scalars6[0] = g_model->kernel.alpha();
        scalars6[1] = g_model->offset.x;
        scalars6[2] = g_model->offset.y;
        for (int k = 0; k < 3; ++k) scalars6[3 + k] = g_model->poly ? (*g_model->poly)[k] : 0.0;
    });
}

int rbfit_io_take_model(double* refs_xy, double* weights) {
    return guarded([&] {
        if (!g_model) throw std::runtime_error("no model loaded");
        std::memcpy(refs_xy, g_model->refs.data(), g_model->refs.size() * sizeof(rbfit_b200::Point2));
        std::memcpy(weights, g_model->weights.data(), g_model->weights.size() * sizeof(double));
        delete g_model;
        g_model = nullptr;
    });
}

int rbfit_io_save_xyz(const char* path, const double* xy, const double* h, uint64_t n) {
    return guarded([&] {
        rbfit_b200::PointCloud c;
        c.points.resize(n);
        if (n) std::memcpy(c.points.data(), xy, n * sizeof(rbfit_b200::Point2));
        c.values.assign(h, h + n);
        rbfit_b200::save_xyz(c, path);
    });
}

// kind: 0 load_xyz (3 columns), 1 load_eval_points (2 or 3), 2 load_ref_points (2)
int rbfit_io_load_records(const char* path, int kind, uint64_t* n, int* arity) {
    return guarded([&] {
        using namespace rbfit_b200;
        g_rows.clear();
        if (kind == 0) {
            const PointCloud c = load_xyz(path);
            g_arity = 3;
            for (std::size_t i = 0; i < c.size(); ++i)
                g_rows.insert(g_rows.end(), {c.points[i].x, c.points[i].y, c.values[i]});
        } else if (kind == 1) {
            const EvalPoints e = load_eval_points(path);
            g_arity = e.has_values ? 3 : 2;
            for (std::size_t i = 0; i < e.points.size(); ++i) {
                g_rows.insert(g_rows.end(), {e.points[i].x, e.points[i].y});
                if (e.has_values) g_rows.push_back(e.values[i]);
            }
        } else {
            const auto r = load_ref_points(path);
            g_arity = 2;
            for (const Point2& p : r) g_rows.insert(g_rows.end(), {p.x, p.y});
        }
        *arity = static_cast<int>(g_arity);
        *n = g_rows.size() / g_arity;
    });
}

int rbfit_io_take_records(double* out) {
    return guarded([&] {
        std::memcpy(out, g_rows.data(), g_rows.size() * sizeof(double));
        g_rows.clear();
        g_rows.shrink_to_fit();
    });
}

int rbfit_io_write_signed_errors(const char* path, const double* xy, const double* h, uint64_t n,
                                 const double* offset, const double* pred) {
    return guarded([&] {
        rbfit_b200::PointCloud c;
        c.points.resize(n);
        if (n) std::memcpy(c.points.data(), xy, n * sizeof(rbfit_b200::Point2));
        c.values.assign(h, h + n);
        if (offset) c.offset = {offset[0], offset[1]};
        rbfit_b200::write_signed_errors(c, std::span<const double>(pred, n), path);
    });
}

int rbfit_io_center_cloud(double* xy, uint64_t n, double* offset) {
    return guarded([&] {
        rbfit_b200::PointCloud c;
        c.points.resize(n);
        if (n) std::memcpy(c.points.data(), xy, n * sizeof(rbfit_b200::Point2));
        c.values.assign(n, 0.0);
        c.offset = {offset[0], offset[1]};
        c = rbfit_b200::center_cloud(std::move(c));
        std::memcpy(xy, c.points.data(), n * sizeof(rbfit_b200::Point2));
        offset[0] = c.offset.x;
        offset[1] = c.offset.y;
    });
}

}  // extern "C"
