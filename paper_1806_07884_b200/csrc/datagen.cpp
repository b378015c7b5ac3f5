// datagen.cpp -- seeded host generators for the BASELINE configs (fixtures,
// not the hot path).  Shared by the GPU path, the oracle and the bench so all
// of them see bit-identical inputs.
//
// Halton and the Franke surface restate the reference's generators bit for
// bit (data.cpp:76-124), and the grid restates uniform_grid_refs
// (data.cpp:225-249).  The other distributions are not in the reference;
// they use a counter-based generator (splitmix64 of seed and index), so every
// value is a pure function of (seed, index) and generation parallelises.
#include <cmath>
#include <cstdint>

namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// uniform [0,1) from (seed, stream, index)
inline double uni01(uint64_t seed, uint64_t stream, uint64_t i) {
    const uint64_t k = splitmix64(seed ^ splitmix64(stream * 0x632be59bd9b4e019ull + i));
    return (double)(k >> 11) * 0x1.0p-53;
}

// standard normal (Box-Muller, cosine branch) from (seed, index)
inline double normal01(uint64_t seed, uint64_t i) {
    const double u1 = 1.0 - uni01(seed, 0x6e6f726d, 2 * i);  // (0, 1]
    const double u2 = uni01(seed, 0x6e6f726d, 2 * i + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

// data.cpp:76-87
inline double radical_inverse(unsigned base, uint64_t index) {
    const double inv_base = 1.0 / base;
    double f = 1.0;
    double r = 0.0;
    while (index > 0) {
        f *= inv_base;
        r += f * (double)(index % base);
        index /= base;
    }
    return r;
}

inline double sq(double v) { return v * v; }

// data.cpp:108-116 (code form: the f2 y-term is (9y+1)/10, unsquared)
inline double franke(double x, double y) {
    const double f1 = 0.75 * std::exp(-(sq(9.0 * x - 2.0) / 4.0 + sq(9.0 * y - 2.0) / 4.0));
    const double f2 = 0.75 * std::exp(-(sq(9.0 * x + 1.0) / 49.0 + (9.0 * y + 1.0) / 10.0));
    const double f3 = 0.5 * std::exp(-(sq(9.0 * x - 7.0) / 4.0 + sq(9.0 * y - 3.0) / 4.0));
    const double f4 = 0.2 * std::exp(-(sq(9.0 * x - 4.0) + sq(9.0 * y - 7.0)));
    return f1 + f2 + f3 - f4;
}

// value noise on the integer lattice, smoothstep-bilinear
inline double lattice(uint64_t seed, int octave, int64_t i, int64_t j) {
    const uint64_t k = splitmix64(seed ^ splitmix64(((uint64_t)octave << 56) ^
                                                    ((uint64_t)(i & 0xfffffff) << 28) ^
                                                    (uint64_t)(j & 0xfffffff)));
    return 2.0 * ((double)(k >> 11) * 0x1.0p-53) - 1.0;
}

inline double value_noise(uint64_t seed, int octave, double x, double y) {
    const double fx = std::floor(x), fy = std::floor(y);
    const int64_t i = (int64_t)fx, j = (int64_t)fy;
    const double tx = x - fx, ty = y - fy;
    const double sx = tx * tx * (3.0 - 2.0 * tx), sy = ty * ty * (3.0 - 2.0 * ty);
    const double v00 = lattice(seed, octave, i, j), v10 = lattice(seed, octave, i + 1, j);
    const double v01 = lattice(seed, octave, i, j + 1), v11 = lattice(seed, octave, i + 1, j + 1);
    const double a = v00 + (v10 - v00) * sx;
    const double b = v01 + (v11 - v01) * sx;
    return a + (b - a) * sy;
}

}  // namespace

extern "C" {

// halton_points (data.cpp:89-98) for indices [start, start+count), point-major.
void dg_halton(uint64_t start, uint64_t count, int dims, double* out) {
    static const unsigned kBases[] = {2, 3, 5};
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)count; ++k)
        for (int d = 0; d < dims; ++d)
            out[(uint64_t)k * dims + d] = radical_inverse(kBases[d], start + (uint64_t)k);
}

// halton_points at indices first, first + stride, ... (count of them), point-major.
void dg_halton_strided(uint64_t first, uint64_t stride, uint64_t count, int dims, double* out) {
    static const unsigned kBases[] = {2, 3, 5};
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)count; ++k)
        for (int d = 0; d < dims; ++d)
            out[(uint64_t)k * dims + d] = radical_inverse(kBases[d], first + stride * (uint64_t)k);
}

// inout[k] += sigma * N(0,1)_{first + stride k}: the noise of the points at those positions.
void dg_add_noise_strided(uint64_t seed, uint64_t first, uint64_t stride, uint64_t count, double sigma,
                          double* inout) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)count; ++k)
        inout[k] += sigma * normal01(seed, first + stride * (uint64_t)k);
}

// uniform_grid_refs(box, nx, ny) (data.cpp:236-249): y-major, x fastest.
void dg_grid_refs(double x0, double y0, double x1, double y1, uint64_t nx, uint64_t ny,
                  double* out) {
    const auto coord = [](double lo, double hi, uint64_t i, uint64_t n) {
        if (n == 1) return 0.5 * (lo + hi);
        return lo + (hi - lo) * (static_cast<double>(i) / static_cast<double>(n - 1));
    };
    for (uint64_t iy = 0; iy < ny; ++iy)
        for (uint64_t ix = 0; ix < nx; ++ix) {
            out[2 * (iy * nx + ix)] = coord(x0, x1, ix, nx);
            out[2 * (iy * nx + ix) + 1] = coord(y0, y1, iy, ny);
        }
}

void dg_franke(const double* xy, uint64_t n, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = franke(xy[2 * i], xy[2 * i + 1]);
}

void dg_uniform(uint64_t seed, uint64_t n, int dims, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        for (int d = 0; d < dims; ++d)
            out[(uint64_t)i * dims + d] = uni01(seed, (uint64_t)d + 1, (uint64_t)i);
}

// inout[i] += sigma * N(0,1)_i  (sigma is the standard deviation)
void dg_add_noise(uint64_t seed, uint64_t n, double sigma, double* inout) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) inout[i] += sigma * normal01(seed, (uint64_t)i);
}

// config 2 surface: sin(4x) cos(4y)
void dg_sincos(const double* xy, uint64_t n, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        out[i] = std::sin(4.0 * xy[2 * i]) * std::cos(4.0 * xy[2 * i + 1]);
}

// config 3 surface: exp(-|x - 0.5|^2 / 0.1) + 0.5 sin(6 z)
void dg_bump3(const double* xyz, uint64_t n, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const double* p = xyz + 3 * i;
        const double r2 = sq(p[0] - 0.5) + sq(p[1] - 0.5) + sq(p[2] - 0.5);
        out[i] = std::exp(-r2 / 0.1) + 0.5 * std::sin(6.0 * p[2]);
    }
}

// config 4 points: 4 isotropic Gaussians (sigma 0.05-0.2) plus a 5% uniform
// floor (keeps every Halton centre's support populated), clamped to [0,1]^2.
// floor = 0 draws BASELINE's pure 4-Gaussian mixture (the same component
// weights renormalised), used to measure the assembly both ways.
void dg_mixture_floor(uint64_t seed, uint64_t n, int floor, double* out);
void dg_mixture(uint64_t seed, uint64_t n, double* out) { dg_mixture_floor(seed, n, 1, out); }
void dg_mixture_floor(uint64_t seed, uint64_t n, int floor, double* out) {
    const double f = floor ? 1.0 : 1.0 / 0.95;
    const double w[5] = {0.30 * f, 0.25 * f, 0.25 * f, floor ? 0.15 : 2.0, 0.05};
    static const double mx[4] = {0.30, 0.70, 0.50, 0.20};
    static const double my[4] = {0.30, 0.35, 0.75, 0.80};
    static const double sg[4] = {0.05, 0.10, 0.20, 0.08};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const double u = uni01(seed, 17, (uint64_t)i);
        int c = 0;
        double acc = w[0];
        while (c < 4 && u >= acc) acc += w[++c];
        double x, y;
        if (c == 4) {
            x = uni01(seed, 18, (uint64_t)i);
            y = uni01(seed, 19, (uint64_t)i);
        } else {
            x = mx[c] + sg[c] * normal01(seed + 1, 2 * (uint64_t)i);
            y = my[c] + sg[c] * normal01(seed + 1, 2 * (uint64_t)i + 1);
        }
        out[2 * i] = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
        out[2 * i + 1] = y < 0.0 ? 0.0 : (y > 1.0 ? 1.0 : y);
    }
}

// config 4 surface: 6-octave fBm of value noise, Hurst 0.7 (gain 2^-0.7),
// lacunarity 2, base frequency 4.
void dg_fbm(uint64_t seed, const double* xy, uint64_t n, double* out) {
    const double gain = std::pow(2.0, -0.7);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        double f = 4.0, a = 1.0, s = 0.0;
        for (int o = 0; o < 6; ++o) {
            s += a * value_noise(seed, o, f * xy[2 * i], f * xy[2 * i + 1]);
            f *= 2.0;
            a *= gain;
        }
        out[i] = s;
    }
}

}  // extern "C"
