/*
 * rbf_oracle.c -- CPU restatement of the reference CS-RBF hot path.
 * TEST INFRASTRUCTURE ONLY (see rbf_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off; no -march so no FMA is ever formed).
 */
#include "rbf_oracle.h"

#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- kernel */

/* kernel.hpp:42-62.  wendland-3-2 (family 3) is the BASELINE extension
 * (1-t)^6 (35t^2+18t+3), written in the same Horner style; phi(0) = 3. */
static double phi_inside(int family, double alpha, double r) {
    const double t = alpha * r;
    if (!(t < 1.0)) return 0.0;
    const double u = 1.0 - t;
    switch (family) {
        case ORC_W30:
            return u * u;
        case ORC_W31: {
            const double u2 = u * u;
            return u2 * u2 * (4.0 * t + 1.0);
        }
        case ORC_W33: {
            const double u2 = u * u;
            const double u4 = u2 * u2;
            return u4 * u4 * (((32.0 * t + 25.0) * t + 8.0) * t + 1.0);
        }
        case ORC_W32: {
            const double u2 = u * u;
            const double u4 = u2 * u2;
            const double u6 = u4 * u2;
            return u6 * ((35.0 * t + 18.0) * t + 3.0);
        }
    }
    return 0.0;
}

int orc_phi(int family, double alpha, double r, double* out) {
    if (family < 0 || family > 3) return ORC_INVALID;
    if (!(alpha > 0.0) || !isfinite(alpha)) return ORC_INVALID; /* kernel.cpp:35-38 */
    if (!(r >= 0.0) || !isfinite(r)) return ORC_DOMAIN;         /* kernel.hpp:43-44 */
    *out = phi_inside(family, alpha, r);
    return ORC_OK;
}

/* ------------------------------------------------------------ fixtures */

double orc_radical_inverse(unsigned base, uint64_t index) { /* data.cpp:76-87 */
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

static double sq(double v) { return v * v; }

double orc_franke(double x, double y) { /* data.cpp:108-116 */
    const double f1 = 0.75 * exp(-(sq(9.0 * x - 2.0) / 4.0 + sq(9.0 * y - 2.0) / 4.0));
    const double f2 = 0.75 * exp(-(sq(9.0 * x + 1.0) / 49.0 + (9.0 * y + 1.0) / 10.0));
    const double f3 = 0.5 * exp(-(sq(9.0 * x - 7.0) / 4.0 + sq(9.0 * y - 3.0) / 4.0));
    const double f4 = 0.2 * exp(-(sq(9.0 * x - 4.0) + sq(9.0 * y - 7.0)));
    return f1 + f2 + f3 - f4;
}

/* -------------------------------------------------------------- geometry */

/* geometry.hpp:16-20 (dx*dx + dy*dy), extended left-to-right for 3-D. */
static double dist2(int dim, const double* a, const double* b) {
    const double dx = a[0] - b[0];
    const double dy = a[1] - b[1];
    double d2 = dx * dx + dy * dy;
    if (dim == 3) {
        const double dz = a[2] - b[2];
        d2 = d2 + dz * dz;
    }
    return d2;
}

/* Uniform cell grid over a point set; cell edge >= the query radius, so a
 * query only visits its own and the adjacent cells.  Stands in for the
 * reference's kd-tree (kdtree.cpp); hit sets are identical because the
 * inclusion test (strict d2 < R^2, kdtree.cpp:74) is applied to every
 * candidate and results are sorted by index (kdtree.cpp:85-86). */
typedef struct {
    int dim;
    double lo[3];
    double cell;
    int64_t n[3];
    uint64_t* start; /* ncell+1 */
    uint32_t* ids;
} grid_t;

static int64_t cell_coord(const grid_t* g, int d, double v) {
    double c = floor((v - g->lo[d]) / g->cell);
    if (c < -2.0) c = -2.0;
    if (c > (double)g->n[d] + 1.0) c = (double)g->n[d] + 1.0;
    return (int64_t)c;
}

static int grid_build(grid_t* g, int dim, const double* p, uint64_t m, double radius) {
    g->dim = dim;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) lo[d] = hi[d] = p[d];
    for (uint64_t i = 0; i < m; ++i)
        for (int d = 0; d < dim; ++d) {
            const double v = p[i * dim + d];
            if (v < lo[d]) lo[d] = v;
            if (v > hi[d]) hi[d] = v;
        }
    g->cell = radius * (1.0 + 1e-9);
    const double max_cells = dim == 2 ? 4.0e6 : 8.0e6;
    for (;;) {
        double total = 1.0;
        for (int d = 0; d < dim; ++d) total *= floor((hi[d] - lo[d]) / g->cell) + 1.0;
        if (total <= max_cells) break;
        g->cell *= 1.5;
    }
    uint64_t ncell = 1;
    for (int d = 0; d < 3; ++d) {
        g->lo[d] = lo[d];
        g->n[d] = d < dim ? (int64_t)floor((hi[d] - lo[d]) / g->cell) + 1 : 1;
        ncell *= (uint64_t)g->n[d];
    }
    g->start = (uint64_t*)calloc(ncell + 1, sizeof(uint64_t));
    g->ids = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
    uint64_t* key = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
    if (!g->start || !g->ids || !key) return ORC_RUNTIME;
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t k = 0;
        for (int d = dim - 1; d >= 0; --d) {
            int64_t c = cell_coord(g, d, p[i * dim + d]);
            if (c < 0) c = 0;
            if (c >= g->n[d]) c = g->n[d] - 1;
            k = k * (uint64_t)g->n[d] + (uint64_t)c;
        }
        key[i] = k;
        g->start[k + 1]++;
    }
    for (uint64_t c = 0; c < ncell; ++c) g->start[c + 1] += g->start[c];
    uint64_t* cur = (uint64_t*)malloc((ncell ? ncell : 1) * sizeof(uint64_t));
    memcpy(cur, g->start, ncell * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) g->ids[cur[key[i]]++] = (uint32_t)i; /* ascending ids per cell */
    free(cur);
    free(key);
    return ORC_OK;
}

static void grid_free(grid_t* g) {
    free(g->start);
    free(g->ids);
}

typedef struct {
    uint32_t id;
    double v;
} hit_t;

static int hit_cmp(const void* a, const void* b) {
    const uint32_t x = ((const hit_t*)a)->id, y = ((const hit_t*)b)->id;
    return (x > y) - (x < y);
}

static void sort_hits(hit_t* h, uint64_t k) {
    if (k > 48) {
        qsort(h, k, sizeof(hit_t), hit_cmp);
        return;
    }
    for (uint64_t i = 1; i < k; ++i) {
        hit_t t = h[i];
        uint64_t j = i;
        while (j > 0 && h[j - 1].id > t.id) {
            h[j] = h[j - 1];
            --j;
        }
        h[j] = t;
    }
}

/* Visit every grid member within the 3^dim cell neighbourhood of q. */
#define GRID_FOR_CANDIDATES(g, q, IDVAR, BODY)                                          \
    do {                                                                                \
        int64_t c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};                                   \
        int empty_ = 0;                                                                 \
        for (int d_ = 0; d_ < 3; ++d_) {                                                \
            if (d_ < (g)->dim) {                                                        \
                const int64_t cc = cell_coord((g), d_, (q)[d_]);                        \
                c0[d_] = cc - 1 < 0 ? 0 : cc - 1;                                       \
                c1[d_] = cc + 1 >= (g)->n[d_] ? (g)->n[d_] - 1 : cc + 1;                \
                if (c0[d_] > c1[d_]) empty_ = 1;                                        \
            }                                                                           \
        }                                                                               \
        if (!empty_)                                                                    \
            for (int64_t cz = c0[2]; cz <= c1[2]; ++cz)                                 \
                for (int64_t cy = c0[1]; cy <= c1[1]; ++cy)                             \
                    for (int64_t cx = c0[0]; cx <= c1[0]; ++cx) {                       \
                        const uint64_t cell_ =                                          \
                            ((uint64_t)cz * (uint64_t)(g)->n[1] + (uint64_t)cy) *       \
                                (uint64_t)(g)->n[0] +                                   \
                            (uint64_t)cx;                                               \
                        for (uint64_t e_ = (g)->start[cell_]; e_ < (g)->start[cell_ + 1]; \
                             ++e_) {                                                    \
                            const uint32_t IDVAR = (g)->ids[e_];                        \
                            BODY                                                        \
                        }                                                               \
                    }                                                                   \
    } while (0)

/* Support hits of one point, sorted by centre index: the same set as
 * radius_query(p, 1/alpha) (kdtree.cpp:57-87) followed by the phi != 0
 * filter of assemble_submatrix (coo.cpp:180-183). */
static uint64_t point_hits(const grid_t* g, int dim, const double* q, const double* centres,
                           int family, double alpha, double r2, hit_t** buf, uint64_t* cap) {
    uint64_t k = 0;
    GRID_FOR_CANDIDATES(g, q, j, {
        const double d2 = dist2(dim, centres + (uint64_t)j * dim, q);
        if (d2 < r2) {
            const double v = phi_inside(family, alpha, sqrt(d2));
            if (v != 0.0) {
                if (k == *cap) {
                    *cap *= 2;
                    *buf = (hit_t*)realloc(*buf, *cap * sizeof(hit_t));
                }
                (*buf)[k].id = j;
                (*buf)[k].v = v;
                ++k;
            }
        }
    });
    sort_hits(*buf, k);
    return k;
}

/* --------------------------------------------------------------- pattern */

/* One pattern row: the ascending j >= i with dist2(c_i, c_j) < lim. */
static uint64_t pattern_row(const grid_t* g, int dim, const double* centres, uint64_t i, double lim,
                            uint32_t** row, uint64_t* cap) {
    const double* ci = centres + i * dim;
    uint64_t k = 0;
    GRID_FOR_CANDIDATES(g, ci, j, {
        if (j >= i && dist2(dim, ci, centres + (uint64_t)j * dim) < lim) {
            if (k == *cap) {
                *cap *= 2;
                *row = (uint32_t*)realloc(*row, *cap * sizeof(uint32_t));
            }
            (*row)[k++] = j;
        }
    });
    for (uint64_t a = 1; a < k; ++a) { /* insertion sort (rows are short) */
        uint32_t t = (*row)[a];
        uint64_t b = a;
        while (b > 0 && (*row)[b - 1] > t) {
            (*row)[b] = (*row)[b - 1];
            --b;
        }
        (*row)[b] = t;
    }
    return k;
}

/* Rows are independent: counted in parallel, prefix-summed, then filled in
 * parallel (the result does not depend on the thread count). */
int orc_pattern(int dim, const double* centres, uint64_t m, double alpha, uint64_t* row_ptr,
                uint32_t* cols) {
    if ((dim != 2 && dim != 3) || m == 0 || !(alpha > 0.0) || !isfinite(alpha))
        return ORC_INVALID;
    const double rad = 1.0 / alpha;
    const double two_r = 2.0 * rad;
    const double lim = two_r * two_r;
    grid_t g;
    if (grid_build(&g, dim, centres, m, two_r) != ORC_OK) return ORC_RUNTIME;
    row_ptr[0] = 0;
#pragma omp parallel
    {
        uint64_t cap = 256;
        uint32_t* row = (uint32_t*)malloc(cap * sizeof(uint32_t));
#pragma omp for schedule(dynamic, 512)
        for (int64_t i = 0; i < (int64_t)m; ++i)
            row_ptr[i + 1] = pattern_row(&g, dim, centres, (uint64_t)i, lim, &row, &cap);
        free(row);
    }
    for (uint64_t i = 0; i < m; ++i) row_ptr[i + 1] += row_ptr[i];
    if (cols) {
#pragma omp parallel
        {
            uint64_t cap = 256;
            uint32_t* row = (uint32_t*)malloc(cap * sizeof(uint32_t));
#pragma omp for schedule(dynamic, 512)
            for (int64_t i = 0; i < (int64_t)m; ++i) {
                const uint64_t k = pattern_row(&g, dim, centres, (uint64_t)i, lim, &row, &cap);
                memcpy(cols + row_ptr[i], row, k * sizeof(uint32_t));
            }
            free(row);
        }
    }
    grid_free(&g);
    return ORC_OK;
}

static int64_t find_slot(const uint64_t* row_ptr, const uint32_t* cols, uint32_t i, uint32_t j) {
    uint64_t lo = row_ptr[i], hi = row_ptr[i + 1];
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (cols[mid] < j)
            lo = mid + 1;
        else
            hi = mid;
    }
    if (lo < row_ptr[i + 1] && cols[lo] == j) return (int64_t)lo;
    return -1;
}

/* -------------------------------------------------------------- assembly */

/* Parallel without changing a single bit: points are processed in chunks;
 * first every point's sorted hit list is computed (parallel over points),
 * then the output rows are partitioned among threads and each thread walks
 * the chunk's points in ascending order, applying only the updates of its
 * own rows.  Every entry therefore receives exactly the sequential
 * (point-ascending) addition sequence of coo.cpp:80 / coo.cpp:144. */
#define ORC_CHUNK (1u << 20)

typedef struct {
    hit_t* buf;
    uint64_t len, cap;
} hitbuf_t;

int orc_assemble(int dim, const double* pts, const double* h, uint64_t n, const double* centres,
                 uint64_t m, int family, double alpha, const uint64_t* row_ptr,
                 const uint32_t* cols, double* vals, double* rhs, uint64_t* hits) {
    if ((dim != 2 && dim != 3) || m == 0 || family < 0 || family > 3 || !(alpha > 0.0) ||
        !isfinite(alpha))
        return ORC_INVALID;
    memset(vals, 0, row_ptr[m] * sizeof(double));
    memset(rhs, 0, m * sizeof(double));
    memset(hits, 0, m * sizeof(uint64_t));
    const double radius = 1.0 / alpha; /* KernelSpec::support_radius, kernel.hpp:37 */
    const double r2 = radius * radius; /* kdtree.cpp:64 */
    grid_t g;
    if (grid_build(&g, dim, centres, m, radius) != ORC_OK) return ORC_RUNTIME;
    const uint64_t chunk = n < ORC_CHUNK ? (n ? n : 1) : ORC_CHUNK;
    const hit_t** plist = (const hit_t**)malloc(chunk * sizeof(hit_t*));
    uint32_t* pk = (uint32_t*)malloc(chunk * sizeof(uint32_t));
    uint64_t* poff = (uint64_t*)malloc(chunk * sizeof(uint64_t));
    int* pthr = (int*)malloc(chunk * sizeof(int));
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    hitbuf_t* tb = (hitbuf_t*)calloc((size_t)nthr, sizeof(hitbuf_t));
    int status = ORC_OK;
    const int64_t nparts = (int64_t)nthr * 8;
    for (uint64_t c0 = 0; c0 < n && status == ORC_OK; c0 += chunk) {
        const uint64_t cn = n - c0 < chunk ? n - c0 : chunk;
#pragma omp parallel
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            hitbuf_t* B = &tb[tid];
            B->len = 0;
            uint64_t cap = 256;
            hit_t* hb = (hit_t*)malloc(cap * sizeof(hit_t));
#pragma omp for schedule(static)
            for (int64_t q = 0; q < (int64_t)cn; ++q) {
                const uint64_t p = c0 + (uint64_t)q;
                const uint64_t k = point_hits(&g, dim, pts + p * dim, centres, family, alpha, r2, &hb, &cap);
                if (B->len + k > B->cap) {
                    B->cap = (B->len + k) * 2 + 1024;
                    B->buf = (hit_t*)realloc(B->buf, B->cap * sizeof(hit_t));
                }
                memcpy(B->buf + B->len, hb, k * sizeof(hit_t));
                poff[q] = B->len;
                pthr[q] = tid;
                pk[q] = (uint32_t)k;
                B->len += k;
            }
            free(hb);
        }
        for (uint64_t q = 0; q < cn; ++q) plist[q] = tb[pthr[q]].buf + poff[q];
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t part = 0; part < nparts; ++part) {
            const uint32_t r0 = (uint32_t)((uint64_t)part * m / (uint64_t)nparts);
            const uint32_t r1 = (uint32_t)((uint64_t)(part + 1) * m / (uint64_t)nparts);
            if (r0 == r1) continue;
            for (uint64_t q = 0; q < cn; ++q) {
                const hit_t* hl = plist[q];
                const uint64_t k = pk[q];
                if (k == 0 || hl[k - 1].id < r0 || hl[0].id >= r1) continue;
                uint64_t a = 0, hi = k; /* first hit with id >= r0 */
                while (a < hi) {
                    const uint64_t mid = (a + hi) >> 1;
                    if (hl[mid].id < r0) a = mid + 1;
                    else hi = mid;
                }
                const double hp = h[c0 + q];
                for (; a < k && hl[a].id < r1; ++a) {
                    const uint32_t ca = hl[a].id;
                    const double va = hl[a].v;
                    hits[ca]++;
                    rhs[ca] += va * hp; /* coo.cpp:80 */
                    for (uint64_t b2 = a; b2 < k; ++b2) {
                        const int64_t s = find_slot(row_ptr, cols, ca, hl[b2].id);
                        if (s < 0) {
#pragma omp atomic write
                            status = ORC_RUNTIME;
                            break;
                        }
                        vals[s] += va * hl[b2].v; /* coo.cpp:144 */
                    }
                }
            }
        }
    }
    for (int t = 0; t < nthr; ++t) free(tb[t].buf);
    free(tb);
    free(plist);
    free(pk);
    free(poff);
    free(pthr);
    grid_free(&g);
    return status;
}

/* ------------------------------------------------------------ evaluation */

int orc_evaluate(int dim, const double* centres, uint64_t m, const double* w, int family,
                 double alpha, const double* q, uint64_t nq, double* f) {
    if ((dim != 2 && dim != 3) || m == 0 || family < 0 || family > 3 || !(alpha > 0.0) ||
        !isfinite(alpha))
        return ORC_INVALID;
    const double radius = 1.0 / alpha;
    const double r2 = radius * radius;
    grid_t g;
    if (grid_build(&g, dim, centres, m, radius) != ORC_OK) return ORC_RUNTIME;
#pragma omp parallel
    {
        uint64_t cap = 256;
        hit_t* hb = (hit_t*)malloc(cap * sizeof(hit_t));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < (int64_t)nq; ++i) {
            const uint64_t k = point_hits(&g, dim, q + (uint64_t)i * dim, centres, family, alpha, r2, &hb, &cap);
            double acc = 0.0;
            for (uint64_t a = 0; a < k; ++a) acc += w[hb[a].id] * hb[a].v; /* model.cpp:63-64 */
            f[i] = acc;
        }
        free(hb);
    }
    grid_free(&g);
    return ORC_OK;
}

int orc_error_report(const double* f, const double* h, uint64_t n, double* mae, double* deviation,
                     double* rel_pct, double* rms, double* max_abs) {
    if (n == 0) return ORC_INVALID; /* model.cpp:198 */
    double abs_sum = 0.0, norm_sum = 0.0, sq_sum = 0.0, mx = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double e = f[i] - h[i];
        abs_sum += fabs(e);
        norm_sum += fabs(h[i]);
        sq_sum += e * e;
        if (fabs(e) > mx) mx = fabs(e);
    }
    const double dn = (double)n;
    const double m_ae = abs_sum / dn;
    double var_sum = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double d = fabs(f[i] - h[i]) - m_ae;
        var_sum += d * d;
    }
    *mae = m_ae;
    *deviation = var_sum / dn;
    const double normalizer = norm_sum / dn;
    *rel_pct = normalizer > 0.0 ? 100.0 * m_ae / normalizer : 0.0;
    *rms = sqrt(sq_sum / dn);
    *max_abs = mx;
    return ORC_OK;
}

/* ----------------------------------------------------------------- solve */

/* Returns -1 on success, else the failing pivot index. */
static int64_t cholesky_inplace(uint64_t n, double* a) {
    for (uint64_t j = 0; j < n; ++j) {
        double d = a[j * n + j];
        for (uint64_t k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
        if (!(d > 0.0) || !isfinite(d)) return (int64_t)j;
        const double ljj = sqrt(d);
        a[j * n + j] = ljj;
        for (uint64_t i = j + 1; i < n; ++i) {
            double s = a[i * n + j];
            const double* li = a + i * n;
            const double* lj = a + j * n;
            for (uint64_t k = 0; k < j; ++k) s -= li[k] * lj[k];
            a[i * n + j] = s / ljj;
        }
    }
    return -1;
}

int orc_cholesky_solve(uint64_t side, const double* b_dense, const double* rhs, double* x,
                       double* ridge_lambda, int* attempts, int64_t* bad_pivot) {
    if (side == 0) return ORC_INVALID;
    static const double lambdas[] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6}; /* solver.cpp:298 */
    double trace = 0.0;
    for (uint64_t i = 0; i < side; ++i) trace += b_dense[i * side + i];
    const double mean_diag = trace / (double)side; /* solver.cpp:296 */
    double* a = (double*)malloc(side * side * sizeof(double));
    if (!a) return ORC_RUNTIME;
    *attempts = 0;
    *bad_pivot = -1;
    for (int li = 0; li < 6; ++li) {
        memcpy(a, b_dense, side * side * sizeof(double));
        if (lambdas[li] > 0.0)
            for (uint64_t i = 0; i < side; ++i) a[i * side + i] += lambdas[li] * mean_diag;
        ++*attempts;
        const int64_t piv = cholesky_inplace(side, a);
        if (piv < 0) {
            for (uint64_t i = 0; i < side; ++i) { /* L y = rhs */
                double s = rhs[i];
                for (uint64_t k = 0; k < i; ++k) s -= a[i * side + k] * x[k];
                x[i] = s / a[i * side + i];
            }
            for (uint64_t ii = side; ii-- > 0;) { /* L^T x = y */
                double s = x[ii];
                for (uint64_t k = ii + 1; k < side; ++k) s -= a[k * side + ii] * x[k];
                x[ii] = s / a[ii * side + ii];
            }
            *ridge_lambda = lambdas[li];
            free(a);
            return ORC_OK;
        }
        *bad_pivot = piv;
    }
    free(a);
    return ORC_RUNTIME; /* solver.cpp:316-322 */
}

/* y = (B + shift I) x for symmetric B stored as upper CSR. */
static void sym_spmv(uint64_t m, const uint64_t* rp, const uint32_t* cols, const double* vals,
                     double shift, const double* x, double* y) {
    for (uint64_t i = 0; i < m; ++i) y[i] = shift * x[i];
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t e = rp[i]; e < rp[i + 1]; ++e) {
            const uint32_t j = cols[e];
            y[i] += vals[e] * x[j];
            if (j != i) y[j] += vals[e] * x[i];
        }
}

int orc_pcg(uint64_t m, const uint64_t* rp, const uint32_t* cols, const double* vals,
            const double* rhs, double shift, double tol, int max_iter, double* x, int* iters,
            double* rel_res) {
    double* r = (double*)malloc(m * sizeof(double));
    double* z = (double*)malloc(m * sizeof(double));
    double* p = (double*)malloc(m * sizeof(double));
    double* q = (double*)malloc(m * sizeof(double));
    double* dinv = (double*)malloc(m * sizeof(double));
    int status = ORC_OK;
    double bb = 0.0;
    for (uint64_t i = 0; i < m; ++i) {
        const int64_t s = find_slot(rp, cols, (uint32_t)i, (uint32_t)i);
        const double d = (s >= 0 ? vals[s] : 0.0) + shift;
        if (!(d > 0.0)) status = ORC_RUNTIME;
        dinv[i] = 1.0 / d;
        x[i] = 0.0;
        r[i] = rhs[i];
        bb += rhs[i] * rhs[i];
    }
    *iters = 0;
    *rel_res = 0.0;
    if (status != ORC_OK || bb == 0.0) goto done;
    double rz = 0.0;
    for (uint64_t i = 0; i < m; ++i) {
        z[i] = r[i] * dinv[i];
        p[i] = z[i];
        rz += r[i] * z[i];
    }
    const double stop = tol * tol * bb;
    double rr = bb;
    int it = 0;
    while (it < max_iter && rr > stop) {
        sym_spmv(m, rp, cols, vals, shift, p, q);
        double pq = 0.0;
        for (uint64_t i = 0; i < m; ++i) pq += p[i] * q[i];
        if (!(pq > 0.0)) {
            status = ORC_RUNTIME;
            break;
        }
        const double alpha = rz / pq;
        double rz_new = 0.0;
        rr = 0.0;
        for (uint64_t i = 0; i < m; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * q[i];
            z[i] = r[i] * dinv[i];
            rz_new += r[i] * z[i];
            rr += r[i] * r[i];
        }
        const double beta = rz_new / rz;
        rz = rz_new;
        for (uint64_t i = 0; i < m; ++i) p[i] = z[i] + beta * p[i];
        ++it;
    }
    *iters = it;
    *rel_res = sqrt(rr / bb);
    if (status == ORC_OK && rr > stop) status = ORC_RUNTIME;
done:
    free(r);
    free(z);
    free(p);
    free(q);
    free(dinv);
    return status;
}

void orc_densify(uint64_t m, const uint64_t* rp, const uint32_t* cols, const double* vals,
                 double* dense) {
    memset(dense, 0, m * m * sizeof(double));
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t e = rp[i]; e < rp[i + 1]; ++e) {
            dense[i * m + cols[e]] = vals[e];
            dense[(uint64_t)cols[e] * m + i] = vals[e];
        }
}

/* ------------------------------------------------ linear-polynomial border */

/* The bordered system's extra blocks (solver.cpp:189-207, 238-262) with
 * P = [x, y, (z), 1], T = dim + 1: atp[t*m + j] = sum_p A[p][j] * P[p][t]
 * accumulated over the points in ascending order (the reference streams the
 * triplets column by column, rows ascending), ptp = P^T P and pth = P^T h in
 * one pass over every point with separate multiply/add. */
int orc_border(int dim, const double* pts, const double* h, uint64_t n, const double* centres,
               uint64_t m, int family, double alpha, double* atp, double* ptp, double* pth) {
    if ((dim != 2 && dim != 3) || m == 0 || family < 0 || family > 3 || !(alpha > 0.0) ||
        !isfinite(alpha))
        return ORC_INVALID;
    const int T = dim + 1;
    memset(atp, 0, (size_t)T * m * sizeof(double));
    const double radius = 1.0 / alpha;
    const double r2 = radius * radius;
    grid_t g;
    if (grid_build(&g, dim, centres, m, radius) != ORC_OK) return ORC_RUNTIME;
    uint64_t cap = 256;
    hit_t* hb = (hit_t*)malloc(cap * sizeof(hit_t));
    for (uint64_t p = 0; p < n; ++p) {
        const double* q = pts + p * dim;
        const uint64_t k = point_hits(&g, dim, q, centres, family, alpha, r2, &hb, &cap);
        for (uint64_t a = 0; a < k; ++a) {
            const uint32_t j = hb[a].id;
            const double v = hb[a].v;
            for (int t = 0; t < dim; ++t) atp[(uint64_t)t * m + j] += v * q[t]; /* solver.cpp:198-200 */
            atp[(uint64_t)dim * m + j] += v;                                   /* solver.cpp:201 */
        }
    }
    free(hb);
    grid_free(&g);
    double s[4][4], sh[4];
    memset(s, 0, sizeof(s));
    memset(sh, 0, sizeof(sh));
    for (uint64_t p = 0; p < n; ++p) { /* solver.cpp:238-250 */
        double v[4];
        for (int t = 0; t < dim; ++t) v[t] = pts[p * dim + t];
        v[dim] = 1.0;
        for (int a = 0; a < T; ++a) {
            for (int b = a; b < T; ++b) s[a][b] += v[a] * v[b];
            sh[a] += v[a] * h[p];
        }
    }
    for (int a = 0; a < T; ++a) {
        for (int b = 0; b < T; ++b) ptp[a * T + b] = a <= b ? s[a][b] : s[b][a];
        pth[a] = sh[a];
    }
    ptp[T * T - 1] = (double)n; /* the reference stores n, not a running sum */
    return ORC_OK;
}

/* evaluate with the polynomial term (model.cpp:65-68): f += a0 x + a1 y (+ a2 z) + a_T-1,
 * the expression evaluated left to right, unfused. */
int orc_evaluate_poly(int dim, const double* centres, uint64_t m, const double* w, const double* a,
                      int family, double alpha, const double* q, uint64_t nq, double* f) {
    const int st = orc_evaluate(dim, centres, m, w, family, alpha, q, nq, f);
    if (st != ORC_OK) return st;
    for (uint64_t i = 0; i < nq; ++i) {
        const double* p = q + i * dim;
        double t = a[0] * p[0] + a[1] * p[1];
        if (dim == 3) t = t + a[2] * p[2];
        t = t + a[dim];
        f[i] += t;
    }
    return ORC_OK;
}
