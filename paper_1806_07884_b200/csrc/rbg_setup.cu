// rbg_setup.cu -- K1 (centre binning) + K2 (symbolic pattern) for a centre set.
//
// Replaces what the reference does per assembly with radius queries
// (assemble_submatrix, coo.cpp:166-192 over PointIndex, kdtree.cpp:57-87) and
// the dense normal-matrix layout (solver.cpp:151-156):
//   * a uniform tile grid over the centres' bounding box grown by the support
//     radius 1/alpha; every tile gets the ascending list of centres whose
//     support can reach it (a superset of every point-in-tile hit set);
//   * the upper-triangle CSR pattern of A^T A: pairs i <= j with
//     dist2(c_i, c_j) < (2/alpha)^2 (the predicate every co-supported pair
//     satisfies), columns ascending; plus the symmetric full pattern and the
//     full->upper slot map the solver uses;
//   * slot maps (tile_map_kernel): per tile list, the packed upper-triangle
//     map local (a,b) -> offset of column c_b within upper row c_a, so the
//     numeric kernel flushes without searching (used by rbg_layout.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

constexpr uint64_t kMaxTiles = 1ull << 25;
constexpr double kTileMargin = 1e-6;  // relative, conservative rect growth

struct TileTestDev {
    GridDev g;
    double edge, margin, r, lim;  // lim = r^2 (1 + 1e-6)
};

// Centres -> the tiles whose (grown) rectangle lies within the support radius.
template <int DIM, bool FILL>
__global__ void tile_lists_kernel(const double* __restrict__ c, uint64_t m, TileTestDev t,
                                  uint32_t* __restrict__ count, const uint64_t* __restrict__ ptr,
                                  uint32_t* __restrict__ ids) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double cc[3] = {c[i * DIM], c[i * DIM + 1], DIM == 3 ? c[i * DIM + 2] : 0.0};
        const double lo[3] = {t.g.lo0, t.g.lo1, t.g.lo2};
        const int64_t n[3] = {t.g.n0, t.g.n1, t.g.n2};
        int64_t a0[3] = {0, 0, 0}, a1[3] = {0, 0, 0};
        for (int d = 0; d < DIM; ++d) {
            int64_t s = (int64_t)floor((cc[d] - t.r - lo[d]) / t.edge) - 1;
            int64_t e = (int64_t)floor((cc[d] + t.r - lo[d]) / t.edge) + 1;
            a0[d] = s < 0 ? 0 : s;
            a1[d] = e >= n[d] ? n[d] - 1 : e;
        }
        for (int64_t iz = a0[2]; iz <= a1[2]; ++iz)
            for (int64_t iy = a0[1]; iy <= a1[1]; ++iy)
                for (int64_t ix = a0[0]; ix <= a1[0]; ++ix) {
                    const int64_t idx[3] = {ix, iy, iz};
                    double d2 = 0.0;
                    for (int d = 0; d < DIM; ++d) {
                        const double rlo = lo[d] + (double)idx[d] * t.edge - t.margin;
                        const double rhi = lo[d] + (double)(idx[d] + 1) * t.edge + t.margin;
                        const double gap = cc[d] < rlo ? rlo - cc[d] : (cc[d] > rhi ? cc[d] - rhi : 0.0);
                        d2 += gap * gap;
                    }
                    if (d2 < t.lim) {
                        const uint64_t tile = ((uint64_t)iz * (uint64_t)n[1] + (uint64_t)iy) *
                                                  (uint64_t)n[0] +
                                              (uint64_t)ix;
                        const uint32_t k = atomicAdd(&count[tile], 1u);
                        if (FILL) ids[ptr[tile] + k] = (uint32_t)i;
                    }
                }
    }
}

// Full symmetric pattern rows: all j with dist2(c_i, c_j) < lim, via a host-
// built cell grid of edge >= 2r (3^DIM neighbour cells).
struct CellDev {
    double lo0, lo1, lo2, inv_edge;
    int64_t n0, n1, n2;
};

template <int DIM, bool FILL>
__global__ void pattern_rows_kernel(const double* __restrict__ c, uint64_t m, CellDev g,
                                    const uint64_t* __restrict__ cell_ptr,
                                    const uint32_t* __restrict__ cell_ids, double lim,
                                    uint32_t* __restrict__ row_len,
                                    const uint64_t* __restrict__ fptr, uint32_t* __restrict__ fcols) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = c[i * DIM], y = c[i * DIM + 1], z = DIM == 3 ? c[i * DIM + 2] : 0.0;
        const double lo[3] = {g.lo0, g.lo1, g.lo2};
        const int64_t n[3] = {g.n0, g.n1, g.n2};
        const double v[3] = {x, y, z};
        int64_t a0[3] = {0, 0, 0}, a1[3] = {0, 0, 0};
        for (int d = 0; d < DIM; ++d) {
            int64_t cc = (int64_t)floor((v[d] - lo[d]) * g.inv_edge);
            cc = cc < 0 ? 0 : (cc >= n[d] ? n[d] - 1 : cc);
            a0[d] = cc - 1 < 0 ? 0 : cc - 1;
            a1[d] = cc + 1 >= n[d] ? n[d] - 1 : cc + 1;
        }
        uint32_t k = 0;
        const uint64_t base = FILL ? fptr[i] : 0;
        for (int64_t iz = a0[2]; iz <= a1[2]; ++iz)
            for (int64_t iy = a0[1]; iy <= a1[1]; ++iy)
                for (int64_t ix = a0[0]; ix <= a1[0]; ++ix) {
                    const uint64_t cell =
                        ((uint64_t)iz * (uint64_t)n[1] + (uint64_t)iy) * (uint64_t)n[0] + (uint64_t)ix;
                    for (uint64_t e = cell_ptr[cell]; e < cell_ptr[cell + 1]; ++e) {
                        const uint32_t j = cell_ids[e];
                        const double d2 = dist2_of<DIM>(x, y, z, c[(uint64_t)j * DIM],
                                                        c[(uint64_t)j * DIM + 1],
                                                        DIM == 3 ? c[(uint64_t)j * DIM + 2] : 0.0);
                        if (d2 < lim) {
                            if (FILL) fcols[base + k] = j;
                            ++k;
                        }
                    }
                }
        if (!FILL) row_len[i] = k;
    }
}

// Position of the diagonal in each sorted full row -> upper row length.
__global__ void upper_len_kernel(const uint64_t* __restrict__ fptr,
                                 const uint32_t* __restrict__ fcols, uint64_t m,
                                 uint32_t* __restrict__ diag_pos, uint32_t* __restrict__ ulen) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = fptr[i], hi = fptr[i + 1];
        const uint64_t b = lo, e = hi;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (fcols[mid] < (uint32_t)i) lo = mid + 1; else hi = mid;
        }
        diag_pos[i] = (uint32_t)(lo - b);
        ulen[i] = (uint32_t)(e - lo);
    }
}

__global__ void upper_fill_kernel(const uint64_t* __restrict__ fptr,
                                  const uint32_t* __restrict__ fcols, uint64_t m,
                                  const uint32_t* __restrict__ diag_pos,
                                  const uint64_t* __restrict__ uptr, uint32_t* __restrict__ ucols) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t src = fptr[i] + diag_pos[i];
        const uint64_t len = fptr[i + 1] - src;
        for (uint64_t k = 0; k < len; ++k) ucols[uptr[i] + k] = fcols[src + k];
    }
}

__device__ __forceinline__ uint64_t find_in_row(const uint32_t* cols, uint64_t lo, uint64_t hi,
                                                uint32_t key) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (cols[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// full entry (i, j) -> upper slot of (min, max).
__global__ void full_to_upper_kernel(const uint64_t* __restrict__ fptr,
                                     const uint32_t* __restrict__ fcols, uint64_t m,
                                     const uint32_t* __restrict__ diag_pos,
                                     const uint64_t* __restrict__ uptr,
                                     const uint32_t* __restrict__ ucols, uint64_t* __restrict__ f2u) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = fptr[i] + diag_pos[i];
        for (uint64_t e = fptr[i]; e < fptr[i + 1]; ++e) {
            const uint32_t j = fcols[e];
            if (e >= d) {
                f2u[e] = uptr[i] + (e - d);
            } else {
                f2u[e] = find_in_row(ucols, uptr[j], uptr[j + 1], (uint32_t)i);
            }
        }
    }
}

// Bounding box of the centres: per-warp min/max, then one atomic per warp on
// an order-preserving integer image of each double.
__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
inline double ord_val(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    std::memcpy(&v, &b, sizeof v);
    return v;
}

template <int DIM>
__global__ void bbox_kernel(const double* __restrict__ c, uint64_t m, unsigned long long* __restrict__ out) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        for (int d = 0; d < DIM; ++d) {
            const double v = c[i * DIM + d];
            lo[d] = fmin(lo[d], v);
            hi[d] = fmax(hi[d], v);
        }
    for (int d = 0; d < DIM; ++d)
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int d = 0; d < DIM; ++d) {
            atomicMin(&out[d], ord_key(lo[d]));
            atomicMax(&out[3 + d], ord_key(hi[d]));
        }
}

// Centres -> cells of edge >= 2r (the K2 neighbour grid): counting sort on
// the cell key (count, scan, scatter); the order inside a cell is irrelevant
// because every pattern row is sorted afterwards.
template <int DIM, bool FILL>
__global__ void cell_bin_kernel(const double* __restrict__ c, uint64_t m, CellDev g,
                                uint32_t* __restrict__ count, const uint64_t* __restrict__ ptr,
                                uint32_t* __restrict__ ids) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double lo[3] = {g.lo0, g.lo1, g.lo2};
        const int64_t n[3] = {g.n0, g.n1, g.n2};
        uint64_t k = 0;
        for (int d = DIM - 1; d >= 0; --d) {
            int64_t cc = (int64_t)floor((c[i * DIM + d] - lo[d]) * g.inv_edge);
            cc = cc < 0 ? 0 : (cc >= n[d] ? n[d] - 1 : cc);
            k = k * (uint64_t)n[d] + (uint64_t)cc;
        }
        const uint32_t pos = atomicAdd(&count[k], 1u);
        if (FILL) ids[ptr[k] + pos] = (uint32_t)i;
    }
}

// Slot maps: per (tile, local row a), the offsets of the tile's columns b >= a within upper
// row c_a.  A warp takes 32 consecutive rows: every lane resolves its own row (tile by binary
// search over cptr, CSR row bounds), then the warp walks the 32 rows one at a time, lanes =
// columns: one binary search per entry in the (L1-resident, few hundred ids) upper row and
// coalesced 16-bit stores.  (One thread per row merging the two ascending lists: 7-8 ms per
// call at cfg3 / cfg5, scattered 2-byte stores and divergent trip counts.)
__global__ void tile_map_kernel(const uint64_t* __restrict__ cptr, uint64_t n_tiles,
                                const uint32_t* __restrict__ cids, uint64_t total,
                                const uint64_t* __restrict__ mptr, const uint64_t* __restrict__ uptr,
                                const uint32_t* __restrict__ ucols, uint16_t* __restrict__ map) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t e0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32ull; e0 < total;
         e0 += nw * 32ull) {
        const uint64_t e = e0 + lane;
        uint64_t c0 = 0, rb = 0, re = 0, mo = 0;
        uint32_t L = 0, a = 0;
        if (e < total) {
            uint64_t lo = 0, hi = n_tiles;  // tile = last t with cptr[t] <= e
            while (hi - lo > 1) {
                const uint64_t mid = (lo + hi) >> 1;
                if (cptr[mid] <= e) lo = mid; else hi = mid;
            }
            c0 = cptr[lo];
            L = (uint32_t)(cptr[lo + 1] - c0);
            a = (uint32_t)(e - c0);
            const uint32_t ga = cids[e];
            rb = uptr[ga];
            re = uptr[ga + 1];
            mo = mptr[lo] + tri_index(a, a, L);
        }
        const int nrows = (int)(total - e0 < 32ull ? total - e0 : 32ull);
        for (int r = 0; r < nrows; ++r) {
            const uint64_t rc0 = __shfl_sync(0xffffffffu, c0, r), rrb = __shfl_sync(0xffffffffu, rb, r);
            const uint64_t rre = __shfl_sync(0xffffffffu, re, r), rmo = __shfl_sync(0xffffffffu, mo, r);
            const uint32_t rL = __shfl_sync(0xffffffffu, L, r), ra = __shfl_sync(0xffffffffu, a, r);
            uint16_t* out = map + rmo;
            for (uint32_t b = ra + lane; b < rL; b += 32) {
                const uint32_t gb = cids[rc0 + b];
                uint64_t l = rrb, h = rre;
                while (l < h) {
                    const uint64_t mid = (l + h) >> 1;
                    if (ucols[mid] < gb) l = mid + 1; else h = mid;
                }
                out[b - ra] = (l < rre && ucols[l] == gb) ? (uint16_t)(l - rrb) : (uint16_t)0xffff;
            }
        }
    }
}

}  // namespace

// Centre lists of every tile of grid g (ascending ids): count, scan, fill, sort.
void tile_lists(rbg_ctx* ctx, const TileGrid& g, DevBuf<uint32_t>& count, DevBuf<uint64_t>& cptr,
                DevBuf<uint32_t>& cids, std::vector<uint64_t>& host_cptr) {
    cudaStream_t st = ctx->stream;
    const uint64_t nt = g.count, m = ctx->m;
    count.reserve(nt + 1);
    cptr.reserve(nt + 1);
    RBG_CUDA(cudaMemsetAsync(count.p, 0, (nt + 1) * sizeof(uint32_t), st));
    TileTestDev tt{grid_dev(g), g.edge, g.edge * kTileMargin, ctx->radius, ctx->r2 * (1.0 + 1e-6)};
    const unsigned cb = blocks_for(m, 128);
    if (g.dim == 2)
        tile_lists_kernel<2, false><<<cb, 128, 0, st>>>(ctx->centres.p, m, tt, count.p, nullptr, nullptr);
    else
        tile_lists_kernel<3, false><<<cb, 128, 0, st>>>(ctx->centres.p, m, tt, count.p, nullptr, nullptr);
    RBG_CHECK_LAUNCH(ctx);
    exclusive_scan_u32_to_u64(ctx, count.p, cptr.p, nt);
    host_cptr.assign(nt + 1, 0);
    RBG_CUDA(cudaMemcpyAsync(host_cptr.data(), cptr.p, (nt + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    const uint64_t total = host_cptr[nt];
    cids.reserve(std::max<uint64_t>(total, 1));
    RBG_CUDA(cudaMemsetAsync(count.p, 0, (nt + 1) * sizeof(uint32_t), st));
    if (g.dim == 2)
        tile_lists_kernel<2, true><<<cb, 128, 0, st>>>(ctx->centres.p, m, tt, count.p, cptr.p, cids.p);
    else
        tile_lists_kernel<3, true><<<cb, 128, 0, st>>>(ctx->centres.p, m, tt, count.p, cptr.p, cids.p);
    RBG_CHECK_LAUNCH(ctx);
    uint32_t max_l = 0;
    for (uint64_t t = 0; t < nt; ++t) max_l = std::max<uint32_t>(max_l, (uint32_t)(host_cptr[t + 1] - host_cptr[t]));
    segmented_sort_u32(ctx, cids.p, cptr.p, nt, max_l);
}

// Packed upper-triangle slot maps of every tile's centre list (needs the pattern).
void slot_maps(rbg_ctx* ctx, const uint64_t* cptr, uint64_t n_tiles, const uint32_t* cids, uint64_t total_ids,
               const uint64_t* mptr, uint16_t* map) {
    if (total_ids == 0) return;
    tile_map_kernel<<<blocks_for(total_ids, 256), 256, 0, ctx->stream>>>(cptr, n_tiles, cids, total_ids, mptr,
                                                                          ctx->uptr.p, ctx->ucols.p, map);
    RBG_CHECK_LAUNCH(ctx);
}

void ensure_grid(rbg_ctx* ctx) {
    if (ctx->have_grid) return;
    RBG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    setup_centres(ctx);
    RBG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    RBG_CUDA(cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    RBG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->setup_ms += ms;
    ctx->have_grid = true;
}

void setup_centres(rbg_ctx* ctx) {
    const int dim = ctx->dim;
    const uint64_t m = ctx->m;
    cudaStream_t st = ctx->stream;
    ctx->bj_built = false;  // solve order and preconditioner pattern follow the centre set
    ctx->fs_built = false;
    ctx->band = BandPlan();  // so does the banded-solve ordering

    // ---- bounding box (device reduction) + tile grid plan -------------------
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    {
        DevBuf<unsigned long long> bb;
        bb.reserve(6);
        unsigned long long init[6];
        for (int d = 0; d < 3; ++d) {
            init[d] = ~0ull;
            init[3 + d] = 0ull;
        }
        RBG_CUDA(cudaMemcpyAsync(bb.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
        const unsigned bbk = blocks_for(m, 256, 148u * 4u);
        if (dim == 2) bbox_kernel<2><<<bbk, 256, 0, st>>>(ctx->centres.p, m, bb.p);
        else bbox_kernel<3><<<bbk, 256, 0, st>>>(ctx->centres.p, m, bb.p);
        RBG_CHECK_LAUNCH(ctx);
        unsigned long long hb[6];
        RBG_CUDA(cudaMemcpyAsync(hb, bb.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        for (int d = 0; d < dim; ++d) {
            lo[d] = ord_val(hb[d]);
            hi[d] = ord_val(hb[3 + d]);
        }
    }
    const double r = ctx->radius;
    TileGrid g;
    g.dim = dim;
    double edge = r / 4.0;
    for (;;) {
        uint64_t total = 1;
        bool over = false;
        for (int d = 0; d < 3; ++d) {
            if (d < dim) {
                g.lo[d] = lo[d] - r * (1.0 + 1e-7) - edge * 1e-3;
                const double span = (hi[d] + r * (1.0 + 1e-7) + edge * 1e-3) - g.lo[d];
                const double nd = std::max(1.0, std::ceil(span / edge));
                if (nd > 1e9) over = true;
                g.n[d] = (int64_t)nd;
            } else {
                g.lo[d] = 0.0;
                g.n[d] = 1;
            }
            total *= (uint64_t)g.n[d];
            if (total > kMaxTiles) over = true;
        }
        if (!over) {
            g.count = total;
            break;
        }
        edge *= 1.25;
    }
    g.edge = edge;
    g.inv_edge = 1.0 / edge;
    ctx->grid = g;
    const uint64_t nt = g.count;

    // ---- K1: query-tile centre lists (evaluation / support counts) ----------
    std::vector<uint64_t> cptr;
    tile_lists(ctx, g, ctx->tile_count, ctx->tile_cptr, ctx->tile_cids, cptr);
    uint32_t max_l = 0;
    for (uint64_t t = 0; t < nt; ++t) max_l = std::max<uint32_t>(max_l, (uint32_t)(cptr[t + 1] - cptr[t]));
    ctx->max_tile_centres = max_l;
    for (int d = 0; d < 3; ++d) {
        ctx->bbox_lo[d] = lo[d];
        ctx->bbox_hi[d] = hi[d];
    }
    ctx->have_pattern = false;  // built at the first call that needs it (setup_pattern)
    ctx->lay = AsmLayout();     // rebuilt at the next assembly for this centre set
}

// K2: the symbolic pattern of the centre set (upper + full CSR, full->upper map).
void setup_pattern(rbg_ctx* ctx) {
    const int dim = ctx->dim;
    const uint64_t m = ctx->m;
    cudaStream_t st = ctx->stream;
    const double r = ctx->radius;
    const double* lo = ctx->bbox_lo;
    const double* hi = ctx->bbox_hi;
    const unsigned cb = blocks_for(m, 128);
    const double two_r = 2.0 * r;
    const double lim = two_r * two_r;
    double cedge = two_r * (1.0 + 1e-9);
    int64_t cn[3] = {1, 1, 1};
    uint64_t ncell = 1;
    for (;;) {
        ncell = 1;
        for (int d = 0; d < 3; ++d) {
            cn[d] = d < dim ? (int64_t)std::floor((hi[d] - lo[d]) / cedge) + 1 : 1;
            ncell *= (uint64_t)cn[d];
        }
        if (ncell <= std::max<uint64_t>(4 * m, 1u << 16)) break;
        cedge *= 1.5;
    }
    const double cinv = 1.0 / cedge;
    CellDev cd{lo[0], lo[1], lo[2], cinv, cn[0], cn[1], cn[2]};
    DevBuf<uint64_t> d_cell_ptr;
    DevBuf<uint32_t> d_cell_ids, d_len;
    DevBuf<uint32_t>& d_diag = ctx->fdiag;  // kept: the full -> upper slot map is built on demand (ensure_f2u)
    d_cell_ptr.reserve(ncell + 1);
    d_cell_ids.reserve(m);
    d_len.reserve(std::max<uint64_t>(m, ncell) + 1);
    d_diag.reserve(m);
    RBG_CUDA(cudaMemsetAsync(d_len.p, 0, (ncell + 1) * sizeof(uint32_t), st));
    if (dim == 2) cell_bin_kernel<2, false><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_len.p, nullptr, nullptr);
    else cell_bin_kernel<3, false><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_len.p, nullptr, nullptr);
    RBG_CHECK_LAUNCH(ctx);
    exclusive_scan_u32_to_u64(ctx, d_len.p, d_cell_ptr.p, ncell);
    RBG_CUDA(cudaMemsetAsync(d_len.p, 0, (ncell + 1) * sizeof(uint32_t), st));
    if (dim == 2) cell_bin_kernel<2, true><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_len.p, d_cell_ptr.p, d_cell_ids.p);
    else cell_bin_kernel<3, true><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_len.p, d_cell_ptr.p, d_cell_ids.p);
    RBG_CHECK_LAUNCH(ctx);
    ctx->fptr.reserve(m + 1);
    if (dim == 2)
        pattern_rows_kernel<2, false><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_cell_ptr.p,
                                                          d_cell_ids.p, lim, d_len.p, nullptr, nullptr);
    else
        pattern_rows_kernel<3, false><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_cell_ptr.p,
                                                          d_cell_ids.p, lim, d_len.p, nullptr, nullptr);
    RBG_CHECK_LAUNCH(ctx);
    exclusive_scan_u32_to_u64(ctx, d_len.p, ctx->fptr.p, m);
    std::vector<uint64_t> hfptr(m + 1);
    RBG_CUDA(cudaMemcpyAsync(hfptr.data(), ctx->fptr.p, (m + 1) * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    ctx->nnz_full = hfptr[m];
    uint32_t max_row = 0;
    for (uint64_t i = 0; i < m; ++i) max_row = std::max<uint32_t>(max_row, (uint32_t)(hfptr[i + 1] - hfptr[i]));
    ctx->max_full_row = max_row;
    if (max_row >= 0xffff)
        throw Error(RBG_INVALID_ARGUMENT, "pattern row of " + std::to_string(max_row) +
                                              " centres exceeds the 65534-entry slot-map limit");
    ctx->fcols.reserve(ctx->nnz_full);
    if (dim == 2)
        pattern_rows_kernel<2, true><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_cell_ptr.p,
                                                         d_cell_ids.p, lim, nullptr, ctx->fptr.p,
                                                         ctx->fcols.p);
    else
        pattern_rows_kernel<3, true><<<cb, 128, 0, st>>>(ctx->centres.p, m, cd, d_cell_ptr.p,
                                                         d_cell_ids.p, lim, nullptr, ctx->fptr.p,
                                                         ctx->fcols.p);
    RBG_CHECK_LAUNCH(ctx);
    segmented_sort_u32(ctx, ctx->fcols.p, ctx->fptr.p, m, max_row);
    upper_len_kernel<<<cb, 128, 0, st>>>(ctx->fptr.p, ctx->fcols.p, m, d_diag.p, d_len.p);
    RBG_CHECK_LAUNCH(ctx);
    ctx->uptr.reserve(m + 1);
    exclusive_scan_u32_to_u64(ctx, d_len.p, ctx->uptr.p, m);
    RBG_CUDA(cudaMemcpyAsync(&ctx->nnz_upper, ctx->uptr.p + m, sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    ctx->ucols.reserve(ctx->nnz_upper);
    upper_fill_kernel<<<cb, 128, 0, st>>>(ctx->fptr.p, ctx->fcols.p, m, d_diag.p, ctx->uptr.p,
                                          ctx->ucols.p);
    RBG_CHECK_LAUNCH(ctx);
    ctx->have_f2u = false;

    // ---- system + point workspace sized for this centre set ----------------
    ctx->sys.reserve(ctx->nnz_upper + 2 * m + 4 * m + 20);  // room for the polynomial border
    // counters: allocated (8) by rbg_create
    RBG_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 4 * sizeof(unsigned long long), st));
    RBG_CUDA(cudaStreamSynchronize(st));
    ctx->have_pattern = true;
}

// Full CSR entry -> upper CSR slot, for the solves that run in centre order
// (point Jacobi, the bordered system, the banded LLT's residual); the default
// solve carries its own map in Morton order (pf2u) and never needs this one.
void ensure_f2u(rbg_ctx* ctx) {
    if (ctx->have_f2u) return;
    ctx->f2u.reserve(ctx->nnz_full);
    full_to_upper_kernel<<<blocks_for(ctx->m, 128), 128, 0, ctx->stream>>>(ctx->fptr.p, ctx->fcols.p, ctx->m,
                                                                           ctx->fdiag.p, ctx->uptr.p, ctx->ucols.p,
                                                                           ctx->f2u.p);
    RBG_CHECK_LAUNCH(ctx);
    ctx->have_f2u = true;
}

}  // namespace rbg
