// rbg_layout.cu -- the two-level assembly layout (super-tiles of S^d sub-tiles)
// for one centre set and a point density.
//
// Everything here depends only on the centres (and on the point density, which
// picks the sub-tile edge); it is built once at the first assembly after
// rbg_set_centres and reused by every later assembly with that centre set.
//   * super-tile centre lists: centres whose support reaches the super-tile
//     (a conservative rectangle-distance test, as tile_lists_kernel);
//   * per super-tile packed upper-triangle slot map (local (A,B) -> offset of
//     centre B in upper CSR row A, 0xFFFF when the pair is not in the pattern);
//   * per sub-tile centre lists as super-local indices (ascending);
//   * per super-tile blobs grouped into launch buckets by (L_S, max L_sub).
// Reference semantics are unaffected: the lists are supersets of every point's
// hit set (kdtree.cpp:64,74 strict radius), the exact test happens per pair in
// the numeric kernel.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>

#include "rbg_internal.cuh"

namespace rbg {

uint32_t assembly_min_smem(int dim, int lsb, int lsub_cap, int sd);  // rbg_assemble.cu
// defined in rbg_setup.cu
void tile_lists(rbg_ctx* ctx, const TileGrid& g, DevBuf<uint32_t>& count, DevBuf<uint64_t>& cptr,
                DevBuf<uint32_t>& cids, std::vector<uint64_t>& host_cptr);
void slot_maps(rbg_ctx* ctx, const uint64_t* cptr, uint64_t n_tiles, const uint32_t* cids,
               uint64_t total_ids, const uint64_t* mptr, uint16_t* map);

namespace {

constexpr double kMargin = 1e-6;  // relative rectangle growth / radius slack (conservative)

struct SubTestDev {
    double lo0, lo1, lo2, edge, margin, lim;  // sub-tile grid origin/edge, lim = r^2 (1 + 1e-6)
    int64_t ns0, ns1;
    int S, SD;
};

// Sub-tile box of (super T, local j) vs centre c: squared rectangle distance.
template <int DIM>
__device__ __forceinline__ bool sub_reaches(const SubTestDev& t, uint64_t T, int j, double cx, double cy,
                                            double cz) {
    const uint64_t sx = T % (uint64_t)t.ns0;
    const uint64_t rest = T / (uint64_t)t.ns0;
    const uint64_t sy = rest % (uint64_t)t.ns1;
    const uint64_t sz = rest / (uint64_t)t.ns1;
    const int jx = j % t.S, jy = (j / t.S) % t.S, jz = j / (t.S * t.S);
    const double idx[3] = {(double)(sx * t.S + jx), (double)(sy * t.S + jy), (double)(sz * t.S + jz)};
    const double lo[3] = {t.lo0, t.lo1, t.lo2};
    const double c[3] = {cx, cy, cz};
    double d2 = 0.0;
    for (int d = 0; d < DIM; ++d) {
        const double rlo = lo[d] + idx[d] * t.edge - t.margin;
        const double rhi = lo[d] + (idx[d] + 1.0) * t.edge + t.margin;
        const double gap = c[d] < rlo ? rlo - c[d] : (c[d] > rhi ? c[d] - rhi : 0.0);
        d2 += gap * gap;
    }
    return d2 < t.lim;
}

// One warp per (super-tile, sub-tile): count the super list's centres that
// reach the sub-tile.
template <int DIM>
__global__ void sub_count_kernel(const uint64_t* __restrict__ scptr, const uint32_t* __restrict__ scids,
                                 const double* __restrict__ centres, uint64_t n_super, SubTestDev t,
                                 uint16_t* __restrict__ sublen) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_super * t.SD;
         w += nw) {
        const uint64_t T = w / t.SD;
        const int j = (int)(w % t.SD);
        const uint64_t c0 = scptr[T], c1 = scptr[T + 1];
        uint32_t cnt = 0;
        for (uint64_t base = c0; base < c1; base += 32) {
            const uint64_t e = base + lane;
            bool hit = false;
            if (e < c1) {
                const uint32_t g = scids[e];
                hit = sub_reaches<DIM>(t, T, j, centres[(uint64_t)g * DIM], centres[(uint64_t)g * DIM + 1],
                                       DIM == 3 ? centres[(uint64_t)g * DIM + 2] : 0.0);
            }
            cnt += __popc(__ballot_sync(0xffffffffu, hit));
        }
        if (lane == 0) sublen[w] = (uint16_t)min(cnt, 0xffffu);
    }
}

// One CTA per bucketed super-tile: pack header, sub table, centres, row
// starts, ids and the sub-tile lists (super-local indices, ascending).
template <int DIM>
__global__ void build_blobs_kernel(const uint32_t* __restrict__ items, uint64_t n, BlobLayout B, int lsub_cap,
                                   int lsb, const uint64_t* __restrict__ scptr, const uint32_t* __restrict__ scids,
                                   const uint64_t* __restrict__ smptr, const double* __restrict__ centres,
                                   const uint64_t* __restrict__ uptr, SubTestDev t,
                                   unsigned char* __restrict__ blobs) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (uint64_t it = blockIdx.x; it < n; it += gridDim.x) {
        const uint32_t T = items[it];
        unsigned char* blob = blobs + it * B.bytes;
        const uint64_t c0 = scptr[T];
        const uint32_t L = (uint32_t)(scptr[T + 1] - c0);
        if (threadIdx.x == 0) {
            reinterpret_cast<uint32_t*>(blob)[0] = L;
            reinterpret_cast<uint32_t*>(blob)[1] = T;
            reinterpret_cast<uint64_t*>(blob)[1] = smptr[T];
            reinterpret_cast<uint32_t*>(blob)[4] = 0;
        }
        double* cx = reinterpret_cast<double*>(blob + B.cx);
        double* cy = reinterpret_cast<double*>(blob + B.cy);
        double* cz = reinterpret_cast<double*>(blob + B.cz);
        uint64_t* up = reinterpret_cast<uint64_t*>(blob + B.uptr);
        uint32_t* id = reinterpret_cast<uint32_t*>(blob + B.cid);
        for (int a = threadIdx.x; a < lsb; a += blockDim.x) {
            if (a < (int)L) {
                const uint32_t g = scids[c0 + a];
                cx[a] = centres[(uint64_t)g * DIM];
                cy[a] = centres[(uint64_t)g * DIM + 1];
                if (DIM == 3) cz[a] = centres[(uint64_t)g * DIM + 2];
                up[a] = uptr[g];
                id[a] = g;
            } else {
                cx[a] = 0.0;
                cy[a] = 0.0;
                if (DIM == 3) cz[a] = 0.0;
                up[a] = 0;
                id[a] = 0;
            }
        }
        uint32_t* sub = reinterpret_cast<uint32_t*>(blob + B.sub);
        uint16_t* lists = reinterpret_cast<uint16_t*>(blob + B.lists);
        for (int j = warp; j < t.SD; j += nwarp) {
            uint16_t* out = lists + j * lsub_cap;
            uint32_t cnt = 0;
            for (uint32_t a0 = 0; a0 < L; a0 += 32) {
                const uint32_t a = a0 + lane;
                bool hit = false;
                if (a < L) {
                    const uint32_t g = scids[c0 + a];
                    hit = sub_reaches<DIM>(t, T, j, centres[(uint64_t)g * DIM], centres[(uint64_t)g * DIM + 1],
                                           DIM == 3 ? centres[(uint64_t)g * DIM + 2] : 0.0);
                }
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
                if (hit && pos < (uint32_t)lsub_cap) out[pos] = (uint16_t)a;
                cnt += __popc(bal);
            }
            for (uint32_t p = cnt + lane; p < (uint32_t)lsub_cap; p += 32) out[p] = 0;
            if (lane == 0) sub[j] = (uint32_t)(j * lsub_cap) | (min(cnt, (uint32_t)lsub_cap) << 16);
        }
    }
}

// sub-tile list capacities (gather rows per warp, see rbg_assemble.cu)
constexpr int kSubCaps[] = {32, 48, 56, 64, 80, 120, 160, 200, 240};
// accumulator classes (shared-memory upper triangle of L_S x L_S)
constexpr int kSuperCaps[] = {32, 40, 48, 56, 64, 72, 80, 88, 96, 112, 128, 160, 192};

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

}  // namespace

// Sub-tile divisor q (sub edge = r/q) and super factor S from the point
// density (measured on B200, profiles/): 2-D sub-tiles of about 34 points
// (about nine 4-point DMMA k-steps per register pass), super-tiles of 2x2
// sub-tiles, 3x3 from q >= 7 and 4x4 from q >= 9 (larger super-tiles amortise
// the flush over more points until the accumulator costs occupancy); 3-D: sub-tiles of
// about 32 points (edge r/2 .. r/4) assembled in direct mode (one sub-tile per super-tile, register
// tiles reduced straight into the CSR values: a 3-D super-tile accumulator
// would not fit shared memory).
constexpr uint64_t kFineAfter = 2;  // assemblies on a centre set before its 3-D tiling is refined

static void choose_layout(const rbg_ctx* ctx, uint64_t n_points, const double* span, int& q, int& S, bool& fine) {
    const int dim = ctx->dim;
    const double r = ctx->radius;
    double vol = 1.0;
    for (int d = 0; d < dim; ++d) vol *= std::max(span[d], r * 1e-3);
    const double rho = std::max(1.0, (double)n_points) / vol;
    if (dim == 2) {
        const double e = std::sqrt(34.0 / rho);
        q = std::max(2, std::min(16, (int)std::lround(r / e)));
        S = q >= 9 ? 4 : q >= 7 ? 3 : 2;
    } else {  // about 32 points per cube (cfg3: r/3, 28 points: K3 5.4 ms; r/2 7.9 ms; r/4 10.6 ms) --
        // once the centre set is reused: the finer tiling's slot maps cost more to build than one
        // assembly gains (cfg3: layout 6.7 -> 10.5 ms for 2.4 ms of K3), so the first assembly of
        // a centre set runs on r/2 cubes and ensure_layout upgrades once it has been used
        // kFineAfter times (rent-or-buy: the regret of either choice stays within ~2x)
        const double e = std::cbrt(32.0 / rho);
        const int qf = std::max(2, std::min(4, (int)std::lround(r / e)));
        q = fine ? qf : 2;
        fine = q == qf;  // (nothing to upgrade to when the density asks for r/2 anyway)
        S = 1;
    }
    // small problems: shrink the super-tiles until there are at least two per
    // resident warp worker (cfg1: 625 super-tiles of 2x2 for 1184 warps ran
    // 0.075 ms, 2500 single sub-tiles 0.056 ms)
    {
        const double e = r / q;
        for (;;) {
            double ns = 1.0;
            for (int d = 0; d < dim; ++d) ns *= std::ceil(std::max(span[d], r * 1e-3) / (e * S));
            if (S == 1 || ns >= 2.0 * 148 * 8) break;
            --S;
        }
    }
    if (ctx->sub_div_req > 0) q = ctx->sub_div_req;
    if (ctx->super_req > 0) S = ctx->super_req;
    const int qe = env_int("RBG_SUB_DIV", 0), se = env_int("RBG_SUPER", 0);
    if (qe > 0) q = qe;
    if (se > 0) S = se;
    if (ctx->sub_div_req > 0 || ctx->super_req > 0 || qe > 0 || se > 0) fine = true;  // explicit choices are final
}

void build_layout(rbg_ctx* ctx, uint64_t n_points) {
    const auto t0 = std::chrono::steady_clock::now();
    const int dim = ctx->dim;
    const double r = ctx->radius;
    AsmLayout& L = ctx->lay;
    cudaStream_t st = ctx->stream;

    // grid origin: the query grid's (centres' bbox grown by r)
    double span[3] = {1, 1, 1};
    for (int d = 0; d < dim; ++d) span[d] = (double)ctx->grid.n[d] * ctx->grid.edge;
    int q = 4, S = 2;
    bool fine = dim == 2 || L.uses >= kFineAfter;
    choose_layout(ctx, n_points, span, q, S, fine);
    double e = r / q;
    int64_t nsup[3] = {1, 1, 1};
    uint64_t n_super = 1;
    for (;;) {
        n_super = 1;
        for (int d = 0; d < dim; ++d) {
            nsup[d] = std::max<int64_t>(1, (int64_t)std::ceil(span[d] / (e * S)));
            n_super *= (uint64_t)nsup[d];
        }
        if (n_super * (uint64_t)std::pow(S, dim) <= (1ull << 31)) break;
        e *= 1.25;
    }
    L.q = q;
    L.S = S;
    L.SD = dim == 2 ? S * S : S * S * S;
    L.sub_edge = e;
    for (int d = 0; d < 3; ++d) {
        L.lo[d] = d < dim ? ctx->grid.lo[d] : 0.0;
        L.nsup[d] = nsup[d];
    }
    L.n_super = n_super;
    L.n_keys = n_super * (uint64_t)L.SD;

    // ---- super-tile centre lists -------------------------------------------
    TileGrid sg;
    sg.dim = dim;
    for (int d = 0; d < 3; ++d) {
        sg.lo[d] = L.lo[d];
        sg.n[d] = nsup[d];
    }
    sg.edge = e * S;
    sg.inv_edge = 1.0 / sg.edge;
    sg.count = n_super;
    std::vector<uint64_t> hcptr;
    DevBuf<uint32_t> cnt;
    tile_lists(ctx, sg, cnt, L.scptr, L.scids, hcptr);
    const uint64_t total_ids = hcptr[n_super];

    // ---- slot maps ----------------------------------------------------------
    std::vector<uint64_t> mptr(n_super + 1, 0);
    uint32_t max_ls = 0;
    for (uint64_t T = 0; T < n_super; ++T) {
        const uint64_t l = hcptr[T + 1] - hcptr[T];
        max_ls = std::max<uint32_t>(max_ls, (uint32_t)l);
        mptr[T + 1] = mptr[T] + ((l * (l + 1) / 2 + 7) & ~7ull);  // 16-B aligned for the cp.async staging
    }
    L.max_ls = max_ls;
    L.mean_ls = n_super ? (double)total_ids / (double)n_super : 0.0;
    L.smptr.reserve(n_super + 1);
    RBG_CUDA(cudaMemcpyAsync(L.smptr.p, mptr.data(), (n_super + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    L.smap.reserve(std::max<uint64_t>(mptr[n_super], 1));
    slot_maps(ctx, L.scptr.p, n_super, L.scids.p, total_ids, L.smptr.p, L.smap.p);

    // ---- sub-tile list lengths -> buckets ------------------------------------
    SubTestDev t{L.lo[0], L.lo[1], L.lo[2], e, e * kMargin, r * r * (1.0 + 1e-6), nsup[0], nsup[1], S, L.SD};
    DevBuf<uint16_t> sublen;
    sublen.reserve(L.n_keys);
    {
        const unsigned blocks = blocks_for(L.n_keys * 32, 256);
        if (dim == 2)
            sub_count_kernel<2><<<blocks, 256, 0, st>>>(L.scptr.p, L.scids.p, ctx->centres.p, n_super, t, sublen.p);
        else
            sub_count_kernel<3><<<blocks, 256, 0, st>>>(L.scptr.p, L.scids.p, ctx->centres.p, n_super, t, sublen.p);
        RBG_CHECK_LAUNCH(ctx);
    }
    std::vector<uint16_t> hsub(L.n_keys);
    RBG_CUDA(cudaMemcpyAsync(hsub.data(), sublen.p, L.n_keys * sizeof(uint16_t), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));

    constexpr int nsc = (int)std::size(kSubCaps), nlc = (int)std::size(kSuperCaps);
    std::vector<std::vector<uint32_t>> lists(nsc * nlc);
    std::vector<uint32_t> fb;
    // work estimate per super-tile (register SYRK blocks summed over its
    // sub-tiles): the work counter hands out the heaviest super-tiles first so
    // the persistent warps finish together (longest-processing-time order)
    std::vector<uint32_t> weight(n_super, 0);
    uint32_t max_lsub = 0;
    double sum_lsub = 0.0;
    uint64_t n_sub_nonempty = 0;
    for (uint64_t T = 0; T < n_super; ++T) {
        const uint32_t ls = (uint32_t)(hcptr[T + 1] - hcptr[T]);
        if (ls == 0) continue;
        uint32_t ml = 0;
        for (int j = 0; j < L.SD; ++j) {
            const uint32_t v = hsub[T * L.SD + j];
            const uint32_t nb = (v + 7) / 8;
            weight[T] += nb * (nb + 1) / 2;
            ml = std::max(ml, v);
            if (v) {
                sum_lsub += v;
                ++n_sub_nonempty;
            }
        }
        max_lsub = std::max(max_lsub, ml);
        int si = 0, li = 0;
        while (si < nsc && (uint32_t)kSubCaps[si] < ml) ++si;
        while (li < nlc && (uint32_t)kSuperCaps[li] < ls) ++li;
        // register tile classes beyond the accumulator size are pointless
        if (si == nsc || li == nlc) {
            fb.push_back((uint32_t)T);
            continue;
        }
        lists[si * nlc + li].push_back((uint32_t)T);
    }
    L.max_lsub = max_lsub;
    L.mean_lsub = n_sub_nonempty ? sum_lsub / (double)n_sub_nonempty : 0.0;

    // One launch for everything when the largest class fits (the register and
    // accumulator sizes adapt per super-tile at run time; only capacity is
    // fixed by the class); else one launch per class.
    int optin = 0;
    RBG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    {
        int smax = -1, lmax = -1;
        for (int si = 0; si < nsc; ++si)
            for (int li = 0; li < nlc; ++li)
                if (!lists[si * nlc + li].empty()) {
                    smax = std::max(smax, si);
                    lmax = std::max(lmax, li);
                }
        if (smax >= 0 && (int)assembly_min_smem(dim, kSuperCaps[lmax], kSubCaps[smax], L.SD) <= optin) {
            std::vector<uint32_t> all;
            for (auto& v : lists) all.insert(all.end(), v.begin(), v.end());
            for (auto& v : lists) v.clear();
            lists[smax * nlc + lmax] = std::move(all);
        }
    }
    // longest-processing-time order: weight descending, ids ascending within a weight
    // (a counting sort -- the weights are small integers; 400k super-tiles at cfg5)
    {
        uint32_t wmax = 0;
        for (const uint32_t w : weight) wmax = std::max(wmax, w);
        std::vector<uint32_t> slot(n_super, 0xffffffffu), start((size_t)wmax + 2, 0), out;
        for (auto& v : lists) {
            if (v.size() < 2) continue;
            std::fill(start.begin(), start.end(), 0u);
            for (const uint32_t T : v) {
                slot[T] = wmax - weight[T];  // sort key: 0 = heaviest
                ++start[slot[T] + 1];
            }
            for (size_t k = 1; k < start.size(); ++k) start[k] += start[k - 1];
            out.resize(v.size());
            uint32_t lo = 0xffffffffu, hi = 0;
            for (const uint32_t T : v) {
                lo = std::min(lo, T);
                hi = std::max(hi, T);
            }
            for (uint32_t T = lo; T <= hi; ++T)  // ascending ids keep the ties ordered
                if (slot[T] != 0xffffffffu) {
                    out[start[slot[T]]++] = T;
                    slot[T] = 0xffffffffu;
                }
            v.swap(out);
        }
    }
    L.buckets.clear();
    for (int si = 0; si < nsc; ++si)
        for (int li = 0; li < nlc; ++li) {
            auto& v = lists[si * nlc + li];
            if (v.empty()) continue;
            if ((int)assembly_min_smem(dim, kSuperCaps[li], kSubCaps[si], L.SD) > optin) {
                fb.insert(fb.end(), v.begin(), v.end());
                continue;
            }
            L.buckets.emplace_back();
            Bucket& b = L.buckets.back();
            b.lsb = kSuperCaps[li];
            b.lsub_cap = kSubCaps[si];
            b.n_items = v.size();
            const BlobLayout B = blob_layout(dim, b.lsb, L.SD, b.lsub_cap);
            b.blob_bytes = B.bytes;
            b.items.reserve(b.n_items);
            RBG_CUDA(cudaMemcpyAsync(b.items.p, v.data(), b.n_items * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            b.blobs.reserve(b.n_items * B.bytes);
            const unsigned g = (unsigned)std::min<uint64_t>(b.n_items, 148u * 16u);
            if (dim == 2)
                build_blobs_kernel<2><<<g, 128, 0, st>>>(b.items.p, b.n_items, B, b.lsub_cap, b.lsb, L.scptr.p,
                                                         L.scids.p, L.smptr.p, ctx->centres.p, ctx->uptr.p, t,
                                                         b.blobs.p);
            else
                build_blobs_kernel<3><<<g, 128, 0, st>>>(b.items.p, b.n_items, B, b.lsub_cap, b.lsb, L.scptr.p,
                                                         L.scids.p, L.smptr.p, ctx->centres.p, ctx->uptr.p, t,
                                                         b.blobs.p);
            RBG_CHECK_LAUNCH(ctx);
            RBG_CUDA(cudaStreamSynchronize(st));  // v (host list) is released at scope end
        }
    L.n_fallback = fb.size();
    if (!fb.empty()) {
        L.fallback.reserve(fb.size());
        RBG_CUDA(cudaMemcpyAsync(L.fallback.p, fb.data(), fb.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    }
    ctx->work.reserve(L.buckets.size() + 1);
    ctx->tile_count.reserve(L.n_keys + 1);
    ctx->tile_pptr.reserve(L.n_keys + 1);
    RBG_CUDA(cudaStreamSynchronize(st));
    L.built = true;
    L.fine = fine;
    L.n_built = n_points;
    L.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// The sub-tile size follows the point density, so a layout built for a very
// different point count (a small first call, then the real one) is rebuilt;
// explicit rbg_set_tile_divisor / rbg_set_super_factor choices are kept.
void ensure_layout(rbg_ctx* ctx, uint64_t n_points) {
    const AsmLayout& L = ctx->lay;
    const bool pinned_choice = ctx->sub_div_req > 0 || ctx->super_req > 0;
    const bool upgrade = L.built && !pinned_choice && !L.fine && L.uses >= kFineAfter;  // 3-D, third assembly
    if (L.built && !upgrade && (pinned_choice || (n_points <= 4 * L.n_built && L.n_built <= 4 * n_points))) return;
    build_layout(ctx, n_points);
}

}  // namespace rbg
