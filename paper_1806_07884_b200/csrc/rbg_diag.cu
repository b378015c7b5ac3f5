// rbg_diag.cu -- measurement helpers for the bench (not on the hot path):
//  * support counts sum_p k_p and sum_p k_p^2 (the algorithmic work of an
//    assembly), with the hot path's exact inclusion rule;
//  * an fp64 FMA throughput microbenchmark (the fp64 roofline denominator,
//    which MEASURED_PEAKS.json does not carry).
#include <algorithm>
#include <cstring>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

template <int DIM>
__global__ void support_count_kernel(GridDev g, const uint64_t* __restrict__ cptr,
                                     const uint32_t* __restrict__ cids,
                                     const double* __restrict__ centres, int family, double alpha,
                                     double r2, const double* __restrict__ q, uint64_t nq,
                                     unsigned long long* out) {
    unsigned long long s1 = 0, s2 = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nq;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = q[i * DIM], y = q[i * DIM + 1], z = DIM == 3 ? q[i * DIM + 2] : 0.0;
        const uint64_t t = tile_of<DIM>(g, x, y, z);
        unsigned long long k = 0;
        if (t != ~0ull)
            for (uint64_t e = cptr[t]; e < cptr[t + 1]; ++e) {
                const uint32_t j = cids[e];
                const double d2 = dist2_of<DIM>(x, y, z, centres[(uint64_t)j * DIM],
                                                centres[(uint64_t)j * DIM + 1],
                                                DIM == 3 ? centres[(uint64_t)j * DIM + 2] : 0.0);
                if (d2 < r2 && phi_of_r(family, alpha, __dsqrt_rn(d2)) != 0.0) ++k;
            }
        s1 += k;
        s2 += k * k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], s1);
        atomicAdd(&out[1], s2);
    }
}

// K3's phi (phi_k3) against the reference's exact arithmetic (phi_of_r of
// the correctly rounded sqrt, strict d2 < r2) on n pseudo-random d2 per
// class: uniform in [0, 1.02 r2) (mantissa noise), within a few thousand ulp
// of the inclusion threshold, spread over every exponent down to the
// subnormals, and exact zero.  out[0] = inclusion mismatches + values that
// are not bitwise equal (wendland-3-0/3-1 only), out[1] = max relative error
// of phi, out[2] = max absolute error.
// FAST = the k-loop's variant (phi_k3<FAM, true>): out[0] counts inclusion mismatches only,
// out[1] is the max relative error over values >= 1e-6 (away from the support's edge, where
// one ulp of alpha r is a large relative change of a tiny phi), out[2] the max absolute error.
template <int FAM, bool FAST>
__global__ void phi_selftest_kernel(double alpha, double r2, long long ib, uint64_t n, uint64_t seed,
                                    unsigned long long* mism, double* rel, double* ab) {
    unsigned long long nbad = 0;
    double mrel = 0.0, mabs = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = (i + 1) * 0x9e3779b97f4a7c15ull ^ seed;
        k ^= k >> 31;
        k *= 0xbf58476d1ce4e5b9ull;
        k ^= k >> 29;
        double d2;
        switch (i & 3) {
            case 0: d2 = 1.02 * r2 * ((double)(k >> 11) * 0x1.0p-53); break;
            case 1: d2 = __longlong_as_double(ib + (long long)(k % 4096) - 2048); break;
            case 2: d2 = __longlong_as_double((long long)(k % 0x7fe0000000000000ull)); break;  // any exponent
            default: d2 = (i & 4) ? 0.0 : __longlong_as_double((long long)(k & 0xfffffffffffffull));  // subnormal
        }
        if (!(d2 >= 0.0)) continue;
        bool in;
        const double v = phi_k3<FAM, FAST>(d2, alpha, ib, in);
        const double r = __dsqrt_rn(d2);
        const double ex = d2 < r2 ? phi_of_r(FAM, alpha, r) : 0.0;
        if (in != (ex != 0.0)) ++nbad;
        if (!FAST && (FAM == 0 || FAM == 1) && __double_as_longlong(v) != __double_as_longlong(ex)) ++nbad;
        const double err = fabs(v - ex);
        mabs = fmax(mabs, err);
        if (FAST ? ex >= 1e-6 : ex != 0.0) mrel = fmax(mrel, err / ex);
    }
    if (nbad) atomicAdd(mism, nbad);
    // fp64 >= 0 compares like its bit pattern
    atomicMax(reinterpret_cast<unsigned long long*>(rel), (unsigned long long)__double_as_longlong(mrel));
    atomicMax(reinterpret_cast<unsigned long long*>(ab), (unsigned long long)__double_as_longlong(mabs));
}

constexpr int kChains = 8;
constexpr int kIters = 2048;

__global__ void fp64_fma_kernel(double seed, double* sink) {
    double a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
    const double b = 0.999999999, d = 1e-12;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = fma(a[c], b, d);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += a[c];
    if (s == 1234.5678) sink[0] = s;  // never true; keeps the chains live
}

}  // namespace
}  // namespace rbg

extern "C" rbg_status rbg_support_counts(rbg_ctx* ctx, const double* q, uint64_t nq,
                                         uint64_t* sum_k, uint64_t* sum_k2) {
    if (!ctx) return RBG_INVALID_ARGUMENT;
    try {
        if (!ctx->have_centres) throw rbg::Error(RBG_NOT_READY, "no reference points set");
        RBG_CUDA(cudaSetDevice(ctx->device));
        rbg::ensure_grid(ctx);
        cudaStream_t st = ctx->stream;
        ctx->ev_q.reserve(nq * ctx->dim + 1);
        // counters: allocated (8) by rbg_create
        RBG_CUDA(cudaMemcpyAsync(ctx->ev_q.p, q, nq * ctx->dim * sizeof(double), cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaMemsetAsync(ctx->counters.p + 2, 0, 2 * sizeof(unsigned long long), st));
        const rbg::GridDev g = rbg::grid_dev(ctx->grid);
        const unsigned blocks = rbg::blocks_for(nq, 256);
        if (ctx->dim == 2)
            rbg::support_count_kernel<2><<<blocks, 256, 0, st>>>(g, ctx->tile_cptr.p, ctx->tile_cids.p,
                                                                 ctx->centres.p, ctx->family, ctx->alpha,
                                                                 ctx->r2, ctx->ev_q.p, nq, ctx->counters.p + 2);
        else
            rbg::support_count_kernel<3><<<blocks, 256, 0, st>>>(g, ctx->tile_cptr.p, ctx->tile_cids.p,
                                                                 ctx->centres.p, ctx->family, ctx->alpha,
                                                                 ctx->r2, ctx->ev_q.p, nq, ctx->counters.p + 2);
        RBG_CHECK_LAUNCH(ctx);
        unsigned long long h[2];
        RBG_CUDA(cudaMemcpyAsync(h, ctx->counters.p + 2, sizeof(h), cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        *sum_k = h[0];
        *sum_k2 = h[1];
        return RBG_OK;
    } catch (const rbg::Error& e) {
        ctx->err = e.what();
        return e.code;
    }
}

extern "C" rbg_status rbg_fp64_peak(rbg_ctx* ctx, double* tflops) {
    if (!ctx || !tflops) return RBG_INVALID_ARGUMENT;
    try {
        RBG_CUDA(cudaSetDevice(ctx->device));
        int sms = 0;
        RBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        cudaStream_t st = ctx->stream;
        // counters: allocated (8) by rbg_create
        const unsigned blocks = (unsigned)sms * 8u, threads = 256;
        double best = 0.0;
        for (int rep = 0; rep < 4; ++rep) {
            RBG_CUDA(cudaEventRecord(ctx->ev0, st));
            rbg::fp64_fma_kernel<<<blocks, threads, 0, st>>>(1.0 + rep, reinterpret_cast<double*>(ctx->counters.p));
            RBG_CUDA(cudaEventRecord(ctx->ev1, st));
            RBG_CUDA(cudaEventSynchronize(ctx->ev1));
            float ms = 0.f;
            RBG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            const double flops = 2.0 * rbg::kChains * rbg::kIters * (double)blocks * threads;
            if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
        }
        *tflops = best;
        return RBG_OK;
    } catch (const rbg::Error& e) {
        ctx->err = e.what();
        return e.code;
    }
}

extern "C" rbg_status rbg_assembly_times(rbg_ctx* ctx, double* bin_ms, double* tiles_ms) {
    if (!ctx) return RBG_INVALID_ARGUMENT;
    try {
        RBG_CUDA(cudaSetDevice(ctx->device));
        RBG_CUDA(cudaEventSynchronize(ctx->ev_asm[2]));
        float a = 0.f, b = 0.f;
        RBG_CUDA(cudaEventElapsedTime(&a, ctx->ev_asm[0], ctx->ev_asm[1]));
        RBG_CUDA(cudaEventElapsedTime(&b, ctx->ev_asm[1], ctx->ev_asm[2]));
        if (bin_ms) *bin_ms = a;
        if (tiles_ms) *tiles_ms = b;
        return RBG_OK;
    } catch (const rbg::Error& e) {
        ctx->err = e.what();
        return e.code;
    }
}

namespace {
rbg_status phi_selftest(rbg_ctx* ctx, bool fast, int family, double alpha, uint64_t n, uint64_t seed,
                        uint64_t* mismatches, double* max_rel, double* max_abs) {
    if (!ctx || !mismatches || family < 0 || family > 3 || !(alpha > 0.0)) return RBG_INVALID_ARGUMENT;
    try {
        RBG_CUDA(cudaSetDevice(ctx->device));
        ctx->counters.reserve(8);
        cudaStream_t st = ctx->stream;
        RBG_CUDA(cudaMemsetAsync(ctx->counters.p + 3, 0, 3 * sizeof(unsigned long long), st));
        const double r2 = (1.0 / alpha) * (1.0 / alpha);
        const long long ib = rbg::inclusion_bits(alpha, r2);
        unsigned long long* c = ctx->counters.p + 3;
        double* rel = reinterpret_cast<double*>(c + 1);
        double* ab = reinterpret_cast<double*>(c + 2);
#define RBG_SELFTEST(F)                                                                                  \
    if (fast) rbg::phi_selftest_kernel<F, true><<<148 * 8, 256, 0, st>>>(alpha, r2, ib, n, seed, c, rel, ab); \
    else rbg::phi_selftest_kernel<F, false><<<148 * 8, 256, 0, st>>>(alpha, r2, ib, n, seed, c, rel, ab)
        switch (family) {
            case 0: RBG_SELFTEST(0); break;
            case 1: RBG_SELFTEST(1); break;
            case 2: RBG_SELFTEST(2); break;
            default: RBG_SELFTEST(3);
        }
#undef RBG_SELFTEST
        RBG_CHECK_LAUNCH(ctx);
        unsigned long long h[3];
        RBG_CUDA(cudaMemcpyAsync(h, c, sizeof(h), cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        *mismatches = h[0];
        if (max_rel) std::memcpy(max_rel, &h[1], sizeof(double));
        if (max_abs) std::memcpy(max_abs, &h[2], sizeof(double));
        return RBG_OK;
    } catch (const rbg::Error& e) {
        ctx->err = e.what();
        return e.code;
    }
}
}  // namespace

extern "C" rbg_status rbg_phi_selftest(rbg_ctx* ctx, int family, double alpha, uint64_t n, uint64_t seed,
                                       uint64_t* mismatches, double* max_rel, double* max_abs) {
    return phi_selftest(ctx, false, family, alpha, n, seed, mismatches, max_rel, max_abs);
}

extern "C" rbg_status rbg_phi_selftest_fast(rbg_ctx* ctx, int family, double alpha, uint64_t n, uint64_t seed,
                                            uint64_t* mismatches, double* max_rel, double* max_abs) {
    return phi_selftest(ctx, true, family, alpha, n, seed, mismatches, max_rel, max_abs);
}

extern "C" rbg_status rbg_set_tile_divisor(rbg_ctx* ctx, double divisor) {
    if (!ctx || !(divisor == 0.0 || (divisor >= 1.0 && divisor <= 16.0))) return RBG_INVALID_ARGUMENT;
    ctx->sub_div_req = (int)(divisor + 0.5);
    ctx->lay.built = false;
    return RBG_OK;
}

extern "C" rbg_status rbg_set_super_factor(rbg_ctx* ctx, int S) {
    if (!ctx || S < 0 || S > 8) return RBG_INVALID_ARGUMENT;
    ctx->super_req = S;
    ctx->lay.built = false;
    return RBG_OK;
}

extern "C" rbg_status rbg_get_layout_info(rbg_ctx* ctx, rbg_layout_info* info) {
    if (!ctx || !info) return RBG_INVALID_ARGUMENT;
    const rbg::AsmLayout& L = ctx->lay;
    info->built = L.built ? 1 : 0;
    info->sub_div = L.q;
    info->super_factor = L.S;
    info->n_buckets = (int)L.buckets.size();
    info->n_super = L.n_super;
    info->n_fallback = L.n_fallback;
    info->max_super_centres = L.max_ls;
    info->max_sub_centres = L.max_lsub;
    info->mean_super_centres = L.mean_ls;
    info->mean_sub_centres = L.mean_lsub;
    info->sub_edge = L.sub_edge;
    info->build_ms = L.build_ms;
    return RBG_OK;
}
