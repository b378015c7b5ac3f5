// rbg_eval.cu -- K5 batched evaluation and K6 error reductions.
//
// evaluate_shifted (model.cpp:50-72): per query, the reference walks a kd-tree
// over the centres, sorts the hits by centre index and accumulates
// f += w_j * phi(d_j) in that order.  Here each query reads its tile's centre
// list, which is already ascending, and accumulates with unfused
// __dmul_rn/__dadd_rn -- bitwise equal to the reference for the same w.
// error_report (model.cpp:196-232) statistics are fixed-order two-level
// reductions (run-to-run deterministic); RMS and max |e| are additions.
#include <cmath>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

constexpr int kThreads = 256;
#ifndef RBG_EVAL_BATCH
#define RBG_EVAL_BATCH 8
#endif
constexpr int kEvalBatch = RBG_EVAL_BATCH;  // candidates whose loads are in flight together in eval_kernel

// Linear-polynomial term of a bordered model (model.cpp:65-68): after the
// support sum, f += a0 x + a1 y (+ a2 z) + a_last, evaluated left to right
// with unfused mul/add like the reference's expression.
struct PolyDev {
    int on;
    double a[4];
};

template <int DIM>
__global__ void eval_kernel(GridDev g, const uint64_t* __restrict__ cptr,
                            const uint32_t* __restrict__ cids, const double* __restrict__ centres,
                            const double* __restrict__ w, int family, double alpha, double r2,
                            PolyDev poly, const double* __restrict__ q, uint64_t nq,
                            double* __restrict__ f) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nq;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = q[i * DIM], y = q[i * DIM + 1], z = DIM == 3 ? q[i * DIM + 2] : 0.0;
        const uint64_t t = tile_of<DIM>(g, x, y, z);
        double acc = 0.0;
        if (t != ~0ull) {
            // kEvalBatch candidates at a time: their index, coordinate and weight loads are all in
            // flight before the first use (the walk is latency-bound: every query of a warp
            // reads another tile's list); the sum still runs in ascending list order
            const uint64_t e1 = cptr[t + 1];
            uint64_t e = cptr[t];
            for (; e + kEvalBatch <= e1; e += kEvalBatch) {
                uint32_t j[kEvalBatch];
                double cx[kEvalBatch], cy[kEvalBatch], cz[kEvalBatch], wj[kEvalBatch];
#pragma unroll
                for (int u = 0; u < kEvalBatch; ++u) j[u] = cids[e + u];
#pragma unroll
                for (int u = 0; u < kEvalBatch; ++u) {
                    cx[u] = centres[(uint64_t)j[u] * DIM];
                    cy[u] = centres[(uint64_t)j[u] * DIM + 1];
                    cz[u] = DIM == 3 ? centres[(uint64_t)j[u] * DIM + 2] : 0.0;
                    wj[u] = w[j[u]];
                }
#pragma unroll
                for (int u = 0; u < kEvalBatch; ++u) {
                    const double d2 = dist2_of<DIM>(x, y, z, cx[u], cy[u], cz[u]);
                    if (d2 < r2) {
                        const double v = phi_of_r(family, alpha, __dsqrt_rn(d2));
                        if (v != 0.0) acc = __dadd_rn(acc, __dmul_rn(wj[u], v));
                    }
                }
            }
            for (; e < e1; ++e) {
                const uint32_t j = cids[e];
                const double d2 = dist2_of<DIM>(x, y, z, centres[(uint64_t)j * DIM],
                                                centres[(uint64_t)j * DIM + 1],
                                                DIM == 3 ? centres[(uint64_t)j * DIM + 2] : 0.0);
                if (d2 < r2) {
                    const double v = phi_of_r(family, alpha, __dsqrt_rn(d2));
                    if (v != 0.0) acc = __dadd_rn(acc, __dmul_rn(w[j], v));
                }
            }
        }
        if (poly.on) {
            double t = __dadd_rn(__dmul_rn(poly.a[0], x), __dmul_rn(poly.a[1], y));
            if (DIM == 3) t = __dadd_rn(t, __dmul_rn(poly.a[2], z));
            t = __dadd_rn(t, poly.a[DIM]);
            acc = __dadd_rn(acc, t);
        }
        f[i] = acc;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-level reduction of NV sums (+ optionally one max in slot NV-1).
template <int NV, bool LAST_IS_MAX>
__device__ void block_reduce_store(double (&v)[NV], double* out) {
    __shared__ double sh[NV][kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double s = (LAST_IS_MAX && k == NV - 1) ? warp_max(v[k]) : warp_sum(v[k]);
        if (lane == 0) sh[k][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = sh[k][0];
            for (int w = 1; w < kThreads / 32; ++w)
                s = (LAST_IS_MAX && k == NV - 1) ? fmax(s, sh[k][w]) : s + sh[k][w];
            out[k] = s;
        }
    }
}

// pass 1 partials per block: sum|e|, sum|h|, sum e^2, max|e|
__global__ void err_pass1(const double* __restrict__ f, const double* __restrict__ h, uint64_t n,
                          double* __restrict__ part, double* __restrict__ signed_err) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double e = f[i] - h[i];
        if (signed_err) signed_err[i] = e;
        v[0] += fabs(e);
        v[1] += fabs(h[i]);
        v[2] += e * e;
        v[3] = fmax(v[3], fabs(e));
    }
    block_reduce_store<4, true>(v, part + 4 * blockIdx.x);
}

__global__ void err_pass2(const double* __restrict__ f, const double* __restrict__ h, uint64_t n,
                          const double* __restrict__ mae_ptr, double* __restrict__ part) {
    const double mae = *mae_ptr;
    double v[1] = {0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double d = fabs(f[i] - h[i]) - mae;
        v[0] += d * d;
    }
    block_reduce_store<1, false>(v, part + blockIdx.x);
}

// single block: fold nb partial rows of width W (last column max if MAXLAST);
// out[k] = total; for pass 1 also out[4] = mae = out[0] / n.
template <int W, bool MAXLAST>
__global__ void err_finish(const double* __restrict__ part, unsigned nb, double n, double* out) {
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = 0.0;
    for (unsigned b = threadIdx.x; b < nb; b += kThreads)
#pragma unroll
        for (int k = 0; k < W; ++k)
            v[k] = (MAXLAST && k == W - 1) ? fmax(v[k], part[(uint64_t)b * W + k]) : v[k] + part[(uint64_t)b * W + k];
    block_reduce_store<W, MAXLAST>(v, out);
    __syncthreads();
    if (threadIdx.x == 0 && W == 4) out[4] = out[0] / n;
}

}  // namespace

void evaluate_points(rbg_ctx* ctx, const double* d_c, const double* d_q, uint64_t nq, double* d_f) {
    if (nq == 0) return;
    const GridDev g = grid_dev(ctx->grid);
    const unsigned blocks = blocks_for(nq, kThreads);
    PolyDev poly{ctx->model_poly, {ctx->model_a[0], ctx->model_a[1], ctx->model_a[2], ctx->model_a[3]}};
    if (ctx->dim == 2)
        eval_kernel<2><<<blocks, kThreads, 0, ctx->stream>>>(g, ctx->tile_cptr.p, ctx->tile_cids.p,
                                                            ctx->centres.p, d_c, ctx->family,
                                                            ctx->alpha, ctx->r2, poly, d_q, nq, d_f);
    else
        eval_kernel<3><<<blocks, kThreads, 0, ctx->stream>>>(g, ctx->tile_cptr.p, ctx->tile_cids.p,
                                                            ctx->centres.p, d_c, ctx->family,
                                                            ctx->alpha, ctx->r2, poly, d_q, nq, d_f);
    RBG_CHECK_LAUNCH(ctx);
}

// d_f doubles as the signed-error output (overwritten with f - h) when the
// caller wants it; stats are written to `out`.
void error_stats(rbg_ctx* ctx, const double* d_f, const double* d_h, uint64_t n,
                 rbg_error_stats* out) {
    cudaStream_t st = ctx->stream;
    const unsigned nb = blocks_for(n, kThreads, 148u * 8u);
    ctx->ev_part.reserve(4ull * nb + 8);
    double* part = ctx->ev_part.p;
    double* fin = part + 4ull * nb;  // 8 slots: [0..3] pass-1 totals, [4] mae, [5] var sum
    err_pass1<<<nb, kThreads, 0, st>>>(d_f, d_h, n, part, nullptr);
    RBG_CHECK_LAUNCH(ctx);
    err_finish<4, true><<<1, kThreads, 0, st>>>(part, nb, (double)n, fin);
    RBG_CHECK_LAUNCH(ctx);
    err_pass2<<<nb, kThreads, 0, st>>>(d_f, d_h, n, fin + 4, part);
    RBG_CHECK_LAUNCH(ctx);
    err_finish<1, false><<<1, kThreads, 0, st>>>(part, nb, (double)n, fin + 5);
    RBG_CHECK_LAUNCH(ctx);
    double h[6];
    RBG_CUDA(cudaMemcpyAsync(h, fin, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    const double dn = (double)n;
    out->mean_absolute_error = h[4];
    out->deviation_of_error = h[5] / dn;
    const double normalizer = h[1] / dn;
    out->mean_relative_error_pct = normalizer > 0.0 ? 100.0 * h[4] / normalizer : 0.0;
    out->rms_error = std::sqrt(h[2] / dn);
    out->max_abs_error = h[3];
}

}  // namespace rbg
