// rbg_band.cu -- the reference's own solve, LLT with the ridge ladder
// (solve_weights, solver.cpp:289-330), as a banded Cholesky on the device.
//
// The normal matrix of compactly supported RBFs is sparse with a local
// pattern: ordering the centres along x gives a band of half-width b ~ M 2r
// (2-D).  Where M b^2 is affordable (configs 1, 2, 4; small fits) the system
// is factored exactly like the reference factors its dense matrix -- a
// Cholesky, first non-positive pivot = failure, next ridge rung -- just on
// the band (no fill-in leaves it) and in that ordering.  Larger bands
// (config 5, 3-D) keep the preconditioned CG of rbg_solve.cu.
//
// Storage: the lower band in 32 x 32 tiles, tile column C holding tiles
// (C + d, C) for d < nbb, each column-major.  Per tile column J (right-looking):
//   band_panel   -- one warp per tile of the column: the diagonal tile is
//                   factored in registers (lane = row, shuffles), the warp of
//                   tile d >= 1 then solves L(J+d, J) = A(J+d, J) L_JJ^-T;
//   band_update  -- one warp per trailing tile: A(J+d2, J+d1) -= L(J+d2, J)
//                   L(J+d1, J)^T on the fp64 tensor cores (DMMA m8n8k4).
// Forward / backward substitution: one CTA each, walking the tile rows (warp 0
// solves the 32 x 32 diagonal block, the 32 warps apply the tiles below/above).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include <cub/cub.cuh>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

constexpr int TB = 32;               // tile edge
constexpr int TE = TB * TB;          // doubles per tile
constexpr double kMaxBandFlops = 1.5e12;  // M b^2 above this: PCG

__device__ __forceinline__ uint64_t ord_key64(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Sort keys: x (2-D: x then y folded into the low bits is unnecessary -- ties
// only reorder centres with equal x, which keeps the band).
__global__ void band_keys_kernel(const double* __restrict__ c, uint64_t m, int dim, uint64_t* __restrict__ keys,
                                 uint32_t* __restrict__ ids) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        keys[i] = ord_key64(c[i * dim]);
        ids[i] = (uint32_t)i;
    }
}

__global__ void band_pos_kernel(const uint32_t* __restrict__ perm, uint64_t m, uint32_t* __restrict__ pos) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
        pos[perm[k]] = (uint32_t)k;
}

// Half-bandwidth max |pos(i) - pos(j)| over the upper pattern.
__global__ void band_width_kernel(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ ucols, uint64_t m,
                                  const uint32_t* __restrict__ pos, unsigned long long* __restrict__ out) {
    unsigned long long w = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t pi = pos[i];
        for (uint64_t e = uptr[i]; e < uptr[i + 1]; ++e) {
            const int64_t d = pi - (int64_t)pos[ucols[e]];
            w = max(w, (unsigned long long)(d < 0 ? -d : d));
        }
    }
    for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, w);
}

__device__ __forceinline__ double* tile_at(double* band, uint64_t nbb, uint64_t R, uint64_t C) {
    return band + ((C * nbb) + (R - C)) * (uint64_t)TE;
}

// Scatter the upper CSR values (+ shift on the diagonal) into the permuted
// lower band; rows past m get an identity diagonal (decoupled padding).
__global__ void band_fill_kernel(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ ucols,
                                 const double* __restrict__ vals, uint64_t m, const uint32_t* __restrict__ pos,
                                 double shift, uint64_t nbb, uint64_t NT, double* __restrict__ band) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint64_t i = warp; i < NT * TB; i += nw) {
        if (i >= m) {
            if (lane == 0) tile_at(band, nbb, i / TB, i / TB)[(i % TB) * TB + i % TB] = 1.0;
            continue;
        }
        const uint64_t pi = pos[i];
        for (uint64_t e = uptr[i] + lane; e < uptr[i + 1]; e += 32) {
            const uint64_t pj = pos[ucols[e]];
            const uint64_t r = pi > pj ? pi : pj, c = pi > pj ? pj : pi;
            double v = vals[e];
            if (r == c) v += shift;
            tile_at(band, nbb, r / TB, c / TB)[(c % TB) * TB + (r % TB)] = v;
        }
    }
}

__global__ void band_trace_kernel(const uint64_t* __restrict__ uptr, const double* __restrict__ vals, uint64_t m,
                                  double* __restrict__ out) {
    double s = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        s += vals[uptr[i]];  // the diagonal leads every upper row
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// Cholesky of the 32 x 32 tile in registers: lane i holds row i (a[j], j <= i
// meaningful).  Returns false (warp-uniform) at the first non-positive pivot,
// whose tile-local index goes to *bad.
__device__ __forceinline__ bool chol32(double (&a)[TB], int lane, int* bad) {
#pragma unroll
    for (int k = 0; k < TB; ++k) {
        const double akk = __shfl_sync(0xffffffffu, a[k], k);
        if (!(akk > 0.0) || !isfinite(akk)) {
            *bad = k;
            return false;
        }
        const double lkk = sqrt(akk);
        a[k] = lane == k ? lkk : (lane > k ? a[k] / lkk : a[k]);
#pragma unroll
        for (int j = k + 1; j < TB; ++j) {
            const double ljk = __shfl_sync(0xffffffffu, a[k], j);
            if (lane >= j) a[j] = fma(-a[k], ljk, a[j]);
        }
    }
    return true;
}

// One warp per tile (J + d, J), d = blockIdx.x.  status[0] = permuted index of
// the first failing pivot (all-ones: none).
__global__ void __launch_bounds__(32) band_panel_kernel(double* __restrict__ band, uint64_t J, uint64_t nbb,
                                                        double* __restrict__ diagL,
                                                        unsigned long long* __restrict__ status) {
    if (status[0] != ~0ull) return;
    const int lane = threadIdx.x;
    const uint64_t d = blockIdx.x;
    double* dt = tile_at(band, nbb, J, J);
    double a[TB];
#pragma unroll
    for (int j = 0; j < TB; ++j) a[j] = dt[j * TB + lane];
    int bad = 0;
    if (!chol32(a, lane, &bad)) {
        if (d == 0 && lane == 0) atomicMin(status, (unsigned long long)(J * TB + bad));
        return;
    }
    if (d == 0) {  // L_JJ goes to its own array: the other warps of this launch still read A_JJ
        double* lt = diagL + J * (uint64_t)TE;
#pragma unroll
        for (int j = 0; j < TB; ++j) lt[j * TB + lane] = j <= lane ? a[j] : 0.0;
        return;
    }
    // x L^T = row (lane) of A(J+d, J): forward substitution over the columns
    double* ot = tile_at(band, nbb, J + d, J);
    double x[TB];
#pragma unroll
    for (int j = 0; j < TB; ++j) x[j] = ot[j * TB + lane];
    // column-oriented: x_k /= L_kk, then x_j -= x_k L_jk for every j > k (independent updates)
#pragma unroll
    for (int k = 0; k < TB; ++k) {
        x[k] = x[k] / __shfl_sync(0xffffffffu, a[k], k);
#pragma unroll
        for (int j = k + 1; j < TB; ++j) x[j] = fma(-x[k], __shfl_sync(0xffffffffu, a[k], j), x[j]);
    }
#pragma unroll
    for (int j = 0; j < TB; ++j) ot[j * TB + lane] = x[j];
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

// Trailing update of tile column J: one warp per tile (J + d2, J + d1),
// 1 <= d1 <= d2 < nbb, J + d2 < NT; A -= L(J+d2, J) L(J+d1, J)^T.
__global__ void __launch_bounds__(128) band_update_kernel(double* __restrict__ band, uint64_t J, uint64_t nbb,
                                                          uint64_t NT, uint64_t ntiles,
                                                          const unsigned long long* __restrict__ status) {
    if (status[0] != ~0ull) return;
    const uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (t >= ntiles) return;
    const int lane = threadIdx.x & 31;
    // t -> (d1, d2): column-wise enumeration of the upper triangle of [1, dmax]^2
    const uint64_t dmax = min(nbb - 1, NT - 1 - J);
    uint64_t d1 = 1, rem = t;
    while (rem >= dmax - d1 + 1) {
        rem -= dmax - d1 + 1;
        ++d1;
    }
    const uint64_t d2 = d1 + rem;
    const double* A = tile_at(band, nbb, J + d2, J);  // rows i of the target
    const double* B = tile_at(band, nbb, J + d1, J);  // rows n of the target's columns
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int n = 0; n < 4; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
    const int r = lane >> 2, q = lane & 3;
#pragma unroll 2
    for (int s = 0; s < TB / 4; ++s) {
        const int col = (4 * s + q) * TB;
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            fa[i] = A[col + 8 * i + r];
            fb[i] = B[col + 8 * i + r];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int n = 0; n < 4; ++n) dmma884(acc[i][n], fa[i], fb[n]);
    }
    double* C = tile_at(band, nbb, J + d2, J + d1);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = 8 * i + r, cc = 8 * n + 2 * q + e;
                C[cc * TB + row] -= acc[i][n][e];
            }
}

// Forward substitution L y = b in one CTA (32 warps) over all tile rows: per
// tile row J, warp 0 solves the 32 x 32 diagonal block (lane = row), then the
// warps apply b_{J+d} -= L(J+d, J) y_J for the tiles below (d = warp + 32 i).
constexpr int kSolveWarps = 32;
__global__ void __launch_bounds__(kSolveWarps * 32) band_forward_kernel(const double* __restrict__ band,
                                                                        const double* __restrict__ diagL,
                                                                        uint64_t NT, uint64_t nbb,
                                                                        double* __restrict__ b, double* __restrict__ y) {
    __shared__ double yJ[TB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t J = 0; J < NT; ++J) {
        if (warp == 0) {
            const double* dt = diagL + J * (uint64_t)TE;
            double v = b[J * TB + lane];
#pragma unroll 4
            for (int k = 0; k < TB; ++k) {
                const double lk = dt[k * TB + lane];  // L(lane, k)
                const double yk = __shfl_sync(0xffffffffu, v, k) / dt[k * TB + k];
                if (lane == k) v = yk;
                if (lane > k) v = fma(-lk, yk, v);
            }
            yJ[lane] = v;
            y[J * TB + lane] = v;
        }
        __syncthreads();
        const uint64_t dmax = min(nbb - 1, NT - 1 - J);
        for (uint64_t d = 1 + warp; d <= dmax; d += kSolveWarps) {
            const double* ot = band + (J * nbb + d) * (uint64_t)TE;  // L(J+d, J)
            double s = 0.0;
#pragma unroll 8
            for (int k = 0; k < TB; ++k) s = fma(ot[k * TB + lane], yJ[k], s);
            b[(J + d) * TB + lane] -= s;
        }
        __syncthreads();
    }
}

// Backward substitution L^T x = y in one CTA, tile rows descending: warp 0
// solves L_JJ^T x_J = y_J, the warps apply y_{J-d} -= L(J, J-d)^T x_J.
__global__ void __launch_bounds__(kSolveWarps * 32) band_backward_kernel(const double* __restrict__ band,
                                                                         const double* __restrict__ diagL,
                                                                         uint64_t NT, uint64_t nbb,
                                                                         double* __restrict__ y, double* __restrict__ x) {
    __shared__ double xJ[TB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t J = NT; J-- > 0;) {
        if (warp == 0) {
            const double* dt = diagL + J * (uint64_t)TE;
            double v = y[J * TB + lane];
#pragma unroll 4
            for (int k = TB - 1; k >= 0; --k) {
                const double xk = __shfl_sync(0xffffffffu, v, k) / dt[k * TB + k];
                if (lane == k) v = xk;
                if (lane < k) v = fma(-dt[lane * TB + k], xk, v);  // L(k, lane)
            }
            xJ[lane] = v;
            x[J * TB + lane] = v;
        }
        __syncthreads();
        const uint64_t dmax = min(nbb - 1, J);
        for (uint64_t d = 1 + warp; d <= dmax; d += kSolveWarps) {
            const double* ot = band + ((J - d) * nbb + d) * (uint64_t)TE;  // L(J, J-d): rows of J, columns of J-d
            double s = 0.0;
#pragma unroll 8
            for (int k = 0; k < TB; ++k) s = fma(ot[lane * TB + k], xJ[k], s);
            y[(J - d) * TB + lane] -= s;
        }
        __syncthreads();
    }
}

template <bool TO_BAND>
__global__ void band_permute_kernel(const uint32_t* __restrict__ perm, uint64_t m, uint64_t padded,
                                    const double* __restrict__ in, double* __restrict__ out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < padded;
         k += (uint64_t)gridDim.x * blockDim.x) {
        if (TO_BAND) out[k] = k < m ? in[perm[k]] : 0.0;
        else if (k < m) out[perm[k]] = in[k];
    }
}

// ||rhs - B c||^2 and ||rhs||^2 over the upper CSR (symmetric product via the full pattern).
__global__ void band_residual_kernel(const uint64_t* __restrict__ fptr, const uint32_t* __restrict__ fcols,
                                     const uint64_t* __restrict__ f2u, const double* __restrict__ vals,
                                     const double* __restrict__ rhs, const double* __restrict__ c, uint64_t m,
                                     double* __restrict__ out) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    double rr = 0.0, bb = 0.0;
    for (uint64_t i = warp; i < m; i += nw) {
        double s = 0.0;
        for (uint64_t e = fptr[i] + lane; e < fptr[i + 1]; e += 32) s = fma(vals[f2u[e]], c[fcols[e]], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double r = rhs[i] - s;
        rr = fma(r, r, rr);
        bb = fma(rhs[i], rhs[i], bb);
    }
    if (lane == 0) {
        atomicAdd(&out[0], rr);
        atomicAdd(&out[1], bb);
    }
}

}  // namespace

// Ordering, bandwidth and the go/no-go of the banded path (once per centre set).
bool band_plan(rbg_ctx* ctx) {
    BandPlan& P = ctx->band;
    if (P.planned) return P.use;
    P.planned = true;
    P.use = false;
    const uint64_t m = ctx->m;
    cudaStream_t st = ctx->stream;
    DevBuf<uint64_t> keys, keys_out;
    DevBuf<uint32_t> ids;
    keys.reserve(m);
    keys_out.reserve(m);
    ids.reserve(m);
    P.perm.reserve(m);
    P.pos.reserve(m);
    band_keys_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->centres.p, m, ctx->dim, keys.p, ids.p);
    RBG_CHECK_LAUNCH(ctx);
    size_t tmp_bytes = 0;
    RBG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_out.p, ids.p, P.perm.p, (int)m, 0, 64,
                                             st));
    DevBuf<unsigned char> tmp;
    tmp.reserve(tmp_bytes);
    RBG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys_out.p, ids.p, P.perm.p, (int)m, 0, 64, st));
    band_pos_kernel<<<blocks_for(m, 256), 256, 0, st>>>(P.perm.p, m, P.pos.p);
    RBG_CHECK_LAUNCH(ctx);
    DevBuf<unsigned long long> w;
    w.reserve(1);
    RBG_CUDA(cudaMemsetAsync(w.p, 0, sizeof(unsigned long long), st));
    band_width_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->uptr.p, ctx->ucols.p, m, P.pos.p, w.p);
    RBG_CHECK_LAUNCH(ctx);
    unsigned long long hw = 0;
    RBG_CUDA(cudaMemcpyAsync(&hw, w.p, sizeof(hw), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    P.b = hw;
    P.NT = (m + TB - 1) / TB;
    P.nbb = std::min<uint64_t>(P.NT, (hw + TB - 1) / TB + 1);
    const double flops = (double)m * (double)(P.nbb * TB) * (double)(P.nbb * TB);
    const double bytes = (double)P.NT * (double)P.nbb * TE * sizeof(double);
    size_t free_b = 0, total_b = 0;
    RBG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    P.use = flops <= kMaxBandFlops && bytes <= 0.25 * (double)free_b;
    return P.use;
}

// LLT of the band with the reference's ridge ladder; c_out (host) in centre order.
void band_solve(rbg_ctx* ctx, double* c_out, rbg_solve_diag* diag) {
    BandPlan& P = ctx->band;
    cudaStream_t st = ctx->stream;
    const uint64_t m = ctx->m, NT = P.NT, nbb = P.nbb, padded = NT * TB;
    const double* uvals = ctx->sys.p;
    const double* rhs = ctx->sys.p + ctx->nnz_upper;
    P.tiles.reserve(NT * nbb * TE);
    P.diag.reserve(NT * TE);
    for (auto* v : {&ctx->x, &ctx->r, &ctx->z, &ctx->q}) v->reserve(padded);
    ctx->scal.reserve(4);
    DevBuf<unsigned long long> status;
    status.reserve(1);
    RBG_CUDA(cudaEventRecord(ctx->ev0, st));
    RBG_CUDA(cudaMemsetAsync(ctx->scal.p, 0, 4 * sizeof(double), st));
    band_trace_kernel<<<blocks_for(m, 256, 148u * 4u), 256, 0, st>>>(ctx->uptr.p, uvals, m, ctx->scal.p);
    RBG_CHECK_LAUNCH(ctx);
    double trace = 0.0;
    RBG_CUDA(cudaMemcpyAsync(&trace, ctx->scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    const double mean_diag = trace / (double)m;  // solver.cpp:296
    static const double kLambdas[] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6};  // solver.cpp:298
    rbg_solve_diag local{};
    unsigned long long bad = ~0ull;
    bool solved = false;
    for (const double lambda : kLambdas) {
        ++local.attempts;
        const double shift = lambda * mean_diag;
        RBG_CUDA(cudaMemsetAsync(P.tiles.p, 0, NT * nbb * TE * sizeof(double), st));
        RBG_CUDA(cudaMemsetAsync(status.p, 0xff, sizeof(unsigned long long), st));
        band_fill_kernel<<<blocks_for(padded * 32, 256), 256, 0, st>>>(ctx->uptr.p, ctx->ucols.p, uvals, m, P.pos.p,
                                                                      shift, nbb, NT, P.tiles.p);
        RBG_CHECK_LAUNCH(ctx);
        for (uint64_t J = 0; J < NT; ++J) {
            const uint64_t dmax = std::min(nbb - 1, NT - 1 - J);
            band_panel_kernel<<<(unsigned)(dmax + 1), 32, 0, st>>>(P.tiles.p, J, nbb, P.diag.p, status.p);
            RBG_CHECK_LAUNCH(ctx);
            const uint64_t ntiles = dmax * (dmax + 1) / 2;
            if (ntiles) {
                band_update_kernel<<<(unsigned)((ntiles + 3) / 4), 128, 0, st>>>(P.tiles.p, J, nbb, NT, ntiles,
                                                                                 status.p);
                RBG_CHECK_LAUNCH(ctx);
            }
        }
        RBG_CUDA(cudaMemcpyAsync(&bad, status.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        if (bad == ~0ull) {
            solved = true;
            local.ridge_lambda = lambda;
            local.ridge_shift = shift;
            break;
        }
    }
    if (!solved) {  // solver.cpp:316-322; the pivot as a centre id of this ordering
        std::vector<uint32_t> perm(m);
        RBG_CUDA(cudaMemcpy(perm.data(), P.perm.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        const uint64_t piv = bad < m ? perm[bad] : 0;
        throw Error(RBG_RUNTIME_ERROR,
                    "normal system is not positive definite even with ridge 1e-06; first "
                    "non-positive pivot at index " + std::to_string(piv));
    }
    band_permute_kernel<true><<<blocks_for(padded, 256), 256, 0, st>>>(P.perm.p, m, padded, rhs, ctx->r.p);
    RBG_CHECK_LAUNCH(ctx);
    band_forward_kernel<<<1, kSolveWarps * 32, 0, st>>>(P.tiles.p, P.diag.p, NT, nbb, ctx->r.p, ctx->z.p);  // L y = P rhs
    RBG_CHECK_LAUNCH(ctx);
    band_backward_kernel<<<1, kSolveWarps * 32, 0, st>>>(P.tiles.p, P.diag.p, NT, nbb, ctx->z.p, ctx->q.p);  // L^T x' = y
    RBG_CHECK_LAUNCH(ctx);
    band_permute_kernel<false><<<blocks_for(padded, 256), 256, 0, st>>>(P.perm.p, m, padded, ctx->q.p, ctx->x.p);
    RBG_CHECK_LAUNCH(ctx);
    RBG_CUDA(cudaMemsetAsync(ctx->scal.p, 0, 2 * sizeof(double), st));
    ensure_f2u(ctx);
    band_residual_kernel<<<blocks_for(m * 32, 256), 256, 0, st>>>(ctx->fptr.p, ctx->fcols.p, ctx->f2u.p, uvals, rhs,
                                                                  ctx->x.p, m, ctx->scal.p);
    RBG_CHECK_LAUNCH(ctx);
    RBG_CUDA(cudaEventRecord(ctx->ev1, st));
    double rb[2] = {0, 0};
    RBG_CUDA(cudaMemcpyAsync(rb, ctx->scal.p, sizeof(rb), cudaMemcpyDeviceToHost, st));
    if (c_out) RBG_CUDA(cudaMemcpyAsync(c_out, ctx->x.p, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    for (double& a : ctx->poly_sol) a = 0.0;
    float ms = 0.f;
    RBG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    local.solve_ms = ms;
    local.iterations = 0;  // direct
    local.rel_residual = rb[1] > 0.0 ? std::sqrt(rb[0] / rb[1]) : 0.0;
    if (diag) *diag = local;
}

}  // namespace rbg
