// rbg_solve.cu -- K4: SPD solve of the assembled normal equations.
//
// Replaces solve_weights (solver.cpp:289-330).  The reference factors the
// dense M x M matrix with Eigen LLT, which is infeasible beyond M ~ 5e4 (the
// dense b alone is 8 TB at M = 1e6).  Here: preconditioned conjugate
// gradients on the symmetric CSR matrix, hand-written fp64 kernels:
//   spmv_dot     q = (B + shift I) p, fused with the p.q reduction
//   update       x += a p, r -= a q, fused with r.r and the stopping rule
//   fsai_lower   u = G r, fused with r.z = u.u          (M^-1 = G^T G, FSAI)
//   fsai_upper   z = G^T u, fused with p = z + b p
// (point Jacobi, for the bordered system: update also forms z = D^-1 r and
// r.z, then direction p = z + b p).  Scalars (alpha, beta, convergence) live on
// the device; reductions finish in the last block to arrive (fixed-order, so
// runs are deterministic) and the iteration loop is replayed from a CUDA graph
// in batches, with one host read of the convergence flags per batch.
// Stopping rule: ||r||_2 <= tol ||b||_2.  The reference's ridge ladder
// (solver.cpp:296-315) is kept: lambda x trace/side is added on breakdown, a
// non-positive pivot of a local factorisation, or non-convergence.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include <cub/cub.cuh>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

// scalar slots
enum : int {
    S_RZ = 0,
    S_PQ,
    S_RR,
    S_BB,
    S_ALPHA,
    S_BETA,
    S_SHIFT,
    S_STOP,
    S_DONE,
    S_FAIL,
    S_ITERS,
    S_MAXIT,
    S_TRACE,
    S_PIV,  // smallest centre id whose local factorisation failed (bit pattern of a double >= 0)
    S_W0,  // S_W0 .. S_W0+3: border products E^T v
    S_COUNT = S_W0 + 4
};

// Linear-polynomial border of the bordered system [[B, E], [E^T, F]]
// (solver.cpp:189-207, 238-262): E = A^T P (T x m, term-major), F = P^T P.
// T = 0 without the border.
struct BorderDev {
    int T;
    uint64_t m;
    const double* E;
    const double* F;
};

constexpr int kThreads = 256;
constexpr int kBatch = 32;
constexpr int kBatchFsai = 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of up to two values -> partials[0*grid + b], partials[1*grid + b];
// returns true in every thread of the last block to finish, after which
// out0/out1 hold the grand totals (fixed reduction order).
template <int NV>
__device__ bool last_block_sum(const double (&v)[NV], double* partials, unsigned* ticket,
                               double (&out)[NV]) {
    __shared__ double sh[NV][kThreads / 32];
    __shared__ bool is_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double s = warp_sum(v[k]);
        if (lane == 0) sh[k][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) s += sh[k][w];
            partials[k * gridDim.x + blockIdx.x] = s;
        }
        __threadfence();
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += kThreads)
            s += ((volatile double*)partials)[k * gridDim.x + b];
        s = warp_sum(s);
        __syncthreads();
        if (lane == 0) sh[k][warp] = s;
        __syncthreads();
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t += sh[k][w];
        out[k] = t;
    }
    if (threadIdx.x == 0) *ticket = 0;
    return true;
}

__global__ void gather_full_kernel(const uint64_t* __restrict__ f2u, const double* __restrict__ uvals,
                                   uint64_t nnz, double* __restrict__ vfull) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (uint64_t)gridDim.x * blockDim.x)
        vfull[e] = uvals[f2u[e]];
}

__global__ void trace_kernel(const uint64_t* __restrict__ uptr, const double* __restrict__ uvals,
                             uint64_t m, double* partials, unsigned* ticket, double* scal) {
    double v[1] = {0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        v[0] += uvals[uptr[i]];
    double out[1];
    if (last_block_sum<1>(v, partials, ticket, out) && threadIdx.x == 0) scal[S_TRACE] = out[0];
}

__global__ void init_kernel(const uint64_t* __restrict__ uptr, const double* __restrict__ uvals,
                            const double* __restrict__ b, uint64_t m, BorderDev bd, double* __restrict__ dinv,
                            double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                            double* __restrict__ p, double* partials, unsigned* ticket, double* scal,
                            double tol2) {
    const double shift = scal[S_SHIFT];
    double v[3] = {0.0, 0.0, 0.0};  // rz, bb, non-positive diagonal count
    const uint64_t nt = m + (uint64_t)bd.T;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
         i += (uint64_t)gridDim.x * blockDim.x) {
        // upper row i starts at the diagonal; border rows take F's diagonal
        const double d = (i < m ? uvals[uptr[i]] : bd.F[(i - m) * bd.T + (i - m)]) + shift;
        if (!(d > 0.0) || !isfinite(d)) v[2] += 1.0;
        const double di = 1.0 / d;
        dinv[i] = di;
        const double bi = b[i];
        x[i] = 0.0;
        r[i] = bi;
        const double zi = bi * di;
        z[i] = zi;
        p[i] = zi;
        v[0] += bi * zi;
        v[1] += bi * bi;
    }
    double out[3];
    if (last_block_sum<3>(v, partials, ticket, out) && threadIdx.x == 0) {
        scal[S_RZ] = out[0];
        scal[S_BB] = out[1];
        scal[S_STOP] = tol2 * out[1];
        scal[S_ITERS] = 0.0;
        scal[S_FAIL] = out[2] > 0.0 ? 1.0 : 0.0;
        scal[S_PIV] = INFINITY;
        scal[S_DONE] = out[1] == 0.0 ? 1.0 : 0.0;
        scal[S_RR] = out[1];
    }
}

// scal[S_W0 + t] = sum_i E[t][i] v[i]  (the E^T v half of the border SpMV)
__global__ void border_dot_kernel(BorderDev bd, const double* __restrict__ v, double* partials,
                                  unsigned* ticket, double* scal, int force) {
    if (!force && (scal[S_DONE] != 0.0 || scal[S_FAIL] != 0.0)) return;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < bd.m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double vi = v[i];
        for (int t = 0; t < bd.T; ++t) acc[t] = fma(bd.E[(uint64_t)t * bd.m + i], vi, acc[t]);
    }
    double out[4];
    if (last_block_sum<4>(acc, partials, ticket, out) && threadIdx.x == 0)
        for (int t = 0; t < 4; ++t) scal[S_W0 + t] = out[t];
}

// six resident CTAs per SM (40 registers, no spills): 48 warps of row streams
// instead of 40 (cfg5 solve 378 -> 351 ms, cfg4 285 -> 269 ms)
#ifndef RBG_SPMV_MINB
#define RBG_SPMV_MINB 6
#endif
#define RBG_SPMV_BOUNDS __launch_bounds__(kThreads, RBG_SPMV_MINB)
// q = (B + shift I) p, one warp per row; pq = p.q.
__global__ void RBG_SPMV_BOUNDS spmv_dot_kernel(const uint64_t* __restrict__ fptr, const uint32_t* __restrict__ fcols,
                                const double* __restrict__ vfull, uint64_t m, BorderDev bd,
                                const double* __restrict__ p, double* __restrict__ q,
                                double* partials, unsigned* ticket, double* scal) {
    if (scal[S_DONE] != 0.0 || scal[S_FAIL] != 0.0) return;
    const double shift = scal[S_SHIFT];
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (kThreads / 32);
    double v[1] = {0.0};
    for (uint64_t row = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < m;
         row += warps) {
        // four independent 32-entry chunks in flight per lane (memory-level
        // parallelism: a row is ~100-200 entries); the matrix streams past L2
        // (evict-first) so the gathered vector p stays resident
        const uint64_t e1 = fptr[row + 1];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        uint64_t e = fptr[row] + lane;
        for (; e + 96 < e1; e += 128) {
            const uint32_t c0 = __ldcs(fcols + e), c1 = __ldcs(fcols + e + 32), c2 = __ldcs(fcols + e + 64),
                           c3 = __ldcs(fcols + e + 96);
            const double v0 = __ldcs(vfull + e), v1 = __ldcs(vfull + e + 32), v2 = __ldcs(vfull + e + 64),
                         v3 = __ldcs(vfull + e + 96);
            s0 = fma(v0, p[c0], s0);
            s1 = fma(v1, p[c1], s1);
            s2 = fma(v2, p[c2], s2);
            s3 = fma(v3, p[c3], s3);
        }
        for (; e < e1; e += 32) s0 = fma(__ldcs(vfull + e), p[__ldcs(fcols + e)], s0);
        double s = warp_sum((s0 + s1) + (s2 + s3));
        if (lane == 0) {
            for (int t = 0; t < bd.T; ++t) s = fma(bd.E[(uint64_t)t * m + row], p[m + t], s);
            const double pi = p[row];
            const double qi = s + shift * pi;
            q[row] = qi;
            v[0] += pi * qi;
        }
    }
    double out[1];
    if (last_block_sum<1>(v, partials, ticket, out) && threadIdx.x == 0) {
        double pq = out[0];
        for (int t = 0; t < bd.T; ++t) {  // border rows: E^T p (border_dot_kernel) + F p_b
            double qt = scal[S_W0 + t] + shift * p[m + t];
            for (int u = 0; u < bd.T; ++u) qt = fma(bd.F[t * bd.T + u], p[m + u], qt);
            q[m + t] = qt;
            pq += p[m + t] * qt;
        }
        scal[S_PQ] = pq;
        if (!(pq > 0.0) || !isfinite(pq)) scal[S_FAIL] = 1.0;
        else scal[S_ALPHA] = scal[S_RZ] / pq;
    }
}

__global__ void update_kernel(uint64_t m, const double* __restrict__ p, const double* __restrict__ q,
                              const double* __restrict__ dinv, double* __restrict__ x,
                              double* __restrict__ r, double* __restrict__ z, double* partials,
                              unsigned* ticket, double* scal) {
    if (scal[S_DONE] != 0.0 || scal[S_FAIL] != 0.0) return;
    const double a = scal[S_ALPHA];
    double v[2] = {0.0, 0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        x[i] += a * p[i];
        const double ri = r[i] - a * q[i];
        r[i] = ri;
        const double zi = ri * dinv[i];
        z[i] = zi;
        v[0] += ri * zi;
        v[1] += ri * ri;
    }
    double out[2];
    if (last_block_sum<2>(v, partials, ticket, out) && threadIdx.x == 0) {
        const double rz_new = out[0];
        scal[S_BETA] = rz_new / scal[S_RZ];
        scal[S_RZ] = rz_new;
        scal[S_RR] = out[1];
        const double it = scal[S_ITERS] + 1.0;
        scal[S_ITERS] = it;
        if (!isfinite(out[1])) scal[S_FAIL] = 1.0;
        else if (out[1] <= scal[S_STOP]) scal[S_DONE] = 1.0;
        else if (it >= scal[S_MAXIT]) scal[S_FAIL] = 2.0;
    }
}

__global__ void direction_kernel(uint64_t m, const double* __restrict__ z, double* __restrict__ p,
                                 const double* scal) {
    if (scal[S_DONE] != 0.0 || scal[S_FAIL] != 0.0) return;
    const double b = scal[S_BETA];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = z[i] + b * p[i];
}

// r = b - (B + shift I) x ; returns ||r||^2 in scal[S_PQ] (reused slot)
__global__ void residual_kernel(const uint64_t* __restrict__ fptr, const uint32_t* __restrict__ fcols,
                                const double* __restrict__ vfull, uint64_t m, BorderDev bd,
                                const double* __restrict__ x, const double* __restrict__ b,
                                double* partials, unsigned* ticket, double* scal) {
    const double shift = scal[S_SHIFT];
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (kThreads / 32);
    double v[1] = {0.0};
    for (uint64_t row = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < m;
         row += warps) {
        double s = 0.0;
        for (uint64_t e = fptr[row] + lane; e < fptr[row + 1]; e += 32) s = fma(vfull[e], x[fcols[e]], s);
        s = warp_sum(s);
        if (lane == 0) {
            for (int t = 0; t < bd.T; ++t) s = fma(bd.E[(uint64_t)t * m + row], x[m + t], s);
            const double ri = b[row] - (s + shift * x[row]);
            v[0] += ri * ri;
        }
    }
    double out[1];
    if (last_block_sum<1>(v, partials, ticket, out) && threadIdx.x == 0) {
        double rr = out[0];
        for (int t = 0; t < bd.T; ++t) {
            double qt = scal[S_W0 + t] + shift * x[m + t];
            for (int u = 0; u < bd.T; ++u) qt = fma(bd.F[t * bd.T + u], x[m + u], qt);
            const double rt = b[m + t] - qt;
            rr += rt * rt;
        }
        scal[S_PQ] = rr;
    }
}


// ------------------------------------------------------ solve order
// The PCG runs in the Morton order of the centres: a permuted copy of the full
// CSR (built once per centre set) makes the SpMV's gathers of p spatially
// local (Halton centres are in random spatial order by index), and "lower
// triangular" for the FSAI factor below means "earlier in Morton order".
__device__ __forceinline__ uint64_t spread_bits(uint64_t v, int dim) {
    if (dim == 2) {  // 32 -> 64 bits
        v &= 0xffffffffull;
        v = (v | (v << 16)) & 0x0000ffff0000ffffull;
        v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
        v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
        v = (v | (v << 2)) & 0x3333333333333333ull;
        v = (v | (v << 1)) & 0x5555555555555555ull;
        return v;
    }
    v &= 0x1fffffull;  // 21 -> 63 bits
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

__global__ void bj_keys_kernel(const double* __restrict__ centres, uint64_t m, int dim, double lo0, double lo1,
                               double lo2, double scale, uint64_t* __restrict__ keys, uint32_t* __restrict__ ids) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const double lo[3] = {lo0, lo1, lo2};
        const double qmax = dim == 2 ? 4294967295.0 : 2097151.0;
        uint64_t key = 0;
        for (int d = 0; d < dim; ++d) {
            const double q = fmin(fmax((centres[i * dim + d] - lo[d]) * scale * qmax, 0.0), qmax);
            key |= spread_bits((uint64_t)q, dim) << d;
        }
        keys[i] = key;
        ids[i] = (uint32_t)i;
    }
}

__global__ void bj_pos_kernel(const uint32_t* __restrict__ perm, uint64_t m, uint32_t* __restrict__ pos) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
        pos[perm[k]] = (uint32_t)k;
}

// Sweep order of the FSAI factor: rank of every Morton position when the
// centres are sorted by (x, y, z).  "Lower" in that order is a half-space, so
// every row of G sees about half of its neighbourhood (in Morton order the
// share swings between none and all of it along the curve).
__global__ void rank_keys_kernel(const double* __restrict__ centres, const uint32_t* __restrict__ perm, uint64_t m,
                                 int dim, double lo0, double lo1, double lo2, double scale,
                                 uint64_t* __restrict__ keys, uint32_t* __restrict__ ids) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = perm[k];
        const double lo[3] = {lo0, lo1, lo2};
        const double qmax = dim == 2 ? 4294967295.0 : 2097151.0;
        uint64_t key = 0;
        for (int d = 0; d < dim; ++d) {
            const double q = fmin(fmax((centres[i * dim + d] - lo[d]) * scale * qmax, 0.0), qmax);
            key = (key << (dim == 2 ? 32 : 21)) | (uint64_t)q;
        }
        keys[k] = key;
        ids[k] = (uint32_t)k;
    }
}

// Full CSR in Morton order: new row k = centre perm[k], columns renumbered by
// pos and sorted ascending within the row (segmented sort), then pf2u = the
// upper-CSR slot of every entry (binary search in the ascending upper rows).
__global__ void perm_len_kernel(const uint64_t* __restrict__ fptr, const uint64_t* __restrict__ uptr,
                                const uint32_t* __restrict__ perm, uint64_t m, uint32_t* __restrict__ len,
                                uint64_t* __restrict__ puptr) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = perm[k];
        len[k] = (uint32_t)(fptr[i + 1] - fptr[i]);
        puptr[k] = uptr[i];
    }
}

__global__ void perm_fill_kernel(const uint64_t* __restrict__ fptr, const uint32_t* __restrict__ fcols,
                                 const uint32_t* __restrict__ perm, const uint32_t* __restrict__ pos, uint64_t m,
                                 const uint64_t* __restrict__ pfptr, uint32_t* __restrict__ pfcols) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t k = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); k < m; k += warps) {
        const uint32_t i = perm[k];
        const uint64_t s0 = fptr[i], n = fptr[i + 1] - s0, d0 = pfptr[k];
        for (uint64_t e = lane; e < n; e += 32) pfcols[d0 + e] = pos[fcols[s0 + e]];
    }
}

__global__ void perm_slots_kernel(const uint64_t* __restrict__ uptr, const uint32_t* __restrict__ ucols,
                                  const uint32_t* __restrict__ perm, uint64_t m, const uint64_t* __restrict__ pfptr,
                                  const uint32_t* __restrict__ pfcols, uint64_t* __restrict__ pf2u) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t k = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); k < m; k += warps) {
        const uint32_t i = perm[k];
        for (uint64_t e = pfptr[k] + lane; e < pfptr[k + 1]; e += 32) {
            const uint32_t j = perm[pfcols[e]];
            const uint32_t a = min(i, j), b = max(i, j);  // upper entry (a, b): ucols of row a ascending
            uint64_t lo = uptr[a], hi = uptr[a + 1];
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (ucols[mid] < b) lo = mid + 1; else hi = mid;
            }
            pf2u[e] = lo;
        }
    }
}

// v_out[k] = v[perm[k]] (to Morton order) or v_out[perm[k]] = v[k] (back).
template <bool TO_MORTON>
__global__ void permute_kernel(const uint32_t* __restrict__ perm, uint64_t m, const double* __restrict__ v,
                               double* __restrict__ out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
        if (TO_MORTON) out[k] = v[perm[k]];
        else out[perm[k]] = v[k];
    }
}

// Grid of a grid-stride kernel: at most one full wave of resident CTAs (a
// partial second wave leaves SMs idle at the tail of every launch).
template <typename K>
unsigned resident_grid(rbg_ctx* ctx, K kern, unsigned needed, size_t smem = 0, int threads = kThreads) {
    int per_sm = 0, sms = 0;
    RBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    RBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    return std::max(1u, std::min(needed, (unsigned)std::max(1, per_sm * sms)));
}

// Morton permutation of the centres, its inverse and the permuted full CSR
// (once per centre set).
void build_solve_order(rbg_ctx* ctx) {
    const uint64_t m = ctx->m;
    cudaStream_t st = ctx->stream;
    DevBuf<uint64_t> keys, keys_out;
    DevBuf<uint32_t> ids;
    keys.reserve(m);
    keys_out.reserve(m);
    ids.reserve(m);
    ctx->bj_perm.reserve(m);
    ctx->bj_pos.reserve(m);
    double span = 0.0;
    for (int d = 0; d < ctx->dim; ++d) span = std::max(span, (double)ctx->grid.n[d] * ctx->grid.edge);
    bj_keys_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->centres.p, m, ctx->dim, ctx->grid.lo[0], ctx->grid.lo[1],
                                                      ctx->grid.lo[2], span > 0.0 ? 1.0 / span : 1.0, keys.p, ids.p);
    RBG_CHECK_LAUNCH(ctx);
    size_t tmp_bytes = 0;
    RBG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_out.p, ids.p, ctx->bj_perm.p, (int)m, 0,
                                             64, st));
    DevBuf<unsigned char> tmp;
    tmp.reserve(tmp_bytes);
    RBG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys_out.p, ids.p, ctx->bj_perm.p, (int)m, 0,
                                             64, st));
    bj_pos_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->bj_perm.p, m, ctx->bj_pos.p);
    RBG_CHECK_LAUNCH(ctx);
    {  // sweep rank of every Morton position (stable sort: ties keep their Morton order)
        DevBuf<uint32_t> order;
        order.reserve(m);
        ctx->prank.reserve(m);
        rank_keys_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->centres.p, ctx->bj_perm.p, m, ctx->dim,
                                                            ctx->grid.lo[0], ctx->grid.lo[1], ctx->grid.lo[2],
                                                            span > 0.0 ? 1.0 / span : 1.0, keys.p, ids.p);
        RBG_CHECK_LAUNCH(ctx);
        RBG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys_out.p, ids.p, order.p, (int)m, 0, 64,
                                                 st));
        bj_pos_kernel<<<blocks_for(m, 256), 256, 0, st>>>(order.p, m, ctx->prank.p);
        RBG_CHECK_LAUNCH(ctx);
        RBG_CUDA(cudaStreamSynchronize(st));
    }
    DevBuf<uint32_t> len;
    len.reserve(m + 1);
    ctx->pfptr.reserve(m + 1);
    ctx->puptr.reserve(m);
    ctx->pfcols.reserve(ctx->nnz_full + 4);  // the FSAI row staging reads whole 16-byte pieces
    ctx->pf2u.reserve(ctx->nnz_full);
    perm_len_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->fptr.p, ctx->uptr.p, ctx->bj_perm.p, m, len.p,
                                                       ctx->puptr.p);
    RBG_CHECK_LAUNCH(ctx);
    exclusive_scan_u32_to_u64(ctx, len.p, ctx->pfptr.p, m);
    const unsigned gf = blocks_for(m, 8, 148u * 16u);
    perm_fill_kernel<<<gf, 256, 0, st>>>(ctx->fptr.p, ctx->fcols.p, ctx->bj_perm.p, ctx->bj_pos.p, m, ctx->pfptr.p,
                                         ctx->pfcols.p);
    RBG_CHECK_LAUNCH(ctx);
    segmented_sort_u32(ctx, ctx->pfcols.p, ctx->pfptr.p, m, ctx->max_full_row);
    perm_slots_kernel<<<gf, 256, 0, st>>>(ctx->uptr.p, ctx->ucols.p, ctx->bj_perm.p, m, ctx->pfptr.p, ctx->pfcols.p,
                                          ctx->pf2u.p);
    RBG_CHECK_LAUNCH(ctx);
    RBG_CUDA(cudaStreamSynchronize(st));  // temporaries are released at scope end
    ctx->bj_built = true;
}

// ------------------------------------------------------ FSAI preconditioner
// Factorised sparse approximate inverse (Kolotilina-Yeremin): G ~ L^-1 for
// B + shift I = L L^T in the sweep order (centres sorted by x, y, z) with the
// prescribed pattern  P_k = the (up to) 31 nearest pattern neighbours of k that
// come before it in the sweep (within rho r) + {k}.  Row k of G is the last row
// of chol(B[P_k, P_k])^-1 with k ordered last -- one 32 x 32 dense SPD
// factorisation per centre, all independent, held in the registers of one
// warp -- and M^-1 = G^T G.  A^T A of compactly supported kernels is
// ill-conditioned through its local oscillatory modes, which these local
// factorisations capture: the CG iteration count drops from O(1000) (block
// Jacobi) to ~40.  (The whole pattern of B as P_k gives 13-17 iterations, but
// its 81 x 81 factorisations cost more than the iterations they save.)  G and
// G^T are stored as two CSRs with Morton-ordered rows (the order the CG
// vectors live in); nothing needs G to be triangular in that order.  A
// non-positive local pivot fails the attempt, so the reference's ridge ladder
// (solver.cpp:296-315) moves to the next lambda.
constexpr int kFsaiN = 32;       // rows of a local system: one per lane
constexpr int kFsaiWarps = 4;    // warps per CTA in the pattern and setup kernels

__device__ __forceinline__ double fsai_dist2(const double* __restrict__ centres, int dim, uint32_t ci, uint32_t cj) {
    double d2 = 0.0;
    for (int d = 0; d < dim; ++d) {
        const double t = centres[(uint64_t)ci * dim + d] - centres[(uint64_t)cj * dim + d];
        d2 += t * t;
    }
    return d2;
}

// tau[k]: squared radius below which row k keeps its earlier-in-sweep
// neighbours -- the largest of 24 bisection steps in (0, rad2] that keeps at
// most kFsaiN - 1 of them; glen[k] = that count + 1 (k itself).
__global__ void __launch_bounds__(kFsaiWarps * 32) fsai_radius_kernel(
    const uint64_t* __restrict__ pfptr, const uint32_t* __restrict__ pfcols, const uint32_t* __restrict__ perm,
    const uint32_t* __restrict__ rank, const double* __restrict__ centres, int dim, double rad2, uint64_t m,
    uint32_t rowcap, double* __restrict__ tau, uint32_t* __restrict__ glen) {
    extern __shared__ double fr_sm[];  // per warp: squared distances of the earlier neighbours
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* dd = fr_sm + (size_t)w * rowcap;
    const uint64_t warps = (uint64_t)gridDim.x * kFsaiWarps;
    for (uint64_t k = blockIdx.x * (uint64_t)kFsaiWarps + w; k < m; k += warps) {
        const uint32_t ci = perm[k], rk = rank[k];
        const uint64_t e0 = pfptr[k];
        const int len = (int)(pfptr[k + 1] - e0);
        for (int e = lane; e < len; e += 32) {
            const uint32_t c = pfcols[e0 + e];
            dd[e] = (c != (uint32_t)k && rank[c] < rk) ? fsai_dist2(centres, dim, ci, perm[c]) : 1e300;
        }
        __syncwarp();
        const auto count_below = [&](double t) {
            int n = 0;
            for (int e = lane; e < len; e += 32) n += dd[e] < t ? 1 : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
            return n;
        };
        double hi = rad2;
        int n = count_below(hi);
        if (n > kFsaiN - 1) {
            double lo = 0.0;  // count_below(lo) = 0
            n = 0;
            for (int it = 0; it < 24; ++it) {
                const double mid = 0.5 * (lo + hi);
                const int nm = count_below(mid);
                if (nm > kFsaiN - 1) {
                    hi = mid;
                } else {
                    lo = mid;
                    n = nm;
                }
            }
            hi = lo;
        }
        if (lane == 0) {
            tau[k] = hi;
            glen[k] = (uint32_t)n + 1u;
        }
        __syncwarp();
    }
}

// FILL = false: row lengths of G^T (row j: every k after j in the sweep that
// keeps j, and j itself); FILL = true: the column lists of G and G^T, ascending
// in Morton position (order-preserving compaction), k itself last in its G row.
template <bool FILL>
__global__ void fsai_pattern_kernel(const uint64_t* __restrict__ pfptr, const uint32_t* __restrict__ pfcols,
                                    const uint32_t* __restrict__ perm, const uint32_t* __restrict__ rank,
                                    const double* __restrict__ centres, int dim, const double* __restrict__ tau,
                                    uint64_t m, uint32_t* __restrict__ tlen, const uint64_t* __restrict__ gptr,
                                    const uint64_t* __restrict__ tptr, uint32_t* __restrict__ gcols,
                                    uint32_t* __restrict__ tcols) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t k = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); k < m; k += warps) {
        const uint32_t ci = perm[k], rk = rank[k];
        const double tk = tau[k];
        const uint64_t e0 = pfptr[k], e1 = pfptr[k + 1];
        uint32_t nl = 0, nu = 0;
        for (uint64_t eb = e0; eb < e1; eb += 32) {
            const uint64_t e = eb + lane;
            uint32_t c = 0;
            bool lower = false, upper = false;
            if (e < e1) {
                c = pfcols[e];
                if (c == (uint32_t)k) {
                    upper = true;  // the diagonal: in G^T's row here, appended to G's row below
                } else {
                    const double d2 = fsai_dist2(centres, dim, ci, perm[c]);
                    if (rank[c] < rk) lower = FILL && d2 < tk;
                    else upper = d2 < tau[c];
                }
            }
            const unsigned lo = __ballot_sync(0xffffffffu, lower);
            const unsigned up = __ballot_sync(0xffffffffu, upper);
            if (FILL) {
                const unsigned below = (1u << lane) - 1u;
                if (lower) gcols[gptr[k] + nl + __popc(lo & below)] = c;
                if (upper) tcols[tptr[k] + nu + __popc(up & below)] = c;
            }
            nl += __popc(lo);
            nu += __popc(up);
        }
        if (lane == 0) {
            if (FILL) gcols[gptr[k] + nl] = (uint32_t)k;
            else tlen[k] = nu;
        }
    }
}

// tmap[e] for the G^T entry (row j, column k): where G's entry (k, j) lives.
__global__ void fsai_tmap_kernel(const uint64_t* __restrict__ tptr, const uint32_t* __restrict__ tcols,
                                 const uint64_t* __restrict__ gptr, const uint32_t* __restrict__ gcols, uint64_t m,
                                 uint32_t* __restrict__ tmap) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t j = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); j < m; j += warps) {
        for (uint64_t e = tptr[j] + lane; e < tptr[j + 1]; e += 32) {
            const uint32_t k = tcols[e];
            uint64_t lo = gptr[k], hi = gptr[k + 1] - 1;  // the last entry of G's row k is k itself
            if (k == (uint32_t)j) lo = hi;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (gcols[mid] < (uint32_t)j) lo = mid + 1; else hi = mid;
            }
            tmap[e] = (uint32_t)lo;
        }
    }
}

__global__ void fsai_transpose_kernel(const uint32_t* __restrict__ tmap, const double* __restrict__ gvals, uint64_t nnz,
                                      double* __restrict__ tvals, const double* scal) {
    if (scal[S_FAIL] != 0.0) return;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * blockDim.x)
        tvals[e] = gvals[tmap[e]];
}

// One warp per row k of G; lane a owns local row a (P[a], k last).
//  gather     for every a, lane b <= a finds P[b] in B's row P[a] (columns
//             ascending: binary search) and files B[P[a], P[b]] into S[a][b]
//             in shared memory, from where lane a takes its row;
//  factorise  right-looking Cholesky of the 32 x 32 system with row a in the
//             registers of lane a: per column one pivot broadcast, the column
//             parked in shared memory, one broadcast load + FMA per trailing
//             column (rows past n are identity);
//  solve      L^T x = e_n from the last row up: x = row k of G.
constexpr int kFsaiStages = 4;  // row buffers in flight per warp (cp.async)
inline size_t fsai_setup_smem(uint32_t rowcap) {
    return (size_t)kFsaiWarps * (kFsaiN * (kFsaiN + 1) * sizeof(double) + (size_t)kFsaiStages * rowcap * sizeof(uint32_t));
}

__global__ void __launch_bounds__(kFsaiWarps * 32) fsai_setup_kernel(
    const uint64_t* __restrict__ pfptr, const uint32_t* __restrict__ pfcols, const double* __restrict__ vfull,
    const uint64_t* __restrict__ gptr, const uint32_t* __restrict__ gcols, uint64_t m, uint32_t rowcap,
    const uint32_t* __restrict__ perm, double* scal, double* __restrict__ gvals) {
    if (scal[S_FAIL] != 0.0) return;
    extern __shared__ __align__(16) unsigned char fs_sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double (*S)[kFsaiN + 1] = reinterpret_cast<double (*)[kFsaiN + 1]>(fs_sm) + (size_t)w * kFsaiN;
    uint32_t* rbuf = reinterpret_cast<uint32_t*>(fs_sm + (size_t)kFsaiWarps * kFsaiN * (kFsaiN + 1) * sizeof(double)) +
                     (size_t)w * kFsaiStages * rowcap;
    const double shift = scal[S_SHIFT];
    const uint64_t warps = (uint64_t)gridDim.x * kFsaiWarps;
    for (uint64_t k = blockIdx.x * (uint64_t)kFsaiWarps + w; k < m; k += warps) {
        const uint64_t g0 = gptr[k];
        const int n = (int)(gptr[k + 1] - g0);
        const uint32_t mine = lane < n ? gcols[g0 + lane] : 0u;
        const uint64_t my0 = pfptr[mine];
        const uint32_t mylen = (uint32_t)(pfptr[mine + 1] - my0);
        // the columns of B's row P[a] -> row buffer a % kFsaiStages (asynchronous)
        const auto issue_row = [&](int a) {
            if (a < n) {
                // 16-byte pieces from the row start rounded down to a multiple of 4 entries
                // (the row then begins at offset e0 & 3 of the buffer)
                const uint64_t e0 = __shfl_sync(0xffffffffu, my0, a);
                const uint32_t len = __shfl_sync(0xffffffffu, mylen, a) + (uint32_t)(e0 & 3);
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(rbuf + (a % kFsaiStages) * rowcap);
                const uint32_t* src = pfcols + (e0 & ~3ull);
                for (uint32_t e = 4 * lane; e < len; e += 128)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 4u * e), "l"(src + e)
                                 : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
#pragma unroll
        for (int a = 0; a < kFsaiStages - 1; ++a) issue_row(a);
#pragma unroll
        for (int j = 0; j < kFsaiN; ++j) S[lane][j] = j == lane && lane >= n ? 1.0 : 0.0;
        // S[a][b] = B[P[a], P[b]] for b <= a: lane b looks P[b] up in B's row P[a]
        // (columns ascending: a branch-free lower bound in the staged row); the
        // value load of one row is consumed while the next row is searched
        double vprev = 0.0;
        bool hprev = false;
        for (int a = 0; a < n; ++a) {
            issue_row(a + kFsaiStages - 1);
            asm volatile("cp.async.wait_group %0;" ::"n"(kFsaiStages - 1) : "memory");
            __syncwarp();
            const uint64_t e0 = __shfl_sync(0xffffffffu, my0, a);
            const uint32_t len = __shfl_sync(0xffffffffu, mylen, a);
            const uint32_t* rc = rbuf + (a % kFsaiStages) * rowcap + (e0 & 3);
            uint32_t lo = 0;
            for (uint32_t step = 1u << (31 - __clz(len)); step > 0; step >>= 1)
                if (lo + step <= len && rc[lo + step - 1] < mine) lo += step;
            const bool hit = lane <= a && lo < len && rc[lo] == mine;
            const double v = hit ? vfull[e0 + lo] : 0.0;
            if (hprev) S[a - 1][lane] = lane == a - 1 ? vprev + shift : vprev;
            vprev = v;
            hprev = hit;
            __syncwarp();  // the buffer is refilled kFsaiStages - 1 rows from now
        }
        if (hprev) S[n - 1][lane] = lane == n - 1 ? vprev + shift : vprev;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        double row[kFsaiN];
#pragma unroll
        for (int j = 0; j < kFsaiN; ++j) row[j] = S[lane][j];
        __syncwarp();
        // S is reused for L, column-major (Lc[j][i] = L[i][j]): every finished column is
        // parked there, the trailing update reads it back as broadcasts (one LDS per
        // column instead of a two-instruction 64-bit shuffle) and the solve below walks it
        double* Lc = &S[0][0];
        constexpr int LD = kFsaiN + 1;
        bool bad = false;
        double myinv = 1.0;
#pragma unroll
        for (int j = 0; j < kFsaiN; ++j) {
            if (j < n) {  // rows past n are identity
                double d = __shfl_sync(0xffffffffu, row[j], j);
                if (!(d > 0.0) || !isfinite(d)) {
                    bad = true;
                    d = 1.0;
                }
                const double inv = rsqrt(d);
                if (lane == j) myinv = inv;      // 1 / L[j][j] for the solve below
                const double lj = row[j] * inv;  // column j of L (rows >= j; lane j: sqrt(d))
                Lc[j * LD + lane] = lj;
                __syncwarp();
#pragma unroll
                for (int c = j + 1; c < kFsaiN; ++c) row[c] = fma(-lj, Lc[j * LD + c], row[c]);
            }
        }
        if (bad) {
            if (lane == 0) {
                scal[S_FAIL] = 1.0;
                atomicMin(reinterpret_cast<unsigned long long*>(scal + S_PIV),
                          (unsigned long long)__double_as_longlong((double)perm[k]));
            }
            __syncwarp();
            continue;
        }
        // L^T x = e_{n-1}, column by column: once x_i is final, row i of L updates x_0 .. x_{i-1}
        double x = lane == n - 1 ? 1.0 : 0.0;
        for (int i = n - 1; i >= 0; --i) {
            if (lane == i) x *= myinv;
            const double xi = __shfl_sync(0xffffffffu, x, i);
            if (lane < i) x = fma(-Lc[lane * LD + i], xi, x);
        }
        if (lane < n) gvals[g0 + lane] = x;
        __syncwarp();
    }
}

// Rows of G and G^T hold about 32 entries, so the applies give a row to a
// group of 8 lanes (4 rows per warp, 3 shuffle steps per row sum).
constexpr int kRowLanes = 8;
constexpr int kRowsPerWarp = 32 / kRowLanes;

__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = kRowLanes / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double sparse_row_dot(const uint64_t* __restrict__ ptr, const uint32_t* __restrict__ cols,
                                                 const double* __restrict__ vals, uint64_t row, bool valid, int sl,
                                                 const double* __restrict__ x) {
    double s0 = 0.0, s1 = 0.0;
    if (valid) {
        const uint64_t e1 = ptr[row + 1];
        uint64_t e = ptr[row] + sl;
        for (; e + kRowLanes < e1; e += 2 * kRowLanes) {
            const uint32_t c0 = __ldcs(cols + e), c1 = __ldcs(cols + e + kRowLanes);
            const double v0 = __ldcs(vals + e), v1 = __ldcs(vals + e + kRowLanes);
            s0 = fma(v0, x[c0], s0);
            s1 = fma(v1, x[c1], s1);
        }
        if (e < e1) s0 = fma(__ldcs(vals + e), x[__ldcs(cols + e)], s0);
    }
    return group_sum(s0 + s1);
}

// u = G r, rz = u.u (= r.M^-1 r); INIT: scal[S_RZ] = rz, else beta = rz / rz_old.
template <bool INIT>
__global__ void __launch_bounds__(kThreads) fsai_lower_kernel(const uint64_t* __restrict__ gptr,
                                                              const uint32_t* __restrict__ gcols,
                                                              const double* __restrict__ gvals, uint64_t m,
                                                              const double* __restrict__ r, double* __restrict__ u,
                                                              double* partials, unsigned* ticket, double* scal) {
    if (scal[S_FAIL] != 0.0 || (!INIT && scal[S_DONE] != 0.0)) return;
    const int lane = threadIdx.x & 31, sub = lane / kRowLanes, sl = lane % kRowLanes;
    const uint64_t stride = (uint64_t)gridDim.x * (kThreads / 32) * kRowsPerWarp;
    double v[1] = {0.0};
    for (uint64_t base = ((uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * kRowsPerWarp; base < m;
         base += stride) {
        const uint64_t row = base + sub;
        const double s = sparse_row_dot(gptr, gcols, gvals, row, row < m, sl, r);
        if (sl == 0 && row < m) {
            u[row] = s;
            v[0] += s * s;
        }
    }
    double out[1];
    if (last_block_sum<1>(v, partials, ticket, out) && threadIdx.x == 0) {
        if (!INIT) scal[S_BETA] = out[0] / scal[S_RZ];
        scal[S_RZ] = out[0];
    }
}

// z = G^T u and the new direction p = z + beta p (INIT: p = z).
template <bool INIT>
__global__ void __launch_bounds__(kThreads) fsai_upper_kernel(const uint64_t* __restrict__ tptr,
                                                              const uint32_t* __restrict__ tcols,
                                                              const double* __restrict__ tvals, uint64_t m,
                                                              const double* __restrict__ u, double* __restrict__ p,
                                                              const double* scal) {
    if (scal[S_FAIL] != 0.0 || (!INIT && scal[S_DONE] != 0.0)) return;
    const double beta = INIT ? 0.0 : scal[S_BETA];
    const int lane = threadIdx.x & 31, sub = lane / kRowLanes, sl = lane % kRowLanes;
    const uint64_t stride = (uint64_t)gridDim.x * (kThreads / 32) * kRowsPerWarp;
    for (uint64_t base = ((uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * kRowsPerWarp; base < m;
         base += stride) {
        const uint64_t row = base + sub;
        const double s = sparse_row_dot(tptr, tcols, tvals, row, row < m, sl, u);
        if (sl == 0 && row < m) p[row] = INIT ? s : fma(beta, p[row], s);
    }
}

// The CG update of the FSAI path: x += a p, r -= a q, rr and the stopping rule
// (z and r.z come from fsai_lower_kernel).
__global__ void update_plain_kernel(uint64_t m, const double* __restrict__ p, const double* __restrict__ q,
                                    double* __restrict__ x, double* __restrict__ r, double* partials,
                                    unsigned* ticket, double* scal) {
    if (scal[S_DONE] != 0.0 || scal[S_FAIL] != 0.0) return;
    const double a = scal[S_ALPHA];
    double v[1] = {0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        x[i] += a * p[i];
        const double ri = r[i] - a * q[i];
        r[i] = ri;
        v[0] += ri * ri;
    }
    double out[1];
    if (last_block_sum<1>(v, partials, ticket, out) && threadIdx.x == 0) {
        scal[S_RR] = out[0];
        const double it = scal[S_ITERS] + 1.0;
        scal[S_ITERS] = it;
        if (!isfinite(out[0])) scal[S_FAIL] = 1.0;
        else if (out[0] <= scal[S_STOP]) scal[S_DONE] = 1.0;
        else if (it >= scal[S_MAXIT]) scal[S_FAIL] = 2.0;
    }
}

// Pattern of G and G^T for the current centre set (once per centre set).
void fsai_build(rbg_ctx* ctx) {
    const uint64_t m = ctx->m;
    cudaStream_t st = ctx->stream;
    static const double rho_env = [] {
        const char* e = std::getenv("RBG_FSAI_RHO");
        return e ? std::atof(e) : 0.0;
    }();
    const double rho = rho_env > 0.0 ? std::min(rho_env, 2.0) : 2.0;  // 2 = anywhere in the pattern of B
    const double rad2 = rho >= 2.0 ? 8.0 * ctx->r2 : rho * rho * ctx->r2;
    DevBuf<uint32_t> glen, tlen;
    DevBuf<double> tau;
    glen.reserve(m + 1);
    tlen.reserve(m + 1);
    tau.reserve(m);
    const unsigned gw = blocks_for(m, kFsaiWarps, 148u * 16u);
    const uint32_t rowcap = (ctx->max_full_row + 31u) & ~31u;
    fsai_radius_kernel<<<gw, kFsaiWarps * 32, (size_t)kFsaiWarps * rowcap * sizeof(double), st>>>(
        ctx->pfptr.p, ctx->pfcols.p, ctx->bj_perm.p, ctx->prank.p, ctx->centres.p, ctx->dim, rad2, m, rowcap, tau.p,
        glen.p);
    RBG_CHECK_LAUNCH(ctx);
    fsai_pattern_kernel<false><<<gw, kFsaiWarps * 32, 0, st>>>(ctx->pfptr.p, ctx->pfcols.p, ctx->bj_perm.p,
                                                                ctx->prank.p, ctx->centres.p, ctx->dim, tau.p, m, tlen.p,
                                                                nullptr, nullptr, nullptr, nullptr);
    RBG_CHECK_LAUNCH(ctx);
    ctx->fs_gptr.reserve(m + 1);
    ctx->fs_tptr.reserve(m + 1);
    exclusive_scan_u32_to_u64(ctx, glen.p, ctx->fs_gptr.p, m);
    exclusive_scan_u32_to_u64(ctx, tlen.p, ctx->fs_tptr.p, m);
    uint64_t nnz = 0;
    RBG_CUDA(cudaMemcpyAsync(&nnz, ctx->fs_gptr.p + m, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    if (nnz >= (1ull << 32)) throw Error(RBG_RUNTIME_ERROR, "internal: FSAI factor beyond 2^32 entries");
    ctx->fs_gcols.reserve(nnz);
    ctx->fs_tcols.reserve(nnz);
    ctx->fs_tmap.reserve(nnz);
    ctx->fs_gvals.reserve(nnz);
    ctx->fs_tvals.reserve(nnz);
    ctx->fs_u.reserve(m);
    fsai_pattern_kernel<true><<<gw, kFsaiWarps * 32, 0, st>>>(ctx->pfptr.p, ctx->pfcols.p, ctx->bj_perm.p, ctx->prank.p,
                                                               ctx->centres.p, ctx->dim, tau.p, m, nullptr,
                                                               ctx->fs_gptr.p, ctx->fs_tptr.p, ctx->fs_gcols.p,
                                                               ctx->fs_tcols.p);
    RBG_CHECK_LAUNCH(ctx);
    fsai_tmap_kernel<<<gw, kFsaiWarps * 32, 0, st>>>(ctx->fs_tptr.p, ctx->fs_tcols.p, ctx->fs_gptr.p, ctx->fs_gcols.p, m,
                                                     ctx->fs_tmap.p);
    RBG_CHECK_LAUNCH(ctx);
    RBG_CUDA(cudaStreamSynchronize(st));  // temporaries are released at scope end
    ctx->fs_rho = rho;
    ctx->fs_nnz = nnz;
    ctx->fs_built = true;
}

// G for the current values and shift, and its transposed copy (once per ridge attempt).
void fsai_setup(rbg_ctx* ctx, cudaStream_t st) {
    const uint32_t rowcap = (ctx->max_full_row + 3u + 31u) & ~31u;  // + the alignment shift of a staged row
    const size_t smem = fsai_setup_smem(rowcap);
    RBG_CUDA(cudaFuncSetAttribute(fsai_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = resident_grid(ctx, fsai_setup_kernel, blocks_for(ctx->m, kFsaiWarps, ~0u), smem,
                                        kFsaiWarps * 32);
    fsai_setup_kernel<<<grid, kFsaiWarps * 32, smem, st>>>(ctx->pfptr.p, ctx->pfcols.p, ctx->vfull.p, ctx->fs_gptr.p,
                                                           ctx->fs_gcols.p, ctx->m, rowcap, ctx->bj_perm.p,
                                                           ctx->scal.p, ctx->fs_gvals.p);
    RBG_CHECK_LAUNCH(ctx);
    fsai_transpose_kernel<<<blocks_for(ctx->fs_nnz, kThreads), kThreads, 0, st>>>(ctx->fs_tmap.p, ctx->fs_gvals.p,
                                                                                  ctx->fs_nnz, ctx->fs_tvals.p,
                                                                                  ctx->scal.p);
    RBG_CHECK_LAUNCH(ctx);
}

}  // namespace

namespace {
int solver_env() {  // RBG_SOLVER=pcg / band forces a method (tests, A/B)
    static const int forced = [] {
        const char* e = std::getenv("RBG_SOLVER");
        return !e ? 0 : std::string(e) == "pcg" ? RBG_SOLVE_PCG : std::string(e) == "band" ? RBG_SOLVE_BAND : 0;
    }();
    return forced;
}
int prec_env() {  // RBG_PREC=jacobi / fsai forces a preconditioner
    static const int forced = [] {
        const char* e = std::getenv("RBG_PREC");
        return !e ? 0 : std::string(e) == "jacobi" ? RBG_PREC_JACOBI : std::string(e) == "fsai" ? RBG_PREC_FSAI : 0;
    }();
    return forced;
}
}  // namespace

// The centre-side structures of the default solve (Morton order, permuted CSR,
// FSAI pattern), built ahead of the first solve where that is free: rbg_assemble
// calls this while a large host input is still uploading.
// The FSAI kernels stage whole rows of B in shared memory; beyond 1024 entries
// per row (hundreds of centres per support -- far outside the method's regime)
// the solve keeps point Jacobi.
bool fsai_fits(const rbg_ctx* ctx) { return ctx->max_full_row <= 1024u; }

void prepare_solver(rbg_ctx* ctx) {
    if (ctx->pterms() != 0 || solver_env() == RBG_SOLVE_BAND || prec_env() == RBG_PREC_JACOBI || !fsai_fits(ctx)) return;
    if (!ctx->bj_built) build_solve_order(ctx);
    if (!ctx->fs_built) fsai_build(ctx);
}

void solve_system(rbg_ctx* ctx, const rbg_solve_options* opts, double* c_out, rbg_solve_diag* diag) {
    // method: FSAI-preconditioned CG unless the caller (rbg_solve_options::method)
    // or the environment asks for the banded LLT of rbg_band.cu, the reference's
    // own factorisation
    const int forced = solver_env();
    const int method = forced ? forced : (opts ? opts->method : 0);
    if (method == RBG_SOLVE_BAND) {
        if (ctx->pterms() != 0)
            throw Error(RBG_INVALID_ARGUMENT, "solve: the banded LLT does not take the polynomial border");
        band_plan(ctx);
        band_solve(ctx, c_out, diag);
        return;
    }
    cudaStream_t st = ctx->stream;
    const uint64_t m = ctx->m, nnz = ctx->nnz_full;
    const double tol = (opts && opts->tol > 0.0) ? opts->tol : 1e-12;
    const int max_iter = (opts && opts->max_iter > 0) ? opts->max_iter : 20000;
    const double* uvals = ctx->sys.p;
    const int T = ctx->pterms();
    const uint64_t nt = m + (uint64_t)T;  // unknowns: c (m) and the border coefficients (T)
    BorderDev bd{T, m, nullptr, nullptr};
    const double* b = ctx->sys.p + ctx->nnz_upper;
    std::vector<double> hF(16, 0.0);
    if (T) {
        bd.E = ctx->sys.p + ctx->border_off();
        bd.F = bd.E + (uint64_t)T * m;
        // contiguous right-hand side [A^T h | P^T h]
        ctx->bvec.reserve(nt);
        RBG_CUDA(cudaMemcpyAsync(ctx->bvec.p, b, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
        RBG_CUDA(cudaMemcpyAsync(ctx->bvec.p + m, bd.F + T * T, T * sizeof(double), cudaMemcpyDeviceToDevice, st));
        RBG_CUDA(cudaMemcpyAsync(hF.data(), bd.F, T * T * sizeof(double), cudaMemcpyDeviceToHost, st));
        b = ctx->bvec.p;
    }

    ctx->vfull.reserve(nnz);
    for (auto* v : {&ctx->x, &ctx->r, &ctx->z, &ctx->p, &ctx->q, &ctx->dinv}) v->reserve(nt);
    const unsigned g_vec = blocks_for(nt, kThreads, 148u * 4u);
    const unsigned g_spmv = resident_grid(ctx, spmv_dot_kernel, blocks_for(m, kThreads / 32, ~0u));
    ctx->partials.reserve(4ull * std::max(g_vec, g_spmv));
    ctx->scal.reserve(S_COUNT);
    ctx->ticket.reserve(1);
    RBG_CUDA(cudaMemsetAsync(ctx->ticket.p, 0, sizeof(unsigned), st));
    RBG_CUDA(cudaMemsetAsync(ctx->scal.p, 0, S_COUNT * sizeof(double), st));

    // preconditioner: FSAI (in the Morton order of the centres) unless the caller
    // or RBG_PREC=jacobi asks for point Jacobi, or the system is bordered
    const int prec = prec_env() ? prec_env() : (opts ? opts->precond : 0);
    const bool fsai = prec != RBG_PREC_JACOBI && T == 0 && fsai_fits(ctx);
    if (fsai && !ctx->bj_built) build_solve_order(ctx);
    if (fsai && !ctx->fs_built) fsai_build(ctx);
    const uint64_t* s_fptr = fsai ? ctx->pfptr.p : ctx->fptr.p;
    const uint32_t* s_fcols = fsai ? ctx->pfcols.p : ctx->fcols.p;
    const uint64_t* s_uptr = fsai ? ctx->puptr.p : ctx->uptr.p;  // diagonal of each solve row

    if (!fsai) ensure_f2u(ctx);
    RBG_CUDA(cudaEventRecord(ctx->ev0, st));
    gather_full_kernel<<<blocks_for(nnz, kThreads), kThreads, 0, st>>>(fsai ? ctx->pf2u.p : ctx->f2u.p, uvals, nnz,
                                                                        ctx->vfull.p);
    RBG_CHECK_LAUNCH(ctx);
    if (fsai) {  // right-hand side to Morton order
        ctx->bvec.reserve(m);
        permute_kernel<true><<<g_vec, kThreads, 0, st>>>(ctx->bj_perm.p, m, b, ctx->bvec.p);
        RBG_CHECK_LAUNCH(ctx);
        b = ctx->bvec.p;
    }
    trace_kernel<<<g_vec, kThreads, 0, st>>>(ctx->uptr.p, uvals, m, ctx->partials.p, ctx->ticket.p,
                                             ctx->scal.p);
    RBG_CHECK_LAUNCH(ctx);
    double trace = 0.0;
    RBG_CUDA(cudaMemcpyAsync(&trace, ctx->scal.p + S_TRACE, sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    for (int t = 0; t < T; ++t) trace += hF[t * T + t];
    const double mean_diag = trace / (double)nt;  // solver.cpp:296 (trace / side)

    const unsigned g_fs =
        fsai ? resident_grid(ctx, fsai_lower_kernel<false>, blocks_for(m, kThreads / 32 * kRowsPerWarp, ~0u)) : 0u;
    if (fsai) ctx->partials.reserve(4ull * std::max({g_vec, g_spmv, g_fs}));

    // one batch of iterations as a graph (kernels read their scalars on device);
    // the FSAI solve takes tens of iterations, so its batches are short
    const int batch = fsai ? kBatchFsai : kBatch;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    RBG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < batch; ++it) {
        if (T)
            border_dot_kernel<<<g_vec, kThreads, 0, st>>>(bd, ctx->p.p, ctx->partials.p, ctx->ticket.p,
                                                          ctx->scal.p, 0);
        spmv_dot_kernel<<<g_spmv, kThreads, 0, st>>>(s_fptr, s_fcols, ctx->vfull.p, m, bd,
                                                     ctx->p.p, ctx->q.p, ctx->partials.p,
                                                     ctx->ticket.p, ctx->scal.p);
        if (fsai) {
            update_plain_kernel<<<g_vec, kThreads, 0, st>>>(m, ctx->p.p, ctx->q.p, ctx->x.p, ctx->r.p,
                                                            ctx->partials.p, ctx->ticket.p, ctx->scal.p);
            fsai_lower_kernel<false><<<g_fs, kThreads, 0, st>>>(ctx->fs_gptr.p, ctx->fs_gcols.p, ctx->fs_gvals.p, m,
                                                                ctx->r.p, ctx->fs_u.p, ctx->partials.p,
                                                                ctx->ticket.p, ctx->scal.p);
            fsai_upper_kernel<false><<<g_fs, kThreads, 0, st>>>(ctx->fs_tptr.p, ctx->fs_tcols.p, ctx->fs_tvals.p, m,
                                                                ctx->fs_u.p, ctx->p.p, ctx->scal.p);
        } else {
            update_kernel<<<g_vec, kThreads, 0, st>>>(nt, ctx->p.p, ctx->q.p, ctx->dinv.p, ctx->x.p,
                                                      ctx->r.p, ctx->z.p, ctx->partials.p,
                                                      ctx->ticket.p, ctx->scal.p);
            direction_kernel<<<g_vec, kThreads, 0, st>>>(nt, ctx->z.p, ctx->p.p, ctx->scal.p);
        }
    }
    RBG_CUDA(cudaStreamEndCapture(st, &graph));
    RBG_CUDA(cudaGraphInstantiate(&exec, graph, 0));

    static const double kLambdas[] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6};  // solver.cpp:298
    rbg_solve_diag local{};
    bool solved = false;
    double flags[3] = {0, 0, 0};
    try {
        for (const double lambda : kLambdas) {
            ++local.attempts;
            const double shift = lambda * mean_diag;
            const double init[2] = {shift, (double)max_iter};
            RBG_CUDA(cudaMemcpyAsync(ctx->scal.p + S_SHIFT, &init[0], sizeof(double),
                                     cudaMemcpyHostToDevice, st));
            RBG_CUDA(cudaMemcpyAsync(ctx->scal.p + S_MAXIT, &init[1], sizeof(double),
                                     cudaMemcpyHostToDevice, st));
            init_kernel<<<g_vec, kThreads, 0, st>>>(s_uptr, uvals, b, m, bd, ctx->dinv.p, ctx->x.p,
                                                    ctx->r.p, ctx->z.p, ctx->p.p, ctx->partials.p,
                                                    ctx->ticket.p, ctx->scal.p, tol * tol);
            RBG_CHECK_LAUNCH(ctx);
            if (fsai) {
                fsai_setup(ctx, st);
                fsai_lower_kernel<true><<<g_fs, kThreads, 0, st>>>(ctx->fs_gptr.p, ctx->fs_gcols.p, ctx->fs_gvals.p,
                                                                   m, ctx->r.p, ctx->fs_u.p, ctx->partials.p,
                                                                   ctx->ticket.p, ctx->scal.p);
                RBG_CHECK_LAUNCH(ctx);
                fsai_upper_kernel<true><<<g_fs, kThreads, 0, st>>>(ctx->fs_tptr.p, ctx->fs_tcols.p, ctx->fs_tvals.p,
                                                                   m, ctx->fs_u.p, ctx->p.p, ctx->scal.p);
                RBG_CHECK_LAUNCH(ctx);
                ctx->launches += 4;
            }
            for (;;) {
                RBG_CUDA(cudaMemcpyAsync(flags, ctx->scal.p + S_DONE, 3 * sizeof(double),
                                         cudaMemcpyDeviceToHost, st));
                RBG_CUDA(cudaStreamSynchronize(st));
                if (flags[0] != 0.0 || flags[1] != 0.0) break;
                RBG_CUDA(cudaGraphLaunch(exec, st));
                ctx->launches += (T || fsai ? 4 : 3) * batch;
            }
            if (flags[0] != 0.0 && flags[1] == 0.0) {
                solved = true;
                local.ridge_lambda = lambda;
                local.ridge_shift = shift;
                local.iterations = (int)flags[2];
                break;
            }
        }
    } catch (...) {
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
        throw;
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (!solved) {
        // solver.cpp:316-322 names the pivot the LLT stopped at: here the first
        // centre (by id) with a non-positive diagonal or a failed local
        // factorisation; running out of iterations is reported as such
        double piv_d = 0.0;
        RBG_CUDA(cudaMemcpyAsync(&piv_d, ctx->scal.p + S_PIV, sizeof(double), cudaMemcpyDeviceToHost, st));
        std::vector<double> dg(nt);
        RBG_CUDA(cudaMemcpyAsync(dg.data(), ctx->dinv.p, nt * sizeof(double), cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        uint64_t piv = nt;
        if (fsai) {  // solve rows are in Morton order
            std::vector<uint32_t> perm(m);
            RBG_CUDA(cudaMemcpy(perm.data(), ctx->bj_perm.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            for (uint64_t k = 0; k < m; ++k)
                if (!(dg[k] > 0.0 && std::isfinite(dg[k]))) piv = std::min<uint64_t>(piv, perm[k]);
            if (std::isfinite(piv_d)) piv = std::min<uint64_t>(piv, (uint64_t)piv_d);
        } else {
            piv = 0;
            while (piv < nt && dg[piv] > 0.0 && std::isfinite(dg[piv])) ++piv;
        }
        if (piv == nt && flags[1] == 2.0)
            throw Error(RBG_RUNTIME_ERROR, "normal system could not be solved even with ridge 1e-06: conjugate "
                                           "gradients did not converge in " + std::to_string(max_iter) +
                                           " iterations");
        if (piv == nt) piv = 0;
        throw Error(RBG_RUNTIME_ERROR,
                    "normal system is not positive definite even with ridge 1e-06; first "
                    "non-positive pivot at index " + std::to_string(piv));
    }
    if (T) {
        border_dot_kernel<<<g_vec, kThreads, 0, st>>>(bd, ctx->x.p, ctx->partials.p, ctx->ticket.p,
                                                      ctx->scal.p, 1);
        RBG_CHECK_LAUNCH(ctx);
    }
    residual_kernel<<<g_spmv, kThreads, 0, st>>>(s_fptr, s_fcols, ctx->vfull.p, m, bd, ctx->x.p,
                                                 b, ctx->partials.p, ctx->ticket.p, ctx->scal.p);
    RBG_CHECK_LAUNCH(ctx);
    if (fsai) {  // solution back to centre order (x stays in centre order for its readers)
        permute_kernel<false><<<g_vec, kThreads, 0, st>>>(ctx->bj_perm.p, m, ctx->x.p, ctx->q.p);
        RBG_CHECK_LAUNCH(ctx);
        RBG_CUDA(cudaMemcpyAsync(ctx->x.p, ctx->q.p, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    RBG_CUDA(cudaEventRecord(ctx->ev1, st));
    double rr_true = 0.0, bb = 0.0;
    RBG_CUDA(cudaMemcpyAsync(&rr_true, ctx->scal.p + S_PQ, sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaMemcpyAsync(&bb, ctx->scal.p + S_BB, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (c_out)
        RBG_CUDA(cudaMemcpyAsync(c_out, ctx->x.p, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    for (double& a : ctx->poly_sol) a = 0.0;
    if (T)
        RBG_CUDA(cudaMemcpyAsync(ctx->poly_sol, ctx->x.p + m, T * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    RBG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    local.solve_ms = ms;
    local.rel_residual = bb > 0.0 ? std::sqrt(rr_true / bb) : 0.0;
    if (diag) *diag = local;
}

}  // namespace rbg
