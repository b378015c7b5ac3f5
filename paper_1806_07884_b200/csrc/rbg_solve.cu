// rbg_solve.cu -- K4: SPD solve of the assembled normal equations.
//
// Replaces solve_weights (solver.cpp:289-330).  The reference factors the
// dense M x M matrix with Eigen LLT, which is infeasible beyond M ~ 5e4 (the
// dense b alone is 8 TB at M = 1e6).  Here: Jacobi-preconditioned conjugate
// gradients on the symmetric CSR matrix, hand-written fp64 kernels:
//   spmv_dot   q = (B + shift I) p, fused with the p.q reduction
//   update     x += a p, r -= a q, z = D^-1 r, fused with r.z and r.r
//   direction  p = z + b p
// Scalars (alpha, beta, convergence) live on the device; reductions finish in
// the last block to arrive (fixed-order, so runs are deterministic) and the
// iteration loop is replayed from a CUDA graph in batches, with one host
// read of the convergence flags per batch.  Stopping rule:
// ||r||_2 <= tol ||b||_2.  The reference's ridge ladder (solver.cpp:296-315)
// is kept: lambda x trace/side is added on breakdown / non-convergence.
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


// ------------------------------------------------------ block-Jacobi
// Preconditioner M = blockdiag(B_bb + shift I) over blocks of kBJ centres that
// are consecutive in Morton order (spatially compact), each inverted exactly
// (Cholesky + triangular inverse in shared memory).  Local oscillatory modes
// -- what makes A^T A ill-conditioned for compactly supported kernels -- are
// solved inside the blocks, which cuts the CG iteration count several-fold
// against point Jacobi for one extra kBJ^2 matvec per iteration.  A
// non-positive pivot in a block flags the attempt as failed, so the
// reference's ridge ladder (solver.cpp:296-315) moves to the next lambda.
#ifndef RBG_BJ
#define RBG_BJ 32
#endif
constexpr int kBJ = RBG_BJ;      // block size (a multiple of 32): one warp per block in the apply
constexpr int kRPL = kBJ / 32;   // block rows per lane in the apply
static_assert(kBJ % 32 == 0, "block-Jacobi block size must be a multiple of 32");

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

// One CTA (kBJ threads, thread t = block row t) per diagonal block: gather the
// dense block from the upper CSR, Cholesky, invert; the inverse is stored
// transposed (= itself) so the apply's loads are coalesced.
__global__ void __launch_bounds__(kBJ) bj_setup_kernel(const uint64_t* __restrict__ uptr,
                                                       const uint32_t* __restrict__ ucols,
                                                       const double* __restrict__ uvals, uint64_t m,
                                                       const uint32_t* __restrict__ perm,
                                                       const uint32_t* __restrict__ pos, double* scal,
                                                       double* __restrict__ inv) {
    extern __shared__ double bj_sm[];  // D and Li, kBJ x (kBJ + 1) each
    double (*D)[kBJ + 1] = reinterpret_cast<double (*)[kBJ + 1]>(bj_sm);
    double (*Li)[kBJ + 1] = reinterpret_cast<double (*)[kBJ + 1]>(bj_sm + kBJ * (kBJ + 1));
    __shared__ int bad;
    const uint64_t b = blockIdx.x;
    const int t = threadIdx.x;
    const double shift = scal[S_SHIFT];
    for (int j = 0; j < kBJ; ++j) D[t][j] = 0.0;
    if (t == 0) bad = 0;
    __syncthreads();
    const uint64_t k = b * kBJ + t;
    if (k < m) {
        const uint32_t i = perm[k];
        for (uint64_t e = uptr[i]; e < uptr[i + 1]; ++e) {
            const uint32_t c = ucols[e];
            const uint32_t pc = pos[c];
            if (pc / kBJ != b) continue;
            const int lj = (int)(pc % kBJ);
            const double v = uvals[e];
            if (c == i) {
                D[t][t] = v + shift;
            } else {  // row i's upper part holds (i, c), c > i: only this thread writes both
                D[t][lj] = v;
                D[lj][t] = v;
            }
        }
    } else {
        D[t][t] = 1.0;  // padding rows of the last block
    }
    __syncthreads();
    for (int kk = 0; kk < kBJ; ++kk) {  // lower Cholesky in place, thread t owns row t
        if (t == kk) {
            const double d = D[kk][kk];
            if (!(d > 0.0) || !isfinite(d)) bad = 1;
            D[kk][kk] = sqrt(d > 0.0 ? d : 1.0);
        }
        __syncthreads();
        if (t > kk) D[t][kk] /= D[kk][kk];
        __syncthreads();
        if (t > kk)
            for (int j = kk + 1; j <= t; ++j) D[t][j] -= D[t][kk] * D[j][kk];
        __syncthreads();
    }
    // column t of L^-1
    for (int i = 0; i < t; ++i) Li[i][t] = 0.0;
    Li[t][t] = 1.0 / D[t][t];
    for (int i = t + 1; i < kBJ; ++i) {
        double acc = 0.0;
        for (int q = t; q < i; ++q) acc += D[i][q] * Li[q][t];
        Li[i][t] = -acc / D[i][i];
    }
    __syncthreads();
    // (B_bb)^-1 = L^-T L^-1, row t
    double* out = inv + b * (uint64_t)(kBJ * kBJ);
    for (int j = 0; j < kBJ; ++j) {
        double acc = 0.0;
        for (int q = max(t, j); q < kBJ; ++q) acc += Li[q][t] * Li[q][j];
        out[j * kBJ + t] = acc;
    }
    if (t == 0 && bad) scal[S_FAIL] = 1.0;
}

// z = M^-1 r over the blocks (one warp per block); with INIT also p = z and
// rz = r.z (start of an attempt), else the CG update first: x += a p,
// r -= a q, then z, rz and rr (same epilogue as update_kernel).
template <bool INIT>
__global__ void __launch_bounds__(kThreads) bj_update_kernel(uint64_t m, uint64_t nblk, const uint32_t* __restrict__ perm,
                                                             const double* __restrict__ inv,
                                                             const double* __restrict__ q, double* __restrict__ x,
                                                             double* __restrict__ r, double* __restrict__ z,
                                                             double* __restrict__ p, double* partials,
                                                             unsigned* ticket, double* scal) {
    if (scal[S_DONE] != 0.0 || scal[S_FAIL] != 0.0) return;
    __shared__ double rs[kThreads / 32][kBJ];
    const double a = INIT ? 0.0 : scal[S_ALPHA];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double v[2] = {0.0, 0.0};
    for (uint64_t b = blockIdx.x * (uint64_t)(kThreads / 32) + w; b < nblk; b += (uint64_t)gridDim.x * (kThreads / 32)) {
        uint32_t i[kRPL];
        double ri[kRPL];
#pragma unroll
        for (int u = 0; u < kRPL; ++u) {
            const uint64_t k = b * kBJ + u * 32 + lane;
            i[u] = 0;
            ri[u] = 0.0;
            if (k < m) {
                i[u] = perm ? perm[k] : (uint32_t)k;  // null: the solve runs in Morton order
                if (INIT) {
                    ri[u] = r[i[u]];
                } else {
                    x[i[u]] += a * p[i[u]];
                    ri[u] = r[i[u]] - a * q[i[u]];
                    r[i[u]] = ri[u];
                }
            }
            rs[w][u * 32 + lane] = ri[u];
        }
        __syncwarp();
        const double* Bi = inv + b * (uint64_t)(kBJ * kBJ);
        double zi[kRPL];
#pragma unroll
        for (int u = 0; u < kRPL; ++u) zi[u] = 0.0;
#pragma unroll 8
        for (int j = 0; j < kBJ; ++j) {
            const double rj = rs[w][j];
#pragma unroll
            for (int u = 0; u < kRPL; ++u) zi[u] = fma(__ldg(Bi + j * kBJ + u * 32 + lane), rj, zi[u]);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kRPL; ++u) {
            const uint64_t k = b * kBJ + u * 32 + lane;
            if (k < m) {
                z[i[u]] = zi[u];
                if (INIT) p[i[u]] = zi[u];
                v[0] += ri[u] * zi[u];
                v[1] += ri[u] * ri[u];
            }
        }
    }
    double out[2];
    if (last_block_sum<2>(v, partials, ticket, out) && threadIdx.x == 0) {
        if (INIT) {
            scal[S_RZ] = out[0];
            return;
        }
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

constexpr int kKeyShift = 12;  // row offsets < 4096 (the segmented-sort limit)

// Full CSR in Morton order: new row k = centre perm[k], columns renumbered by
// pos (unsorted within the row: the SpMV does not need it), f2u carried along.
__global__ void perm_len_kernel(const uint64_t* __restrict__ fptr, const uint64_t* __restrict__ uptr,
                                const uint32_t* __restrict__ perm, uint64_t m, uint32_t* __restrict__ len,
                                uint64_t* __restrict__ puptr) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = perm[k];
        len[k] = (uint32_t)(fptr[i + 1] - fptr[i]);
        puptr[k] = uptr[i];
    }
}

// SORTED: pass 1 writes keys (new column << 12 | source offset in the row) for a
// segmented sort, pass 2 (perm_unpack_kernel) turns the sorted keys into
// columns ascending in Morton position -- a warp's gathers of p then fall on
// few L2 sectors.
template <bool SORTED>
__global__ void perm_fill_kernel(const uint64_t* __restrict__ fptr, const uint32_t* __restrict__ fcols,
                                 const uint64_t* __restrict__ f2u, const uint32_t* __restrict__ perm,
                                 const uint32_t* __restrict__ pos, uint64_t m, const uint64_t* __restrict__ pfptr,
                                 uint32_t* __restrict__ pfcols, uint64_t* __restrict__ pf2u) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t k = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); k < m; k += warps) {
        const uint32_t i = perm[k];
        const uint64_t s0 = fptr[i], n = fptr[i + 1] - s0, d0 = pfptr[k];
        for (uint64_t e = lane; e < n; e += 32) {
            if (SORTED) {
                pfcols[d0 + e] = (pos[fcols[s0 + e]] << kKeyShift) | (uint32_t)e;
            } else {
                pfcols[d0 + e] = pos[fcols[s0 + e]];
                pf2u[d0 + e] = f2u[s0 + e];
            }
        }
    }
}

__global__ void perm_unpack_kernel(const uint64_t* __restrict__ fptr, const uint64_t* __restrict__ f2u,
                                   const uint32_t* __restrict__ perm, uint64_t m, const uint64_t* __restrict__ pfptr,
                                   uint32_t* __restrict__ pfcols, uint64_t* __restrict__ pf2u) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t k = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5); k < m; k += warps) {
        const uint64_t s0 = fptr[perm[k]], d0 = pfptr[k], n = pfptr[k + 1] - d0;
        for (uint64_t e = lane; e < n; e += 32) {
            const uint32_t key = pfcols[d0 + e];
            pfcols[d0 + e] = key >> kKeyShift;
            pf2u[d0 + e] = f2u[s0 + (key & ((1u << kKeyShift) - 1u))];
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

constexpr int kBJSetupSmem = 2 * kBJ * (kBJ + 1) * (int)sizeof(double);

// Grid of a grid-stride kernel: at most one full wave of resident CTAs (a
// partial second wave leaves SMs idle at the tail of every launch).
template <typename K>
unsigned resident_grid(rbg_ctx* ctx, K kern, unsigned needed) {
    int per_sm = 0, sms = 0;
    RBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0));
    RBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    return std::max(1u, std::min(needed, (unsigned)std::max(1, per_sm * sms)));
}

// Morton permutation of the centres and its inverse (once per centre set).
void bj_build_order(rbg_ctx* ctx) {
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
    RBG_CUDA(cudaStreamSynchronize(st));  // temporaries are released at scope end
    RBG_CUDA(cudaFuncSetAttribute(bj_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBJSetupSmem));
    ctx->bj_nblk = (m + kBJ - 1) / kBJ;
    ctx->bj_inv.reserve(ctx->bj_nblk * kBJ * kBJ);
    {
        DevBuf<uint32_t> len;
        len.reserve(m + 1);
        ctx->pfptr.reserve(m + 1);
        ctx->puptr.reserve(m);
        ctx->pfcols.reserve(ctx->nnz_full);
        ctx->pf2u.reserve(ctx->nnz_full);
        perm_len_kernel<<<blocks_for(m, 256), 256, 0, st>>>(ctx->fptr.p, ctx->uptr.p, ctx->bj_perm.p, m, len.p,
                                                           ctx->puptr.p);
        RBG_CHECK_LAUNCH(ctx);
        exclusive_scan_u32_to_u64(ctx, len.p, ctx->pfptr.p, m);
        const unsigned gf = blocks_for(m, 8, 148u * 16u);
        const bool sorted = m <= (1ull << (32 - kKeyShift)) && ctx->max_full_row <= (1u << kKeyShift) &&
                            !std::getenv("RBG_PERM_UNSORTED");
        if (sorted) {
            perm_fill_kernel<true><<<gf, 256, 0, st>>>(ctx->fptr.p, ctx->fcols.p, ctx->f2u.p, ctx->bj_perm.p,
                                                       ctx->bj_pos.p, m, ctx->pfptr.p, ctx->pfcols.p, ctx->pf2u.p);
            RBG_CHECK_LAUNCH(ctx);
            segmented_sort_u32(ctx, ctx->pfcols.p, ctx->pfptr.p, m, ctx->max_full_row);
            perm_unpack_kernel<<<gf, 256, 0, st>>>(ctx->fptr.p, ctx->f2u.p, ctx->bj_perm.p, m, ctx->pfptr.p,
                                                   ctx->pfcols.p, ctx->pf2u.p);
        } else {
            perm_fill_kernel<false><<<gf, 256, 0, st>>>(ctx->fptr.p, ctx->fcols.p, ctx->f2u.p, ctx->bj_perm.p,
                                                        ctx->bj_pos.p, m, ctx->pfptr.p, ctx->pfcols.p, ctx->pf2u.p);
        }
        RBG_CHECK_LAUNCH(ctx);
        RBG_CUDA(cudaStreamSynchronize(st));
    }
    ctx->bj_built = true;
}

}  // namespace

void solve_system(rbg_ctx* ctx, const rbg_solve_options* opts, double* c_out, rbg_solve_diag* diag) {
    // the reference's method (LLT + ridge ladder) wherever the band is affordable
    // (rbg_band.cu); RBG_SOLVER=pcg / band forces a path (tests, A/B)
    static const int forced = [] {
        const char* e = std::getenv("RBG_SOLVER");
        return !e ? 0 : std::string(e) == "pcg" ? 1 : std::string(e) == "band" ? 2 : 0;
    }();
    if (ctx->pterms() == 0 && forced != 1 && (band_plan(ctx) || forced == 2)) {
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
    const unsigned g_max = std::max(g_vec, g_spmv);
    ctx->partials.reserve(4ull * g_max);
    ctx->scal.reserve(S_COUNT);
    ctx->ticket.reserve(1);
    RBG_CUDA(cudaMemsetAsync(ctx->ticket.p, 0, sizeof(unsigned), st));
    RBG_CUDA(cudaMemsetAsync(ctx->scal.p, 0, S_COUNT * sizeof(double), st));

    // preconditioner: block Jacobi unless RBG_PREC=jacobi or the system is bordered;
    // the block-Jacobi solve runs in the Morton order of its blocks
    static const bool bj_env = [] {
        const char* e = std::getenv("RBG_PREC");
        return !(e && std::string(e) == "jacobi");
    }();
    const bool use_bj = bj_env && T == 0;
    if (use_bj && !ctx->bj_built) bj_build_order(ctx);
    const uint64_t* s_fptr = use_bj ? ctx->pfptr.p : ctx->fptr.p;
    const uint32_t* s_fcols = use_bj ? ctx->pfcols.p : ctx->fcols.p;
    const uint64_t* s_uptr = use_bj ? ctx->puptr.p : ctx->uptr.p;  // diagonal of each solve row

    RBG_CUDA(cudaEventRecord(ctx->ev0, st));
    gather_full_kernel<<<blocks_for(nnz, kThreads), kThreads, 0, st>>>(use_bj ? ctx->pf2u.p : ctx->f2u.p, uvals,
                                                                        nnz, ctx->vfull.p);
    RBG_CHECK_LAUNCH(ctx);
    if (use_bj) {  // right-hand side to Morton order
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

    const unsigned g_bj =
        use_bj ? resident_grid(ctx, bj_update_kernel<false>, blocks_for(ctx->bj_nblk, kThreads / 32, ~0u)) : 0u;
    if (use_bj) ctx->partials.reserve(std::max<uint64_t>(4ull * g_max, 4ull * g_bj));

    // one batch of iterations as a graph (kernels read their scalars on device)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    RBG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < kBatch; ++it) {
        if (T)
            border_dot_kernel<<<g_vec, kThreads, 0, st>>>(bd, ctx->p.p, ctx->partials.p, ctx->ticket.p,
                                                          ctx->scal.p, 0);
        spmv_dot_kernel<<<g_spmv, kThreads, 0, st>>>(s_fptr, s_fcols, ctx->vfull.p, m, bd,
                                                     ctx->p.p, ctx->q.p, ctx->partials.p,
                                                     ctx->ticket.p, ctx->scal.p);
        if (use_bj)
            bj_update_kernel<false><<<g_bj, kThreads, 0, st>>>(m, ctx->bj_nblk, nullptr, ctx->bj_inv.p,
                                                               ctx->q.p, ctx->x.p, ctx->r.p, ctx->z.p, ctx->p.p,
                                                               ctx->partials.p, ctx->ticket.p, ctx->scal.p);
        else
            update_kernel<<<g_vec, kThreads, 0, st>>>(nt, ctx->p.p, ctx->q.p, ctx->dinv.p, ctx->x.p,
                                                      ctx->r.p, ctx->z.p, ctx->partials.p,
                                                      ctx->ticket.p, ctx->scal.p);
        direction_kernel<<<g_vec, kThreads, 0, st>>>(nt, ctx->z.p, ctx->p.p, ctx->scal.p);
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
            if (use_bj) {
                bj_setup_kernel<<<(unsigned)ctx->bj_nblk, kBJ, kBJSetupSmem, st>>>(ctx->uptr.p, ctx->ucols.p, uvals, m,
                                                                        ctx->bj_perm.p, ctx->bj_pos.p, ctx->scal.p,
                                                                        ctx->bj_inv.p);
                RBG_CHECK_LAUNCH(ctx);
                bj_update_kernel<true><<<g_bj, kThreads, 0, st>>>(m, ctx->bj_nblk, nullptr, ctx->bj_inv.p,
                                                                  ctx->q.p, ctx->x.p, ctx->r.p, ctx->z.p, ctx->p.p,
                                                                  ctx->partials.p, ctx->ticket.p, ctx->scal.p);
                RBG_CHECK_LAUNCH(ctx);
            }
            for (;;) {
                RBG_CUDA(cudaMemcpyAsync(flags, ctx->scal.p + S_DONE, 3 * sizeof(double),
                                         cudaMemcpyDeviceToHost, st));
                RBG_CUDA(cudaStreamSynchronize(st));
                if (flags[0] != 0.0 || flags[1] != 0.0) break;
                RBG_CUDA(cudaGraphLaunch(exec, st));
                ctx->launches += (T ? 4 : 3) * kBatch;
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
        // first non-positive diagonal (the pivot an LLT meets first on an
        // empty-support column), else the last row reached.
        std::vector<double> dg(nt);
        RBG_CUDA(cudaMemcpyAsync(dg.data(), ctx->dinv.p, nt * sizeof(double), cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        uint64_t piv = 0;
        if (use_bj) {  // solve rows are in Morton order: the first bad centre id
            std::vector<uint32_t> perm(m);
            RBG_CUDA(cudaMemcpy(perm.data(), ctx->bj_perm.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            piv = nt;
            for (uint64_t k = 0; k < m; ++k)
                if (!(dg[k] > 0.0 && std::isfinite(dg[k]))) piv = std::min<uint64_t>(piv, perm[k]);
        } else {
            while (piv < nt && dg[piv] > 0.0 && std::isfinite(dg[piv])) ++piv;
        }
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
    if (use_bj) {  // solution back to centre order (x stays in centre order for its readers)
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
