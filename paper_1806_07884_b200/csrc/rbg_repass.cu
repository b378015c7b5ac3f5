// rbg_repass.cu -- the orthogonal least-squares re-pass (least_squares_repass,
// solver.cpp:345-397) for small reference sets.
//
// When the plain factorisation of the normal equations fails, fit()
// (solver.cpp:439-464) makes one more pass over the data and solves the
// least-squares problem min ||[A P] w - h|| at cond(A) instead of cond(A)^2:
// fixed 4096-row chunks of the augmented design [A P | h] are pushed through
// an incremental Householder QR (the running aug x aug factor R stacked on the
// chunk, factored, its top rows kept), and w comes from the triangular solve
// R w = R[:, width].  A non-finite w (rank-deficient design) means "keep the
// ridge solution".
//
// B200 version: the stack S = [R; chunk] lives column-major in HBM (it fits
// L2 for every M this path accepts).  Each chunk's rows are formed densely on
// the device with the reference's exact arithmetic (every entry is the
// reference's A entry: strict d2 < r2, phi_of_r of the correctly rounded
// sqrt), then one kernel per column j applies the Householder reflector of
// column j to the columns k > j (one CTA per column; each CTA recomputes the
// column-j norm, so no extra launch or grid barrier is needed).  The chunk
// layout (consecutive 4096-point chunks in input order) is the reference's, so
// the result does not depend on anything but the data, like the reference.
#include <cmath>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

constexpr int kRepassThreads = 256;
constexpr uint64_t kChunkRows = 4096;  // solver.cpp:359-360

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) sh[32] = s;
    }
    __syncthreads();
    return sh[32];
}

// Chunk rows of the augmented design [A P | h] (solver.cpp:365-381): row r,
// column j < m: phi_j(p) (0 outside the strict support), then x, y, (z), 1,
// then h.  Written below the running factor (rows aug .. aug + rows - 1).
template <int DIM>
__global__ void chunk_rows_kernel(const double* __restrict__ pts, const double* __restrict__ h, uint64_t rows,
                                  const double* __restrict__ centres, uint64_t m, int T, int family, double alpha,
                                  double r2, double* __restrict__ S, uint64_t ld, uint64_t aug) {
    const uint64_t width = m + (uint64_t)T;
    const uint64_t total = rows * (width + 1);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e % rows, j = e / rows;  // column-major: consecutive threads, consecutive rows
        const double* p = pts + r * DIM;
        double v;
        if (j < m) {
            const double* c = centres + j * DIM;
            const double d2 = dist2_of<DIM>(p[0], p[1], DIM == 3 ? p[2] : 0.0, c[0], c[1], DIM == 3 ? c[2] : 0.0);
            v = d2 < r2 ? phi_of_r(family, alpha, __dsqrt_rn(d2)) : 0.0;  // kdtree.cpp:74, kernel.hpp:42-62
        } else if (j < width) {
            const uint64_t t = j - m;
            v = (int)t < DIM ? p[t] : 1.0;  // P = [x, y, (z), 1]
        } else {
            v = h[r];
        }
        S[j * ld + aug + r] = v;
    }
}

// Householder step j on the stack (column-major, leading dimension ld): the
// reflector of x = [S(j,j); S(aug.., j)] (the factor rows below j are zero in
// column j) applied to column k = j + 1 + blockIdx.x.  alpha_out[j] receives
// the new diagonal (written by block 0 only; S(j,j) itself is read by every
// block, so it is not overwritten here).
__global__ void householder_kernel(double* __restrict__ S, uint64_t ld, uint64_t aug, uint64_t rows, uint64_t j,
                                   double* __restrict__ alpha_out) {
    __shared__ double sh[33];
    const double* xj = S + j * ld;
    const uint64_t k = j + 1 + blockIdx.x;
    double ss = 0.0;
    for (uint64_t i = threadIdx.x; i < rows; i += blockDim.x) ss += xj[aug + i] * xj[aug + i];
    const double ynorm2 = block_sum(ss, sh);
    const double x0 = xj[j];
    if (ynorm2 == 0.0) {  // nothing below the diagonal: H = I
        if (blockIdx.x == 0 && threadIdx.x == 0) alpha_out[j] = x0;
        return;
    }
    const double nrm = sqrt(x0 * x0 + ynorm2);
    const double a = x0 >= 0.0 ? -nrm : nrm;  // u0 = x0 - a has no cancellation
    const double u0 = x0 - a;
    const double utu = u0 * u0 + ynorm2;
    if (blockIdx.x == 0 && threadIdx.x == 0) alpha_out[j] = a;
    if (k >= aug) return;
    double* col = S + k * ld;
    double dot = 0.0;
    for (uint64_t i = threadIdx.x; i < rows; i += blockDim.x) dot += xj[aug + i] * col[aug + i];
    const double s = block_sum(dot, sh) + u0 * col[j];
    const double f = 2.0 * s / utu;
    for (uint64_t i = threadIdx.x; i < rows; i += blockDim.x) col[aug + i] -= f * xj[aug + i];
    if (threadIdx.x == 0) col[j] -= f * u0;
}

__global__ void set_diag_kernel(double* __restrict__ S, uint64_t ld, uint64_t aug, const double* __restrict__ a) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < aug; j += (uint64_t)gridDim.x * blockDim.x)
        S[j * ld + j] = a[j];
}

// R w = z (upper triangular, width x width, column-major in S; z = column
// `width`): back substitution, one CTA; w[i] non-finite marks a rank-deficient
// design (solver.cpp:390-393).
__global__ void back_substitute_kernel(const double* __restrict__ S, uint64_t ld, uint64_t width,
                                       double* __restrict__ w) {
    __shared__ double sh[33];
    const double* z = S + width * ld;
    for (uint64_t ii = width; ii-- > 0;) {
        double s = 0.0;
        for (uint64_t k = ii + 1 + threadIdx.x; k < width; k += blockDim.x) s += S[k * ld + ii] * w[k];
        const double tot = block_sum(s, sh);
        if (threadIdx.x == 0) w[ii] = (z[ii] - tot) / S[ii * ld + ii];
        __syncthreads();
    }
}

}  // namespace

uint64_t repass_max_refs() { return 4096; }

bool least_squares_repass(rbg_ctx* ctx, const double* d_pts, const double* d_h, uint64_t n, double* w_out) {
    cudaStream_t st = ctx->stream;
    const int dim = ctx->dim;
    const uint64_t m = ctx->m;
    const int T = ctx->pterms();
    const uint64_t width = m + (uint64_t)T, aug = width + 1;
    const uint64_t chunk = n < kChunkRows ? n : kChunkRows;
    const uint64_t ld = aug + chunk;
    DevBuf<double> S, alpha, w;
    S.reserve(ld * aug);
    alpha.reserve(aug);
    w.reserve(width);
    RBG_CUDA(cudaMemsetAsync(S.p, 0, ld * aug * sizeof(double), st));
    for (uint64_t base = 0; base < n; base += chunk) {
        const uint64_t rows = n - base < chunk ? n - base : chunk;
        if (rows < chunk)  // a shorter last chunk: clear the stale rows below it
            RBG_CUDA(cudaMemset2DAsync(S.p + aug + rows, ld * sizeof(double), 0, (chunk - rows) * sizeof(double),
                                       aug, st));
        const unsigned g = blocks_for(rows * aug, kRepassThreads);
        if (dim == 2)
            chunk_rows_kernel<2><<<g, kRepassThreads, 0, st>>>(d_pts + base * 2, d_h + base, rows, ctx->centres.p, m,
                                                               T, ctx->family, ctx->alpha, ctx->r2, S.p, ld, aug);
        else
            chunk_rows_kernel<3><<<g, kRepassThreads, 0, st>>>(d_pts + base * 3, d_h + base, rows, ctx->centres.p, m,
                                                               T, ctx->family, ctx->alpha, ctx->r2, S.p, ld, aug);
        RBG_CHECK_LAUNCH(ctx);
        for (uint64_t j = 0; j < aug; ++j) {
            const unsigned blocks = (unsigned)(aug - j - 1 > 0 ? aug - j - 1 : 1);
            householder_kernel<<<blocks, kRepassThreads, 0, st>>>(S.p, ld, aug, chunk, j, alpha.p);
            RBG_CHECK_LAUNCH(ctx);
        }
        set_diag_kernel<<<blocks_for(aug, 256), 256, 0, st>>>(S.p, ld, aug, alpha.p);
        RBG_CHECK_LAUNCH(ctx);
    }
    back_substitute_kernel<<<1, 1024, 0, st>>>(S.p, ld, width, w.p);
    RBG_CHECK_LAUNCH(ctx);
    std::vector<double> hw(width);
    RBG_CUDA(cudaMemcpyAsync(hw.data(), w.p, width * sizeof(double), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    for (double v : hw)
        if (!std::isfinite(v)) return false;  // solver.cpp:392: keep the ridge solution
    std::copy(hw.begin(), hw.end(), w_out);
    return true;
}

}  // namespace rbg
