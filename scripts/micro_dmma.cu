// Microbenchmark: DMMA (mma.sync m8n8k4 f64) issue rate vs independent
// accumulator chains per warp and warps per SM, with register operands and
// with operands loaded from shared memory every step (the SYRK pattern);
// plus the latency of the exact phi(r) chain (dist2, correctly rounded sqrt,
// Wendland 3,1) per pair vs pairs in flight per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_dmma micro_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int C, bool LDS>
__global__ void k_dmma(double* sink, long long* cyc) {
    __shared__ double sm[16 * 36 * 8];
    for (int i = threadIdx.x; i < 16 * 36 * 8; i += blockDim.x) sm[i] = 1e-3 * (i % 7);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int frag = (lane >> 2) * 36 + (lane & 3);
    double acc[C][2];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = c;
    double a = 1e-3 + lane * 1e-9, b = 0.5;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (LDS) {
                const int base = ((it + c) & 7) * 36 * 8;
                a = sm[base + frag + ((it >> 3) & 3) * 4];
                b = sm[base + 8 * 36 + frag];
            }
            dmma(acc[c], a, b);
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) sink[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ double sqrt_rn_nonneg(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double t = fma(-hx * y, y, 0.5);
    y = fma(y, t, y);
    t = fma(-hx * y, y, 0.5);
    y = fma(y, t, y);
    double r = x * y;
    const double e = fma(-r, r, x);
    r = fma(e, 0.5 * y, r);
    return x > 0.0 ? r : 0.0;
}
__device__ __forceinline__ double phi31(double alpha, double r) {
    const double t = __dmul_rn(alpha, r);
    const double u = __dsub_rn(1.0, t);
    const double u2 = __dmul_rn(u, u);
    const double v = __dmul_rn(__dmul_rn(u2, u2), __dadd_rn(__dmul_rn(4.0, t), 1.0));
    return t < 1.0 ? v : 0.0;
}

// K independent pairs per iteration per thread; the next iteration's point
// depends on the previous results (so iterations serialise like a real loop
// whose trip work is the chain).
template <int K>
__global__ void k_phi(double* sink, long long* cyc) {
    double px[K], acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        px[k] = 0.1 + 1e-5 * (threadIdx.x + k);
        acc[k] = 0;
    }
    const double cy = 0.3, alpha = 10.0, r2 = 0.01;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double dx = __dsub_rn(px[k], 0.15), dy = __dsub_rn(0.31, cy);
            const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
            const double f = phi31(alpha, sqrt_rn_nonneg(d2));
            acc[k] += d2 < r2 ? f : 0.0;
            px[k] = __dadd_rn(px[k], acc[k] * 1e-30);
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += acc[k];
    if (s == 1.2345) sink[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
double run(K kern, int sms, int warps, long long* dcyc, double* sink) {
    kern<<<sms, warps * 32>>>(sink, dcyc);
    kern<<<sms, warps * 32>>>(sink, dcyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, dcyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < sms; ++i) s += (double)h[i];
    return s / sms;
}

template <int C, bool LDS>
void dmma_row(int sms, long long* dcyc, double* sink) {
    printf("DMMA %s C=%d :", LDS ? "lds" : "reg", C);
    for (int w : {1, 2, 4, 8, 16, 32}) {
        const double cyc = run(k_dmma<C, LDS>, sms, w, dcyc, sink);
        const double per_smsp = (double)ITERS * C * w / 4.0;  // DMMAs issued per SMSP (w >= 4)
        printf("  w%-2d %6.1f", w, cyc / (w >= 4 ? per_smsp : (double)ITERS * C));
    }
    printf("   [cycles per DMMA per SMSP; ideal 16]\n");
}

template <int K>
void phi_row(int sms, long long* dcyc, double* sink) {
    printf("phi K=%d      :", K);
    for (int w : {1, 2, 4, 8, 16, 32}) {
        const double cyc = run(k_phi<K>, sms, w, dcyc, sink);
        const double pairs = (double)(ITERS / 8) * K;  // per thread
        printf("  w%-2d %6.1f", w, cyc / pairs / (w >= 4 ? w / 4.0 : 1.0));
    }
    printf("   [cycles per warp-pair per SMSP; 1 thread-pair = ~26 fp64 ops -> ideal ~52]\n");
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* dcyc;
    double* sink;
    cudaMalloc(&dcyc, 1024 * sizeof(long long));
    cudaMalloc(&sink, 8);
    dmma_row<1, false>(sms, dcyc, sink);
    dmma_row<2, false>(sms, dcyc, sink);
    dmma_row<4, false>(sms, dcyc, sink);
    dmma_row<8, false>(sms, dcyc, sink);
    dmma_row<1, true>(sms, dcyc, sink);
    dmma_row<2, true>(sms, dcyc, sink);
    dmma_row<4, true>(sms, dcyc, sink);
    dmma_row<8, true>(sms, dcyc, sink);
    phi_row<1>(sms, dcyc, sink);
    phi_row<2>(sms, dcyc, sink);
    phi_row<4>(sms, dcyc, sink);
    phi_row<8>(sms, dcyc, sink);
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
