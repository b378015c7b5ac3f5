// Microbenchmark: fp64 FMA pipe vs fp64 tensor-core MMA (mma.sync m8n8k4 f64)
// on sm_100a, alone and concurrently.  Informs whether the assembly SYRK
// should run on DMMA while phi evaluation uses the FMA pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_fp64 micro_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void k_dfma(double* sink, double seed) {
    double a[8];
    for (int c = 0; c < 8; ++c) a[c] = seed + c + threadIdx.x * 1e-9;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] = fma(a[c], 0.999999, 1e-12);
    double s = 0;
    for (int c = 0; c < 8; ++c) s += a[c];
    if (s == 1.2345) sink[0] = s;
}

__global__ void k_dmma(double* sink, double seed) {
    double acc[4][2];
    for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = seed + c;
    double a = 1e-3 + threadIdx.x * 1e-9, b = 0.5;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(acc[c], a, b);
    double s = 0;
    for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) sink[0] = s;
}

// even warps DMMA, odd warps DFMA
__global__ void k_mixed(double* sink, double seed) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if (warp & 1) {
        double a[8];
        for (int c = 0; c < 8; ++c) a[c] = seed + c + threadIdx.x * 1e-9;
        for (int it = 0; it < ITERS; ++it)
#pragma unroll
            for (int c = 0; c < 8; ++c) a[c] = fma(a[c], 0.999999, 1e-12);
        for (int c = 0; c < 8; ++c) s += a[c];
    } else {
        double acc[4][2];
        for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = seed + c;
        double a = 1e-3 + threadIdx.x * 1e-9, b = 0.5;
        for (int it = 0; it < ITERS; ++it)
#pragma unroll
            for (int c = 0; c < 4; ++c) dmma(acc[c], a, b);
        for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
    }
    if (s == 1.2345) sink[0] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, double* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, threads>>>(sink, 1.0);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(sink, 1.0 + r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    const double warps = (double)blocks * threads / 32;
    float t = timeit(k_dfma, blocks, threads, sink);
    double fl = 2.0 * 8 * ITERS * (double)blocks * threads;
    printf("DFMA only : %.3f ms  %.2f TFLOP/s\n", t, fl / t / 1e9);
    t = timeit(k_dmma, blocks, threads, sink);
    fl = 512.0 * 4 * ITERS * warps;
    printf("DMMA only : %.3f ms  %.2f TFLOP/s\n", t, fl / t / 1e9);
    t = timeit(k_mixed, blocks, threads, sink);
    fl = 0.5 * (2.0 * 8 * ITERS * (double)blocks * threads) + 0.5 * (512.0 * 4 * ITERS * warps);
    printf("mixed     : %.3f ms  %.2f TFLOP/s combined (half warps each)\n", t, fl / t / 1e9);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
