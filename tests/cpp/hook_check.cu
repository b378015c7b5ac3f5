// The C++ layer's multi-GPU hook (rbfit_b200::AllReduce) on one GPU: two
// contexts each assemble half of the points; the hook of the first adds the
// second's device system into its own with a kernel enqueued on the stream
// the hook is given, without any synchronisation of its own.  The result read
// back by the host layer (rbg_get_system on the context's stream) must equal a
// single-pass assembly of all points.
//   hook_check <in.bin>   in.bin: u64 n, u64 m, f64 alpha, f64 xy[n*2], f64 h[n], f64 refs[m*2]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <vector>

#include "rbfit_gpu.hpp"
#include "rbg.h"

using namespace rbfit_b200;

__global__ void add_kernel(double* dst, const double* src, std::uint64_t n) {
    for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (std::uint64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream in(argv[1], std::ios::binary);
    std::uint64_t n = 0, m = 0;
    double alpha = 0;
    in.read(reinterpret_cast<char*>(&n), 8);
    in.read(reinterpret_cast<char*>(&m), 8);
    in.read(reinterpret_cast<char*>(&alpha), 8);
    PointCloud all, a, b;
    all.points.resize(n);
    all.values.resize(n);
    std::vector<Point2> refs(m);
    in.read(reinterpret_cast<char*>(all.points.data()), n * 16);
    in.read(reinterpret_cast<char*>(all.values.data()), n * 8);
    in.read(reinterpret_cast<char*>(refs.data()), m * 16);
    const std::size_t half = n / 2;
    a.points.assign(all.points.begin(), all.points.begin() + half);
    a.values.assign(all.values.begin(), all.values.begin() + half);
    b.points.assign(all.points.begin() + half, all.points.end());
    b.values.assign(all.values.begin() + half, all.values.end());
    const KernelSpec kernel(KernelFamily::wendland_3_1, alpha);

    std::fprintf(stderr, "read %llu points, %llu refs\n", (unsigned long long)n, (unsigned long long)m);
    Device dev_b(0);  // "rank 1": its partial system stays on the device
    build_normal_system(b, refs, kernel, false, nullptr, &dev_b);
    double* other = nullptr;
    std::uint64_t other_count = 0;
    if (rbg_system_device(dev_b.ctx(), &other, &other_count) != RBG_OK) return 3;

    std::fprintf(stderr, "rank-1 partial built\n");
    Device dev_a(0);
    cudaStream_t mine;
    cudaStreamCreateWithFlags(&mine, cudaStreamNonBlocking);
    dev_a.set_stream(mine);
    int calls = 0, bad_stream = 0;
    const AllReduce hook = [&](double* buf, std::uint64_t count, void* stream) {
        ++calls;
        if (stream != (void*)mine || count != other_count) ++bad_stream;
        add_kernel<<<148, 256, 0, (cudaStream_t)stream>>>(buf, other, count);  // no sync: ordered by the stream
    };
    const NormalSystem two = build_normal_system(a, refs, kernel, false, nullptr, &dev_a, hook);

    std::fprintf(stderr, "hooked build done\n");
    Device dev_c(0);
    const NormalSystem one = build_normal_system(all, refs, kernel, false, nullptr, &dev_c);
    double worst = 0.0, scale = 0.0;
    for (std::size_t i = 0; i < one.values.size(); ++i) {
        worst = std::max(worst, std::abs(one.values[i] - two.values[i]));
        scale = std::max(scale, std::abs(one.values[i]));
    }
    double wr = 0.0, sr = 0.0;
    for (std::size_t i = 0; i < m; ++i) {
        wr = std::max(wr, std::abs(one.rhs[i] - two.rhs[i]));
        sr = std::max(sr, std::abs(one.rhs[i]));
    }
    const bool same_empty = one.empty_support_refs == two.empty_support_refs;
    std::printf("hook calls=%d bad_stream=%d |dB|=%.3g |drhs|=%.3g empty_same=%d\n", calls, bad_stream,
                worst / scale, wr / sr, (int)same_empty);
    dev_a.set_stream(nullptr);  // the context must not outlive the caller's stream on it
    cudaStreamDestroy(mine);
    return (calls == 1 && bad_stream == 0 && worst / scale < 1e-12 && wr / sr < 1e-12 && same_empty) ? 0 : 1;
}
