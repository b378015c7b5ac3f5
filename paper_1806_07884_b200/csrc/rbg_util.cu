// rbg_util.cu -- exclusive scans and a warp-per-segment bitonic sort used by
// the binning (counting sort) and symbolic (pattern) phases.
#include <algorithm>
#include <cstdint>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <cstring>
#include <condition_variable>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "rbg_internal.cuh"

namespace rbg {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanChunk = kScanThreads * kScanItems;

template <typename In>
__device__ __forceinline__ uint64_t load_val(const In* p, uint64_t i, uint64_t n) {
    return i < n ? (uint64_t)p[i] : 0ull;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ uint64_t block_exclusive(uint64_t v, uint64_t* total) {
    __shared__ uint64_t warp_sums[kScanThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t s = lane < kScanThreads / 32 ? warp_sums[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        if (lane < kScanThreads / 32) warp_sums[lane] = s;  // inclusive
    }
    __syncthreads();
    const uint64_t warp_off = warp == 0 ? 0ull : warp_sums[warp - 1];
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();
    return warp_off + incl - v;
}

template <typename In>
__global__ void scan_block_sums(const In* in, uint64_t n, uint64_t* sums) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanChunk + threadIdx.x * kScanItems;
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += load_val(in, base + k, n);
    uint64_t total;
    block_exclusive(s, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Single-block exclusive scan of the block sums (any length, chunked with carry).
__global__ void scan_sums_inplace(uint64_t* sums, uint64_t nb) {
    uint64_t carry = 0;
    for (uint64_t c0 = 0; c0 < nb; c0 += kScanChunk) {
        const uint64_t base = c0 + threadIdx.x * kScanItems;
        uint64_t v[kScanItems];
        uint64_t s = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            v[k] = base + k < nb ? sums[base + k] : 0ull;
            s += v[k];
        }
        uint64_t total;
        uint64_t ex = block_exclusive(s, &total) + carry;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (base + k < nb) sums[base + k] = ex;
            ex += v[k];
        }
        carry += total;
    }
}

template <typename In>
__global__ void scan_apply(const In* in, uint64_t n, const uint64_t* sums, uint64_t* out) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanChunk + threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = load_val(in, base + k, n);
        s += v[k];
    }
    uint64_t total;
    uint64_t ex = block_exclusive(s, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k <= n) out[base + k] = ex;  // out has n+1 entries: out[n] = total
        ex += v[k];
    }
}

template <typename In>
void exclusive_scan_impl(rbg_ctx* ctx, const In* in, uint64_t* out, uint64_t n) {
    // out[0..n] (n+1 entries); out[n] = sum.
    const uint64_t nb = (n + 1 + kScanChunk - 1) / kScanChunk;
    ctx->scan_tmp.reserve(nb);
    scan_block_sums<In><<<(unsigned)nb, kScanThreads, 0, ctx->stream>>>(in, n, ctx->scan_tmp.p);
    RBG_CHECK_LAUNCH(ctx);
    scan_sums_inplace<<<1, kScanThreads, 0, ctx->stream>>>(ctx->scan_tmp.p, nb);
    RBG_CHECK_LAUNCH(ctx);
    scan_apply<In><<<(unsigned)nb, kScanThreads, 0, ctx->stream>>>(in, n, ctx->scan_tmp.p, out);
    RBG_CHECK_LAUNCH(ctx);
}

// One warp per segment: load into shared memory padded with UINT32_MAX to a
// power of two, bitonic sort, write back.
__global__ void segsort_warp(uint32_t* keys, const uint64_t* seg_ptr, uint64_t n_segs, int p2) {
    extern __shared__ uint32_t sm[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint32_t* s = sm + (size_t)wib * p2;
    const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t seg = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; seg < n_segs;
         seg += warps_total) {
        const uint64_t b = seg_ptr[seg];
        const int len = (int)(seg_ptr[seg + 1] - b);
        if (len <= 1) continue;
        int n2 = 32;
        while (n2 < len) n2 <<= 1;
        for (int i = lane; i < n2; i += 32) s[i] = i < len ? keys[b + i] : 0xffffffffu;
        __syncwarp();
        for (int k = 2; k <= n2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < n2; i += 32) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const uint32_t a = s[i], c = s[ixj];
                        const bool up = (i & k) == 0;
                        if ((a > c) == up) {
                            s[i] = c;
                            s[ixj] = a;
                        }
                    }
                }
                __syncwarp();
            }
        for (int i = lane; i < len; i += 32) keys[b + i] = s[i];
        __syncwarp();
    }
}

}  // namespace

void exclusive_scan_u32_to_u64(rbg_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t n) {
    exclusive_scan_impl<uint32_t>(ctx, in, out, n);
}

void exclusive_scan_u64(rbg_ctx* ctx, const uint64_t* in, uint64_t* out, uint64_t n) {
    exclusive_scan_impl<uint64_t>(ctx, in, out, n);
}

void segmented_sort_u32(rbg_ctx* ctx, uint32_t* keys, const uint64_t* seg_ptr, uint64_t n_segs,
                        uint32_t max_len) {
    if (n_segs == 0 || max_len <= 1) return;
    int p2 = 32;
    while ((uint32_t)p2 < max_len) p2 <<= 1;
    if (p2 > 4096)
        throw Error(RBG_INVALID_ARGUMENT,
                    "support neighbourhood too large: a segment holds " + std::to_string(max_len) +
                        " centres (limit 4096); reduce the support radius");
    const int warps = p2 >= 2048 ? 2 : 4;
    const size_t smem = (size_t)warps * p2 * sizeof(uint32_t);
    const uint64_t blocks = (n_segs + warps - 1) / warps;
    segsort_warp<<<(unsigned)(blocks > 148u * 128u ? 148u * 128u : blocks), warps * 32, smem,
                   ctx->stream>>>(keys, seg_ptr, n_segs, p2);
    RBG_CHECK_LAUNCH(ctx);
}


// ------------------------------------------------------- device memory cache
namespace {

struct CachedBlock {
    int device;
    size_t bytes;
    void* p;
};
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;
thread_local int g_recycle_depth = 0;

void trim_cache(int device) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (auto it = g_cache.begin(); it != g_cache.end();) {
        if (it->device == device) {
            cudaFree(it->p);
            it = g_cache.erase(it);
        } else {
            ++it;
        }
    }
}

}  // namespace

RecycleScope::RecycleScope() { ++g_recycle_depth; }
RecycleScope::~RecycleScope() { --g_recycle_depth; }

namespace {
thread_local cudaStream_t g_scope_stream = nullptr;
thread_local bool g_scope_on = false;
}  // namespace
StreamScope::StreamScope(cudaStream_t st) : prev(g_scope_stream), had(g_scope_on) {
    g_scope_stream = st;
    g_scope_on = true;
}
StreamScope::~StreamScope() {
    g_scope_stream = prev;
    g_scope_on = had;
}

namespace {
// RBG_ALLOC_STATS=1: every cudaMalloc / cudaFree that misses the block cache is
// reported on stderr (diagnostics for stalls of the fresh-context fit).
void alloc_note(int kind, size_t bytes, std::chrono::steady_clock::time_point t0) {
    static const bool on = std::getenv("RBG_ALLOC_STATS") != nullptr;
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[rbg alloc] %s %.1f MB %.3f ms\n", kind ? "cudaFree" : "cudaMalloc", bytes / 1048576.0, ms);
}
}  // namespace

void* dev_alloc(size_t bytes, size_t* got) {
    int device = 0;
    RBG_CUDA(cudaGetDevice(&device));
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        size_t best = ~size_t{0};
        size_t bi = 0;
        for (size_t i = 0; i < g_cache.size(); ++i) {
            const CachedBlock& c = g_cache[i];
            if (c.device == device && c.bytes >= bytes && c.bytes <= 2 * bytes + (size_t{2} << 20) && c.bytes < best) {
                best = c.bytes;
                bi = i;
            }
        }
        if (best != ~size_t{0}) {
            void* p = g_cache[bi].p;
            *got = g_cache[bi].bytes;
            g_cache.erase(g_cache.begin() + (std::ptrdiff_t)bi);
            return p;
        }
    }
    void* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMalloc(&p, bytes);
    alloc_note(0, bytes, t0);
    if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
        cudaGetLastError();
        trim_cache(device);
        e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess)
        throw Error(RBG_CUDA_ERROR, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    *got = bytes;
    return p;
}

void dev_free(void* p, size_t bytes) {
    if (!p) return;
    const bool drained = g_recycle_depth > 0;
    if ((drained || g_scope_on) && bytes >= (size_t{64} << 10)) {
        int device = 0;
        // outside a context teardown the block may still be in use by kernels queued on the
        // calling context's stream (the only stream temporaries are used on): drain it first
        if (cudaGetDevice(&device) == cudaSuccess && (drained || cudaStreamSynchronize(g_scope_stream) == cudaSuccess)) {
            std::vector<CachedBlock> evict;
            {
                std::lock_guard<std::mutex> lk(g_cache_mu);
                g_cache.push_back({device, bytes, p});
                // bounded: beyond 64 GB (or 4096 blocks) the oldest blocks go back to the driver
                size_t total = 0;
                for (const CachedBlock& c : g_cache) total += c.bytes;
                while (!g_cache.empty() && (total > (size_t{64} << 30) || g_cache.size() > 4096)) {
                    total -= g_cache.front().bytes;
                    evict.push_back(g_cache.front());
                    g_cache.erase(g_cache.begin());
                }
            }
            for (const CachedBlock& c : evict) cudaFree(c.p);
            return;
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    cudaFree(p);
    alloc_note(1, bytes, t0);
}

// ------------------------------------------------------- staged host copies
// Pageable host memory cannot be DMA'd directly: chunks are copied into a
// process-wide ring of pinned buffers by a persistent pool of host threads
// while the copy engine drains the previous chunks.
namespace {

constexpr size_t kStageBytes = size_t{64} << 20;
constexpr int kStageBufs = 4;
constexpr size_t kDirectBytes = size_t{16} << 20;

class CopyPool {
  public:
    CopyPool() {
        // leave a quarter of the cores to the caller: the centre-side setup overlaps the upload
        const unsigned hw = std::thread::hardware_concurrency();
        nthreads_ = std::max(1u, std::min(12u, hw ? (hw * 3) / 4 : 1u));
        for (unsigned t = 1; t < nthreads_; ++t) workers_.emplace_back([this, t] { run(t); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    // memcpy split over every pool thread (the caller takes part 0)
    void copy(void* dst, const void* src, size_t bytes) {
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        bytes_ = bytes;
        pending_ = nthreads_ - 1;
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        part(0);
        lk.lock();
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void part(unsigned t) {
        const size_t per = ((bytes_ + nthreads_ - 1) / nthreads_ + 63) & ~size_t{63};
        const size_t off = std::min(bytes_, (size_t)t * per), len = std::min(per, bytes_ - off);
        if (len) stream_copy(dst_ + off, src_ + off, len);
    }
    // memcpy with non-temporal stores: the destination (a pinned staging buffer, or the
    // caller's result array) is not read again by this core, so write-allocating it in the
    // cache only adds a third memory stream to a copy that is bandwidth-bound
    static void stream_copy(char* dst, const char* src, size_t n) {
#if defined(__SSE2__)
        if (n >= 4096) {
            const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
            std::memcpy(dst, src, head);
            dst += head;
            src += head;
            n -= head;
            const size_t blocks = n / 64;
            for (size_t b = 0; b < blocks; ++b, dst += 64, src += 64) {
                const __m128i a0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src));
                const __m128i a1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 16));
                const __m128i a2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 32));
                const __m128i a3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 48));
                _mm_stream_si128(reinterpret_cast<__m128i*>(dst), a0);
                _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 16), a1);
                _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 32), a2);
                _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 48), a3);
            }
            _mm_sfence();
            n -= blocks * 64;
        }
#endif
        if (n) std::memcpy(dst, src, n);
    }
    void run(unsigned t) {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            lk.unlock();
            part(t);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    unsigned nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

struct Staging {
    std::mutex mu;  // one staged copy at a time per process
    void* buf[kStageBufs] = {};
    cudaEvent_t ev[kStageBufs] = {};
    CopyPool* pool = nullptr;
    void ensure() {
        if (!pool) pool = new CopyPool();  // never destroyed: threads outlive static teardown order
        for (int b = 0; b < kStageBufs; ++b) {
            if (!buf[b]) RBG_CUDA(cudaHostAlloc(&buf[b], kStageBytes, cudaHostAllocPortable));
            if (!ev[b]) RBG_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
        }
    }
};
Staging& staging() {
    static Staging* s = new Staging();
    return *s;
}

}  // namespace

bool page_locked(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void h2d(rbg_ctx* ctx, void* dst, const void* src, size_t bytes) { h2d_on(ctx->stream, dst, src, bytes); }

void h2d_on(cudaStream_t st, void* dst, const void* src, size_t bytes) {
    if (bytes < kDirectBytes || page_locked(src)) {
        RBG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> lk(S.mu);
    S.ensure();
    size_t off = 0;
    for (int i = 0; off < bytes; ++i) {
        const int b = i % kStageBufs;
        const size_t len = std::min(kStageBytes, bytes - off);
        RBG_CUDA(cudaEventSynchronize(S.ev[b]));  // the copy that last read this buffer is done
        S.pool->copy(S.buf[b], static_cast<const char*>(src) + off, len);
        RBG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, S.buf[b], len, cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaEventRecord(S.ev[b], st));
        off += len;
    }
    for (int b = 0; b < kStageBufs; ++b) RBG_CUDA(cudaEventSynchronize(S.ev[b]));
}

void d2h(rbg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    cudaStream_t st = ctx->stream;
    if (bytes < kDirectBytes || page_locked(dst)) {
        RBG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        return;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> lk(S.mu);
    S.ensure();
    const size_t n_chunks = (bytes + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t i) {
        const size_t off = i * kStageBytes, len = std::min(kStageBytes, bytes - off);
        RBG_CUDA(cudaMemcpyAsync(S.buf[i % kStageBufs], static_cast<const char*>(src) + off, len,
                                 cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaEventRecord(S.ev[i % kStageBufs], st));
    };
    for (size_t i = 0; i < std::min<size_t>(n_chunks, kStageBufs - 1); ++i) issue(i);
    for (size_t i = 0; i < n_chunks; ++i) {
        RBG_CUDA(cudaEventSynchronize(S.ev[i % kStageBufs]));
        if (i + kStageBufs - 1 < n_chunks) issue(i + kStageBufs - 1);  // later chunks land while this one drains
        const size_t off = i * kStageBytes, len = std::min(kStageBytes, bytes - off);
        S.pool->copy(static_cast<char*>(dst) + off, S.buf[i % kStageBufs], len);
    }
}

void release_staging(rbg_ctx*) {}  // the ring is process-wide

namespace {
__global__ void first_nonfinite_kernel(const double* __restrict__ p, uint64_t n, int dim,
                                       unsigned long long* __restrict__ first) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        bool ok = true;
        for (int d = 0; d < dim; ++d) ok = ok && isfinite(p[i * dim + d]);
        if (!ok) atomicMin(first, (unsigned long long)i);
    }
}
}  // namespace

uint64_t first_nonfinite(rbg_ctx* ctx, const double* d_pts, uint64_t n, int dim) {
    if (n == 0) return 0;
    cudaStream_t st = ctx->stream;
    unsigned long long* slot = ctx->counters.p + 1;  // [1] scratch
    const unsigned long long init = n;
    RBG_CUDA(cudaMemcpyAsync(slot, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    first_nonfinite_kernel<<<blocks_for(n, 256), 256, 0, st>>>(d_pts, n, dim, slot);
    RBG_CHECK_LAUNCH(ctx);
    unsigned long long first = n;
    RBG_CUDA(cudaMemcpyAsync(&first, slot, sizeof(first), cudaMemcpyDeviceToHost, st));
    RBG_CUDA(cudaStreamSynchronize(st));
    return first;
}

}  // namespace rbg
