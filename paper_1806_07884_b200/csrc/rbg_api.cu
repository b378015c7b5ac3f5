// rbg_api.cu -- the C ABI (include/rbg.h): validation with the reference's
// messages, host<->device staging, status codes.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <cstdlib>
#include <exception>
#include <atomic>
#include <chrono>
#include <thread>

#include "rbg_internal.cuh"

using rbg::Error;

namespace {

template <typename F>
rbg_status guarded(rbg_ctx* ctx, F&& f) {
    if (!ctx) return RBG_INVALID_ARGUMENT;
    try {
        ctx->err.clear();
        rbg::StreamScope scope(ctx->stream);  // temporaries released inside are recycled after draining this stream
        f();
        return RBG_OK;
    } catch (const Error& e) {
        ctx->err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failed";
        return RBG_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return RBG_RUNTIME_ERROR;
    }
}

void bind(rbg_ctx* ctx) { RBG_CUDA(cudaSetDevice(ctx->device)); }

void require_centres(const rbg_ctx* ctx) {
    if (!ctx->have_centres)
        throw Error(RBG_NOT_READY, "no reference points set (call rbg_set_centres first)");
}
// The symbolic pattern (K2) is built at the first call that needs it, after
// the tile grid (rbg::ensure_grid); the system buffer is sized for it.
void require_pattern(rbg_ctx* ctx) {
    require_centres(ctx);
    RBG_CUDA(cudaSetDevice(ctx->device));
    rbg::ensure_grid(ctx);
    if (!ctx->have_pattern) {
        RBG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        rbg::setup_pattern(ctx);
        RBG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        RBG_CUDA(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        RBG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->setup_ms += ms;
    }
    ctx->sys.reserve(ctx->sys_count());
}

void require_system(const rbg_ctx* ctx) {
    require_centres(ctx);
    if (!ctx->have_system)
        throw Error(RBG_NOT_READY, "no assembled system (call rbg_assemble first)");
}

void check_points_finite(const double* p, uint64_t n, int dim, const char* what) {
    for (uint64_t i = 0; i < n; ++i)
        for (int d = 0; d < dim; ++d)
            if (!std::isfinite(p[i * dim + d]))
                throw Error(RBG_INVALID_ARGUMENT,
                            std::string(what) + std::to_string(i));
}

void check_misses(rbg_ctx* ctx) {
    unsigned long long c[8] = {};
    RBG_CUDA(cudaMemcpyAsync(c, ctx->counters.p, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    RBG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (c[7]) {  // the dense-centre fallback path keeps 512 hits per point
        RBG_CUDA(cudaMemsetAsync(ctx->counters.p + 7, 0, sizeof(unsigned long long), ctx->stream));
        ctx->have_system = false;
        throw Error(RBG_INVALID_ARGUMENT, std::to_string(c[7]) + " points lie in the support of more than 512 "
                                          "centres of a dense centre cluster; reduce the support radius");
    }
    if (c[0])
        throw Error(RBG_RUNTIME_ERROR, "internal: " + std::to_string(c[0]) +
                                           " assembly updates fell outside the symbolic pattern");
}

// Host copy of the device kernel (kernel.hpp:42-62); x86-64 baseline has no
// FMA, so this is the reference's arithmetic.
double phi_host(int family, double alpha, double r) {
    const double t = alpha * r;
    if (!(t < 1.0)) return 0.0;
    const double u = 1.0 - t;
    switch (family) {
        case RBG_WENDLAND_3_0: return u * u;
        case RBG_WENDLAND_3_1: {
            const double u2 = u * u;
            return u2 * u2 * (4.0 * t + 1.0);
        }
        case RBG_WENDLAND_3_3: {
            const double u2 = u * u, u4 = u2 * u2;
            return u4 * u4 * (((32.0 * t + 25.0) * t + 8.0) * t + 1.0);
        }
        default: {
            const double u2 = u * u, u4 = u2 * u2, u6 = u4 * u2;
            return u6 * ((35.0 * t + 18.0) * t + 3.0);
        }
    }
}

}  // namespace

extern "C" {

rbg_status rbg_create(int device, rbg_ctx** out) {
    if (!out) return RBG_INVALID_ARGUMENT;
    *out = nullptr;
    auto* ctx = new rbg_ctx();
    ctx->device = device;
    const rbg_status s = guarded(ctx, [&] {
        int n = 0;
        RBG_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n)
            throw Error(RBG_INVALID_ARGUMENT, "CUDA device " + std::to_string(device) +
                                                  " does not exist (" + std::to_string(n) + " visible)");
        bind(ctx);
        RBG_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
        RBG_CUDA(cudaEventCreate(&ctx->ev0));
        RBG_CUDA(cudaEventCreate(&ctx->ev1));
        for (auto& e : ctx->ev_asm) RBG_CUDA(cudaEventCreate(&e));
        // [0] pattern misses, [1] scratch (first_nonfinite), [2..7] diagnostics
        ctx->counters.reserve(8);
        RBG_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 8 * sizeof(unsigned long long), ctx->stream));
    });
    if (s != RBG_OK) {
        // keep the message reachable through a static buffer
        static thread_local std::string last;
        last = ctx->err;
        delete ctx;
        return s;
    }
    *out = ctx;
    return RBG_OK;
}

rbg_status rbg_destroy(rbg_ctx* ctx) {
    if (!ctx) return RBG_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    rbg::RecycleScope recycle;  // the streams are drained: the work buffers go to the device cache
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (auto& e : ctx->ev_asm)
        if (e) cudaEventDestroy(e);
    rbg::release_staging(ctx);
    for (auto& e : ctx->chunk_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return RBG_OK;
}

const char* rbg_last_error(const rbg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

rbg_status rbg_set_stream(rbg_ctx* ctx, void* stream) {
    return guarded(ctx, [&] { ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream; });
}

rbg_status rbg_get_stream(rbg_ctx* ctx, void** stream) {
    return guarded(ctx, [&] {
        if (!stream) throw Error(RBG_INVALID_ARGUMENT, "null stream pointer");
        *stream = (void*)ctx->stream;
    });
}

rbg_status rbg_synchronize(rbg_ctx* ctx) {
    return guarded(ctx, [&] {
        bind(ctx);
        RBG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

uint64_t rbg_launch_count(const rbg_ctx* ctx) { return ctx ? ctx->launches : 0; }

rbg_status rbg_set_centres(rbg_ctx* ctx, int dim, const double* centres, uint64_t m, int family,
                           double alpha) {
    return guarded(ctx, [&] {
        if (dim != 2 && dim != 3) throw Error(RBG_INVALID_ARGUMENT, "dimension must be 2 or 3");
        if (family < 0 || family > 3) throw Error(RBG_INVALID_ARGUMENT, "unknown kernel family");
        if (!(alpha > 0.0) || !std::isfinite(alpha))  // kernel.cpp:35-38
            throw Error(RBG_INVALID_ARGUMENT, "kernel shape parameter must be positive and finite");
        if (m == 0 || !centres)  // coo.cpp:168
            throw Error(RBG_INVALID_ARGUMENT, "assemble_submatrix: empty reference block");
        if (m > 0xffffffffull)  // coo.cpp:13-16
            throw Error(RBG_INVALID_ARGUMENT, "reference count exceeds 32-bit triplet index range");
        check_points_finite(centres, m, dim, "non-finite reference point at index ");  // coo.cpp:172-175
        bind(ctx);
        // the same centre set and kernel again (e.g. evaluate_model after fit): everything
        // derived from the centres -- grid, pattern, assembly layout, solver order -- stays
        if (ctx->have_centres && ctx->dim == dim && ctx->m == m && ctx->family == family &&
            ctx->alpha == alpha && ctx->host_centres.size() == m * (uint64_t)dim &&
            std::memcmp(ctx->host_centres.data(), centres, m * dim * sizeof(double)) == 0)
            return;
        ctx->host_centres.assign(centres, centres + m * (uint64_t)dim);
        ctx->have_centres = false;
        ctx->have_system = false;
        ctx->dim = dim;
        ctx->m = m;
        ctx->family = family;
        ctx->alpha = alpha;
        ctx->radius = 1.0 / alpha;                // kernel.hpp:37
        ctx->r2 = ctx->radius * ctx->radius;      // kdtree.cpp:64
        ctx->centres.reserve(m * dim);
        RBG_CUDA(cudaMemcpyAsync(ctx->centres.p, centres, m * dim * sizeof(double),
                                 cudaMemcpyHostToDevice, ctx->stream));
        // everything derived from the centres is built at the first call that needs
        // it (rbg::ensure_grid / require_pattern / the layout at the first assembly),
        // so a host-array assembly can overlap it with the upload of the points
        ctx->have_grid = false;
        ctx->have_pattern = false;
        ctx->bj_built = false;
        ctx->fs_built = false;
        ctx->lay = rbg::AsmLayout();
        ctx->setup_ms = 0.0;
        ctx->have_centres = true;
    });
}

rbg_status rbg_get_pattern_info(rbg_ctx* ctx, rbg_pattern_info* info) {
    return guarded(ctx, [&] {
        require_pattern(ctx);
        if (!info) throw Error(RBG_INVALID_ARGUMENT, "null info");
        info->m = ctx->m;
        info->nnz_upper = ctx->nnz_upper;
        info->nnz_full = ctx->nnz_full;
        info->n_tiles = ctx->grid.count;
        info->n_fallback = ctx->lay.n_fallback;
        info->max_tile_centres = ctx->max_tile_centres;
        info->tile_edge = ctx->grid.edge;
        info->setup_ms = ctx->setup_ms;
    });
}

rbg_status rbg_get_pattern(rbg_ctx* ctx, uint64_t* row_ptr, uint32_t* cols) {
    return guarded(ctx, [&] {
        require_pattern(ctx);
        bind(ctx);
        if (row_ptr)
            RBG_CUDA(cudaMemcpyAsync(row_ptr, ctx->uptr.p, (ctx->m + 1) * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        if (cols)
            RBG_CUDA(cudaMemcpyAsync(cols, ctx->ucols.p, ctx->nnz_upper * sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        RBG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

rbg_status rbg_assemble(rbg_ctx* ctx, const double* points, const double* h, uint64_t n,
                        int accumulate, int validate) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        if (n > 0 && (!points || !h)) throw Error(RBG_INVALID_ARGUMENT, "null point or value array");
        bind(ctx);
        const int dim = ctx->dim;
        // Large inputs are uploaded in chunks on a copy stream (pinned: direct
        // copies; pageable: through the staging ring), each chunk assembled
        // (accumulating) as soon as it has landed, so the upload overlaps the
        // binning and assembly of the chunks before it.
        static const int chunks_env = [] {
            const char* e = std::getenv("RBG_H2D_CHUNKS");
            return e ? std::max(1, std::min(8, std::atoi(e))) : 0;
        }();
        int K = 1;
        // measured on B200 over PCIe: 3 chunks pay from ~1e7 points (cfg5 e2e +12 %),
        // below that the extra per-chunk binning and flushes cost more than the overlap
        if (n >= 1000000 && rbg::page_locked(points) && rbg::page_locked(h))
            K = chunks_env ? chunks_env : (n >= 10000000 ? 3 : 1);
        if (n > 0) {
            ctx->in_pts.reserve(n * dim);
            ctx->in_h.reserve(n);
        }
        if (K == 1) {
            if (n > 0 && n * dim * sizeof(double) >= (size_t{64} << 20) && !rbg::page_locked(points)) {
                // large pageable inputs: the staged upload (host copy threads + the copy
                // engine, on the copy stream) overlaps the centre-side setup of this context
                // -- tile grid, pattern, assembly layout and the solver's structures, on the
                // compute stream -- and, from 5e7 points, the assembly of the first half while
                // the second half is still on its way
                if (!ctx->copy_stream) RBG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
                if (!ctx->chunk_ev[0]) RBG_CUDA(cudaEventCreateWithFlags(&ctx->chunk_ev[0], cudaEventDisableTiming));
                RBG_CUDA(cudaEventRecord(ctx->chunk_ev[0], ctx->stream));  // earlier readers of in_pts / in_h
                RBG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[0], 0));
                // measured at cfg5 (fresh-context fit): 1 chunk 231 ms, 2 chunks 218, 3 chunks 233, 4 chunks 250
                const int KP = chunks_env ? chunks_env : (n >= 50000000 ? 2 : 1);
                std::vector<uint64_t> off(KP + 1);
                for (int c = 0; c <= KP; ++c) off[c] = n * (uint64_t)c / (uint64_t)KP;
                std::atomic<int> landed{0};
                std::exception_ptr up_err;
                std::thread up([&] {
                    try {
                        RBG_CUDA(cudaSetDevice(ctx->device));
                        for (int c = 0; c < KP; ++c) {  // h2d_on returns once the chunk is on the device
                            const uint64_t a = off[c], len = off[c + 1] - a;
                            rbg::h2d_on(ctx->copy_stream, ctx->in_pts.p + a * dim, points + a * dim,
                                        len * dim * sizeof(double));
                            rbg::h2d_on(ctx->copy_stream, ctx->in_h.p + a, h + a, len * sizeof(double));
                            landed.store(c + 1, std::memory_order_release);
                        }
                    } catch (...) {
                        up_err = std::current_exception();
                        landed.store(KP, std::memory_order_release);
                    }
                });
                try {
                    require_pattern(ctx);
                    rbg::ensure_layout(ctx, n);
                    rbg::prepare_solver(ctx);
                    for (int c = 0; c < KP; ++c) {
                        while (landed.load(std::memory_order_acquire) <= c)
                            std::this_thread::sleep_for(std::chrono::microseconds(100));
                        if (up_err) break;
                        const uint64_t a = off[c], len = off[c + 1] - a;
                        if (validate) {
                            const uint64_t bad = rbg::first_nonfinite(ctx, ctx->in_pts.p + a * dim, len, dim);
                            if (bad < len) {
                                ctx->have_system = false;
                                throw Error(RBG_INVALID_ARGUMENT,
                                            "non-finite coordinate at point index " + std::to_string(a + bad));
                            }
                        }
                        rbg::assemble_points(ctx, ctx->in_pts.p + a * dim, ctx->in_h.p + a, len,
                                             accumulate != 0 || c > 0);
                    }
                } catch (...) {
                    up.join();
                    throw;
                }
                up.join();
                if (up_err) std::rethrow_exception(up_err);
                return;
            } else if (n > 0) {
                require_pattern(ctx);
                rbg::h2d(ctx, ctx->in_pts.p, points, n * dim * sizeof(double));
                rbg::h2d(ctx, ctx->in_h.p, h, n * sizeof(double));
                if (validate) {  // kdtree.cpp:14-17, checked on the device copy (first offending index)
                    const uint64_t bad = rbg::first_nonfinite(ctx, ctx->in_pts.p, n, dim);
                    if (bad < n)
                        throw Error(RBG_INVALID_ARGUMENT, "non-finite coordinate at point index " + std::to_string(bad));
                }
            }
            require_pattern(ctx);  // (no-op when built above)
            if (n > 0) rbg::ensure_layout(ctx, n);
            rbg::assemble_points(ctx, ctx->in_pts.p, ctx->in_h.p, n, accumulate != 0);
            return;
        }
        require_pattern(ctx);
        rbg::ensure_layout(ctx, n);  // tile sizes follow the whole batch's density
        if (!ctx->copy_stream) RBG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int c = 0; c < K; ++c)
            if (!ctx->chunk_ev[c]) RBG_CUDA(cudaEventCreateWithFlags(&ctx->chunk_ev[c], cudaEventDisableTiming));
        // the copy stream must not overwrite inputs a previous call is still reading
        RBG_CUDA(cudaEventRecord(ctx->chunk_ev[0], ctx->stream));
        RBG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[0], 0));
        std::vector<uint64_t> off(K + 1);
        for (int c = 0; c <= K; ++c) off[c] = n * (uint64_t)c / (uint64_t)K;
        for (int c = 0; c < K; ++c) {
            const uint64_t a = off[c], len = off[c + 1] - a;
            RBG_CUDA(cudaMemcpyAsync(ctx->in_pts.p + a * dim, points + a * dim, len * dim * sizeof(double),
                                     cudaMemcpyHostToDevice, ctx->copy_stream));
            RBG_CUDA(cudaMemcpyAsync(ctx->in_h.p + a, h + a, len * sizeof(double), cudaMemcpyHostToDevice,
                                     ctx->copy_stream));
            RBG_CUDA(cudaEventRecord(ctx->chunk_ev[c], ctx->copy_stream));
        }
        for (int c = 0; c < K; ++c) {
            const uint64_t a = off[c], len = off[c + 1] - a;
            RBG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->chunk_ev[c], 0));
            if (validate) {
                const uint64_t bad = rbg::first_nonfinite(ctx, ctx->in_pts.p + a * dim, len, dim);
                if (bad < len) {
                    RBG_CUDA(cudaStreamSynchronize(ctx->copy_stream));
                    ctx->have_system = false;
                    throw Error(RBG_INVALID_ARGUMENT, "non-finite coordinate at point index " + std::to_string(a + bad));
                }
            }
            rbg::assemble_points(ctx, ctx->in_pts.p + a * dim, ctx->in_h.p + a, len, accumulate != 0 || c > 0);
        }
    });
}

rbg_status rbg_assemble_device(rbg_ctx* ctx, const double* d_points, const double* d_h, uint64_t n,
                               int accumulate) {
    return guarded(ctx, [&] {
        require_pattern(ctx);
        bind(ctx);
        if (n > 0) rbg::ensure_layout(ctx, n);
        rbg::assemble_points(ctx, d_points, d_h, n, accumulate != 0);
    });
}

rbg_status rbg_system_device(rbg_ctx* ctx, double** d_buffer, uint64_t* count) {
    return guarded(ctx, [&] {
        require_pattern(ctx);
        if (d_buffer) *d_buffer = ctx->sys.p;
        if (count) *count = ctx->sys_count();
    });
}

rbg_status rbg_get_system(rbg_ctx* ctx, double* values, double* rhs, double* hits,
                          uint64_t* design_nnz) {
    return guarded(ctx, [&] {
        require_system(ctx);
        bind(ctx);
        check_misses(ctx);
        cudaStream_t st = ctx->stream;
        const uint64_t m = ctx->m;
        if (values) rbg::d2h(ctx, values, ctx->sys.p, ctx->nnz_upper * sizeof(double));
        if (rhs)
            RBG_CUDA(cudaMemcpyAsync(rhs, ctx->sys.p + ctx->nnz_upper, m * sizeof(double),
                                     cudaMemcpyDeviceToHost, st));
        std::vector<double> hbuf;
        double* hp = hits;
        if (!hp && design_nnz) {
            hbuf.resize(m);
            hp = hbuf.data();
        }
        if (hp)
            RBG_CUDA(cudaMemcpyAsync(hp, ctx->sys.p + ctx->nnz_upper + m, m * sizeof(double),
                                     cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        if (design_nnz) {
            uint64_t s = 0;
            for (uint64_t i = 0; i < m; ++i) s += (uint64_t)hp[i];
            *design_nnz = s;
        }
    });
}

rbg_status rbg_set_system(rbg_ctx* ctx, const double* values, const double* rhs, const double* hits) {
    return guarded(ctx, [&] {
        require_pattern(ctx);
        if (!values || !rhs) throw Error(RBG_INVALID_ARGUMENT, "null system array");
        bind(ctx);
        cudaStream_t st = ctx->stream;
        RBG_CUDA(cudaMemcpyAsync(ctx->sys.p, values, ctx->nnz_upper * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaMemcpyAsync(ctx->sys.p + ctx->nnz_upper, rhs, ctx->m * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
        if (hits)
            RBG_CUDA(cudaMemcpyAsync(ctx->sys.p + ctx->nnz_upper + ctx->m, hits,
                                     ctx->m * sizeof(double), cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaStreamSynchronize(st));
        ctx->have_system = true;
    });
}

rbg_status rbg_solve(rbg_ctx* ctx, const rbg_solve_options* opts, double* c_out, rbg_solve_diag* diag) {
    return guarded(ctx, [&] {
        require_system(ctx);
        bind(ctx);
        check_misses(ctx);
        rbg::solve_system(ctx, opts, c_out, diag);
    });
}

uint64_t rbg_repass_max_unknowns(void) { return rbg::repass_max_refs(); }

rbg_status rbg_least_squares_repass(rbg_ctx* ctx, const double* points, const double* h, uint64_t n,
                                    double* w_out, int* ok) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        if (n == 0 || !points || !h || !w_out || !ok) throw Error(RBG_INVALID_ARGUMENT, "null or empty input");
        const uint64_t unknowns = ctx->m + (uint64_t)ctx->pterms();
        if (unknowns > rbg::repass_max_refs())
            throw Error(RBG_INVALID_ARGUMENT, "least-squares re-pass: " + std::to_string(unknowns) +
                                                  " unknowns exceed the GPU path's limit of " +
                                                  std::to_string(rbg::repass_max_refs()));
        bind(ctx);
        const int dim = ctx->dim;
        ctx->in_pts.reserve(n * dim);
        ctx->in_h.reserve(n);
        rbg::h2d(ctx, ctx->in_pts.p, points, n * dim * sizeof(double));
        rbg::h2d(ctx, ctx->in_h.p, h, n * sizeof(double));
        if (const uint64_t bad = rbg::first_nonfinite(ctx, ctx->in_pts.p, n, dim); bad < n)
            throw Error(RBG_INVALID_ARGUMENT, "non-finite coordinate at point index " + std::to_string(bad));
        *ok = rbg::least_squares_repass(ctx, ctx->in_pts.p, ctx->in_h.p, n, w_out) ? 1 : 0;
    });
}

rbg_status rbg_evaluate_device(rbg_ctx* ctx, const double* d_c, const double* d_q, uint64_t nq,
                               double* d_f) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        bind(ctx);
        rbg::ensure_grid(ctx);
        rbg::evaluate_points(ctx, d_c, d_q, nq, d_f);
    });
}

rbg_status rbg_evaluate(rbg_ctx* ctx, const double* c, const double* q, uint64_t nq, double* f) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        if (!c || (nq > 0 && (!q || !f))) throw Error(RBG_INVALID_ARGUMENT, "null array");
        bind(ctx);
        rbg::ensure_grid(ctx);
        cudaStream_t st = ctx->stream;
        ctx->ev_c.reserve(ctx->m);
        RBG_CUDA(cudaMemcpyAsync(ctx->ev_c.p, c, ctx->m * sizeof(double), cudaMemcpyHostToDevice, st));
        if (nq == 0) return;
        ctx->ev_q.reserve(nq * ctx->dim);
        ctx->ev_f.reserve(nq);
        rbg::h2d(ctx, ctx->ev_q.p, q, nq * ctx->dim * sizeof(double));
        if (const uint64_t bad = rbg::first_nonfinite(ctx, ctx->ev_q.p, nq, ctx->dim); bad < nq)  // model.cpp:60
            throw Error(RBG_INVALID_ARGUMENT, "evaluate_model: non-finite query point at index " + std::to_string(bad));
        rbg::evaluate_points(ctx, ctx->ev_c.p, ctx->ev_q.p, nq, ctx->ev_f.p);
        rbg::d2h(ctx, f, ctx->ev_f.p, nq * sizeof(double));
    });
}

rbg_status rbg_error_report(rbg_ctx* ctx, const double* c, const double* points, const double* h,
                            uint64_t n, rbg_error_stats* out, double* signed_errors) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        if (n == 0) throw Error(RBG_INVALID_ARGUMENT, "error_report: empty cloud");  // model.cpp:198
        if (!c || !points || !h || !out) throw Error(RBG_INVALID_ARGUMENT, "null array");
        bind(ctx);
        rbg::ensure_grid(ctx);
        cudaStream_t st = ctx->stream;
        ctx->ev_c.reserve(ctx->m);
        ctx->ev_q.reserve(n * ctx->dim);
        ctx->ev_f.reserve(n);
        ctx->ev_h.reserve(n);
        RBG_CUDA(cudaMemcpyAsync(ctx->ev_c.p, c, ctx->m * sizeof(double), cudaMemcpyHostToDevice, st));
        rbg::h2d(ctx, ctx->ev_q.p, points, n * ctx->dim * sizeof(double));
        if (const uint64_t bad = rbg::first_nonfinite(ctx, ctx->ev_q.p, n, ctx->dim); bad < n)  // model.cpp:60
            throw Error(RBG_INVALID_ARGUMENT, "evaluate_model: non-finite query point at index " + std::to_string(bad));
        rbg::h2d(ctx, ctx->ev_h.p, h, n * sizeof(double));
        rbg::evaluate_points(ctx, ctx->ev_c.p, ctx->ev_q.p, n, ctx->ev_f.p);
        rbg::error_stats(ctx, ctx->ev_f.p, ctx->ev_h.p, n, out);
        if (signed_errors) {
            rbg::d2h(ctx, signed_errors, ctx->ev_f.p, n * sizeof(double));
            for (uint64_t i = 0; i < n; ++i) signed_errors[i] = signed_errors[i] - h[i];  // model.cpp:208
        }
    });
}

rbg_status rbg_set_poly(rbg_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        if (ctx->poly_on != (enable != 0)) ctx->have_system = false;  // the system layout changes
        ctx->poly_on = enable != 0;
    });
}

rbg_status rbg_get_border(rbg_ctx* ctx, double* atp, double* ptp, double* pth) {
    return guarded(ctx, [&] {
        require_system(ctx);
        const int T = ctx->pterms();
        if (T == 0) throw Error(RBG_INVALID_ARGUMENT, "no polynomial border (call rbg_set_poly first)");
        bind(ctx);
        cudaStream_t st = ctx->stream;
        const double* E = ctx->sys.p + ctx->border_off();
        if (atp)
            RBG_CUDA(cudaMemcpyAsync(atp, E, (uint64_t)T * ctx->m * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (ptp)
            RBG_CUDA(cudaMemcpyAsync(ptp, E + (uint64_t)T * ctx->m, T * T * sizeof(double),
                                     cudaMemcpyDeviceToHost, st));
        if (pth)
            RBG_CUDA(cudaMemcpyAsync(pth, E + (uint64_t)T * ctx->m + T * T, T * sizeof(double),
                                     cudaMemcpyDeviceToHost, st));
        RBG_CUDA(cudaStreamSynchronize(st));
    });
}

rbg_status rbg_set_border(rbg_ctx* ctx, const double* atp, const double* ptp, const double* pth) {
    return guarded(ctx, [&] {
        require_pattern(ctx);
        const int T = ctx->pterms();
        if (T == 0) throw Error(RBG_INVALID_ARGUMENT, "no polynomial border (call rbg_set_poly first)");
        if (!atp || !ptp || !pth) throw Error(RBG_INVALID_ARGUMENT, "null border array");
        bind(ctx);
        cudaStream_t st = ctx->stream;
        double* E = ctx->sys.p + ctx->border_off();
        RBG_CUDA(cudaMemcpyAsync(E, atp, (uint64_t)T * ctx->m * sizeof(double), cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaMemcpyAsync(E + (uint64_t)T * ctx->m, ptp, T * T * sizeof(double), cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaMemcpyAsync(E + (uint64_t)T * ctx->m + T * T, pth, T * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
        RBG_CUDA(cudaStreamSynchronize(st));
    });
}

rbg_status rbg_get_poly_solution(rbg_ctx* ctx, double* a) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        if (!a) throw Error(RBG_INVALID_ARGUMENT, "null array");
        for (int t = 0; t < ctx->pterms(); ++t) a[t] = ctx->poly_sol[t];
    });
}

rbg_status rbg_set_model_poly(rbg_ctx* ctx, const double* a) {
    return guarded(ctx, [&] {
        require_centres(ctx);
        ctx->model_poly = a != nullptr;
        for (int t = 0; t < 4; ++t) ctx->model_a[t] = (a && t <= ctx->dim) ? a[t] : 0.0;
    });
}

rbg_status rbg_partition_slabs(int dim, const double* points, uint64_t n, int axis, int n_slabs,
                               double* bounds, uint32_t* slab_of) {
    if ((dim != 2 && dim != 3) || axis < 0 || axis >= dim || n_slabs < 1 || !bounds ||
        (n > 0 && !points))
        return RBG_INVALID_ARGUMENT;
    try {
        std::vector<double> v(n);
        for (uint64_t i = 0; i < n; ++i) v[i] = points[i * dim + axis];
        bounds[0] = -std::numeric_limits<double>::infinity();
        bounds[n_slabs] = std::numeric_limits<double>::infinity();
        for (int k = 1; k < n_slabs; ++k) {
            const uint64_t at = (uint64_t)((__int128)k * n / n_slabs);
            if (at >= n) {
                bounds[k] = std::numeric_limits<double>::infinity();
                continue;
            }
            std::nth_element(v.begin(), v.begin() + at, v.end());
            bounds[k] = v[at];
        }
        for (int k = 1; k < n_slabs; ++k)  // monotone (nth_element is per call)
            if (bounds[k] < bounds[k - 1]) bounds[k] = bounds[k - 1];
        if (slab_of)
            for (uint64_t i = 0; i < n; ++i) {
                const double x = points[i * dim + axis];
                const int s = (int)(std::upper_bound(bounds + 1, bounds + n_slabs, x) - (bounds + 1));
                slab_of[i] = (uint32_t)s;
            }
        return RBG_OK;
    } catch (...) {
        return RBG_RUNTIME_ERROR;
    }
}

rbg_status rbg_kernel_value(int family, double alpha, double r, double* out) {
    if (family < 0 || family > 3 || !(alpha > 0.0) || !std::isfinite(alpha) || !out)
        return RBG_INVALID_ARGUMENT;
    if (!(r >= 0.0) || !std::isfinite(r)) return RBG_DOMAIN_ERROR;  // kernel.hpp:43-44
    *out = phi_host(family, alpha, r);
    return RBG_OK;
}

}  // extern "C"
