/*
 * rbg.h -- C ABI of the B200-native CS-RBF normal-equation engine (librbg.so).
 *
 * Plain pointers and sizes only; no C++ or torch types.  Host pointers unless a
 * name says "device".  Every call returns an rbg_status; on failure
 * rbg_last_error(ctx) holds the message.  A context is NOT thread-safe; use
 * one per host thread / GPU.  All work of a context runs on one CUDA stream
 * (rbg_set_stream), in issue order.
 *
 * Each entry point replaces one reference (rbfit, /root/reference/proj/core)
 * interface; the citation is given per function.  The C++ host layer in
 * paper_1806_07884_b200/csrc/rbfit_gpu.hpp re-exposes these with the
 * reference's C++ signatures and exception types.
 */
#ifndef RBG_H
#define RBG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rbg_ctx rbg_ctx;

/* Status codes map 1:1 onto the reference's exception classes. */
typedef enum {
    RBG_OK = 0,
    RBG_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    RBG_RUNTIME_ERROR = 2,    /* std::runtime_error (e.g. unsolvable system) */
    RBG_DOMAIN_ERROR = 3,     /* std::domain_error */
    RBG_CUDA_ERROR = 4,       /* device failure (no reference analogue) */
    RBG_NOT_READY = 5         /* call order violated (e.g. assemble before set_centres) */
} rbg_status;

/* Kernel families: 0..2 follow rbfit::KernelFamily (kernel.hpp:21-25);
 * 3 is the wendland-3-2 extension BASELINE config 3 needs (phi(0)=3). */
typedef enum {
    RBG_WENDLAND_3_0 = 0,
    RBG_WENDLAND_3_1 = 1,
    RBG_WENDLAND_3_3 = 2,
    RBG_WENDLAND_3_2 = 3
} rbg_kernel;

/* ---- context ------------------------------------------------------------ */
/* New context bound to CUDA device `device`, with its own stream. */
rbg_status rbg_create(int device, rbg_ctx** out);
rbg_status rbg_destroy(rbg_ctx* ctx);
const char* rbg_last_error(const rbg_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores
 * the context's own stream. */
rbg_status rbg_set_stream(rbg_ctx* ctx, void* cuda_stream);
rbg_status rbg_synchronize(rbg_ctx* ctx);
/* The CUDA stream (cudaStream_t) all work of the context is issued on: an
 * external all-reduce of rbg_system_device must be enqueued on it (or be
 * ordered with it) -- e.g. ncclAllReduce(..., stream) -- so that it runs after
 * the assembly and before rbg_get_system / rbg_solve. */
rbg_status rbg_get_stream(rbg_ctx* ctx, void** cuda_stream);
/* Number of kernel launches issued by this context so far (bench evidence). */
uint64_t rbg_launch_count(const rbg_ctx* ctx);

/* ---- centres: binning + symbolic pattern ---------------------------------
 * Replaces the per-reference radius queries of assemble_submatrix
 * (coo.cpp:166-192) and the implicit dense pattern of NormalSystem::b
 * (solver.hpp:61-69, solver.cpp:151-156).  centres: m points, AoS, `dim`
 * (2 or 3) doubles each.  Validation as KernelSpec (kernel.cpp:35-38) and
 * assemble_submatrix (coo.cpp:168-175).  Builds the uniform tile grid, the
 * per-tile centre lists (evaluation) and the upper CSR pattern {(i,j): i<=j,
 * |c_i-c_j|^2 < (2/alpha)^2}; the assembly layout (super/sub-tiles, slot
 * maps) follows at the first assembly.  Calling it again with an identical
 * centre set, family and alpha keeps all of it (no device work). */
rbg_status rbg_set_centres(rbg_ctx* ctx, int dim, const double* centres, uint64_t m,
                           int kernel_family, double alpha);

typedef struct {
    uint64_t m;            /* centres */
    uint64_t nnz_upper;    /* pattern entries, upper triangle incl. diagonal */
    uint64_t nnz_full;     /* symmetric pattern entries */
    uint64_t n_tiles;      /* tile grid size */
    uint64_t n_fallback;   /* super-tiles on the slow path (0 before the first assembly) */
    uint32_t max_tile_centres;
    double tile_edge;
    double setup_ms;       /* device time of rbg_set_centres */
} rbg_pattern_info;
rbg_status rbg_get_pattern_info(rbg_ctx* ctx, rbg_pattern_info* info);
/* Copies the upper CSR pattern: row_ptr[m+1], cols[nnz_upper]. */
rbg_status rbg_get_pattern(rbg_ctx* ctx, uint64_t* row_ptr, uint32_t* cols);

/* ---- numeric assembly -----------------------------------------------------
 * Replaces build_normal_system's assembly + gram + rhs (solver.cpp:131-236:
 * assemble_submatrix, transpose_matvec coo.cpp:75-82, gram_self
 * coo.cpp:134-151).  Adds the contribution of n points (AoS, dim doubles
 * each) with values h to the device system [values | rhs | hits]; the
 * system is zeroed first unless `accumulate` != 0 (slab-by-slab builds).
 * Points outside every support contribute nothing.  Non-finite coordinates
 * are rejected (kdtree.cpp:14-17) when `validate` != 0. */
rbg_status rbg_assemble(rbg_ctx* ctx, const double* points, const double* h, uint64_t n,
                        int accumulate, int validate);
/* Same on device-resident inputs (no host copies, no validation). */
rbg_status rbg_assemble_device(rbg_ctx* ctx, const double* d_points, const double* d_h,
                               uint64_t n, int accumulate);

/* Device system buffer [values (nnz_upper) | rhs (m) | hits (m)], contiguous
 * fp64, for an external sum-allreduce across ranks (NCCL). */
rbg_status rbg_system_device(rbg_ctx* ctx, double** d_buffer, uint64_t* count);
/* Host copies of the assembled system.  Any pointer may be NULL.
 * design_nnz = sum of hits (BuildStats::design_nnz, solver.hpp:76). */
rbg_status rbg_get_system(rbg_ctx* ctx, double* values, double* rhs, double* hits,
                          uint64_t* design_nnz);
/* Replaces the device system from host arrays (hits may be NULL -> unchanged). */
rbg_status rbg_set_system(rbg_ctx* ctx, const double* values, const double* rhs,
                          const double* hits);

/* ---- solve ------------------------------------------------------------------
 * Replaces solve_weights (solver.cpp:289-330).  Method: preconditioned CG on
 * the assembled SPD system, stopping when ||r||_2 <= tol*||b||_2 (tol <= 0
 * selects 1e-12) within max_iter (<= 0 selects 20000) iterations.  The
 * preconditioner is a factorised sparse approximate inverse G^T G ~ B^-1 (one
 * small dense Cholesky per centre over its pattern neighbours); point Jacobi
 * for the bordered system or on request.  method RBG_SOLVE_BAND runs the
 * reference's own factorisation instead: LLT of the x-ordered band.
 * Ridge ladder as the reference: lambda in {0,1e-10,1e-9,1e-8,1e-7,1e-6} x
 * trace/side added to the diagonal, next rung on breakdown, a non-positive
 * pivot or non-convergence; all rungs failing -> RBG_RUNTIME_ERROR with
 * the reference's message.  c_out: m doubles (host). */
enum { RBG_SOLVE_AUTO = 0, RBG_SOLVE_PCG = 1, RBG_SOLVE_BAND = 2 };
enum { RBG_PREC_AUTO = 0, RBG_PREC_FSAI = 1, RBG_PREC_JACOBI = 2 };
typedef struct {
    double tol;
    int max_iter;
    int method;  /* RBG_SOLVE_* (0 = automatic: PCG) */
    int precond; /* RBG_PREC_*  (0 = automatic: FSAI, Jacobi with the border) */
} rbg_solve_options;
typedef struct {
    double ridge_lambda; /* SolveDiag::ridge_lambda */
    double ridge_shift;  /* SolveDiag::ridge_shift */
    int attempts;        /* SolveDiag::attempts */
    int iterations;      /* CG iterations of the successful rung */
    double rel_residual; /* recomputed ||b - A c|| / ||b|| */
    double solve_ms;     /* device time */
} rbg_solve_diag;
rbg_status rbg_solve(rbg_ctx* ctx, const rbg_solve_options* opts, double* c_out,
                     rbg_solve_diag* diag);

/* Orthogonal least-squares re-pass (least_squares_repass, solver.cpp:345-397),
 * the reference's last resort when the normal equations are numerically
 * singular (fit, solver.cpp:439-464): 4096-row chunks of the augmented design
 * [A P | h] of the n points (host arrays, AoS) through an incremental
 * Householder QR on the device, then R w = R[:, width].  w_out receives the
 * m (+ T with the polynomial border) unknowns; *ok = 0 when w is not finite
 * (rank-deficient design: the caller keeps the ridge solution).  Limited to
 * m + T <= rbg_repass_max_unknowns() (RBG_INVALID_ARGUMENT beyond). */
rbg_status rbg_least_squares_repass(rbg_ctx* ctx, const double* points, const double* h, uint64_t n,
                                    double* w_out, int* ok);
uint64_t rbg_repass_max_unknowns(void);

/* ---- evaluation -------------------------------------------------------------
 * Replaces evaluate_model / evaluate_shifted (model.cpp:50-72,192-194) with a
 * zero offset: f_q = sum_j c_j phi(|q - xi_j|) over the
 * support hits in ascending j, unfused mul/add -- bitwise equal to the
 * reference for the same c, plus the polynomial term when one is set
 * (rbg_set_model_poly).  c: m doubles; q: nq points (AoS). */
rbg_status rbg_evaluate(rbg_ctx* ctx, const double* c, const double* q, uint64_t nq, double* f);
rbg_status rbg_evaluate_device(rbg_ctx* ctx, const double* d_c, const double* d_q, uint64_t nq,
                               double* d_f);

/* error_report (model.cpp:196-232) plus RMS and max: evaluates c at the n
 * points and compares with h.  signed_errors (n, nullable) = f - h. */
typedef struct {
    double mean_absolute_error;
    double deviation_of_error;
    double mean_relative_error_pct;
    double rms_error;
    double max_abs_error;
} rbg_error_stats;
rbg_status rbg_error_report(rbg_ctx* ctx, const double* c, const double* points, const double* h,
                            uint64_t n, rbg_error_stats* out, double* signed_errors);

/* ---- linear-polynomial border (FitOptions::poly, solver.hpp:113-118) ---------
 * With the border enabled the system is the reference's bordered one
 * (solver.cpp:189-207, 238-262): side = m + T with T = dim + 1 terms
 * P = [x, y, (z), 1] per point; rbg_assemble then also accumulates
 * A^T P (T x m, term-major), P^T P (T x T) and P^T h (T), appended to the
 * device system buffer [values | rhs | hits | A^T P | P^T P | P^T h] (the unit
 * of the multi-GPU all-reduce, rbg_system_device), and rbg_solve solves the
 * bordered system; its border coefficients come from rbg_get_poly_solution
 * (Weights::poly, solver.hpp:102-105).  rbg_set_model_poly makes evaluation
 * add a_0 x + a_1 y (+ a_2 z) + a_T-1 (model.cpp:65-68); NULL removes it. */
rbg_status rbg_set_poly(rbg_ctx* ctx, int enable);
rbg_status rbg_get_border(rbg_ctx* ctx, double* atp, double* ptp, double* pth);
rbg_status rbg_set_border(rbg_ctx* ctx, const double* atp, const double* ptp, const double* pth);
rbg_status rbg_get_poly_solution(rbg_ctx* ctx, double* a);
rbg_status rbg_set_model_poly(rbg_ctx* ctx, const double* a);

/* ---- host-side helpers (no device work) ------------------------------------ */
/* Spatial slabs for multi-GPU sharding: writes n_slabs+1 boundaries along
 * `axis` at equal-count quantiles of the coordinates (bounds[0] = -inf,
 * bounds[n_slabs] = +inf) and the slab id of every point. */
rbg_status rbg_partition_slabs(int dim, const double* points, uint64_t n, int axis, int n_slabs,
                               double* bounds, uint32_t* slab_of);
/* ---- measurement helpers (bench; not on the hot path) ------------------- */
/* sum_p k_p and sum_p k_p^2 over nq host points (k_p = centres whose support
 * holds p with phi != 0): the algorithmic work of an assembly. */
rbg_status rbg_support_counts(rbg_ctx* ctx, const double* points, uint64_t nq, uint64_t* sum_k,
                              uint64_t* sum_k2);
/* fp64 FMA throughput of this GPU (TFLOP/s, FMA = 2 flops), microbenchmark. */
rbg_status rbg_fp64_peak(rbg_ctx* ctx, double* tflops);
/* The reference-exact phi of the numeric kernels (border, and the assembly's
 * inclusion test) against the reference arithmetic (kernel.hpp:42-62
 * with sqrt_rn, kdtree.cpp:64,74) on n sampled distances of every magnitude:
 * mismatches = inclusion differences + (wendland-3-0/3-1) values not bitwise
 * equal (must be 0); max relative / absolute error of phi. */
rbg_status rbg_phi_selftest(rbg_ctx* ctx, int kernel_family, double alpha, uint64_t n, uint64_t seed,
                            uint64_t* mismatches, double* max_rel, double* max_abs);
/* The same sampling for the variant the assembly's k-loop evaluates (one
 * Goldschmidt step + residual correction, FMA-contracted polynomial; A is
 * never output): mismatches = inclusion differences only (must be 0); max
 * relative error over values >= 1e-6; max absolute error. */
rbg_status rbg_phi_selftest_fast(rbg_ctx* ctx, int kernel_family, double alpha, uint64_t n, uint64_t seed,
                                 uint64_t* mismatches, double* max_rel, double* max_abs);
/* Assembly layout knobs (performance only; results are unaffected beyond
 * fp64 summation order): sub-tile edge = support radius / divisor (1..16,
 * 0 = automatic from the point density) and super-tile = S x S (x S)
 * sub-tiles (1..8, 0 = automatic).  The layout is rebuilt at the next
 * assembly. */
rbg_status rbg_set_tile_divisor(rbg_ctx* ctx, double divisor);
rbg_status rbg_set_super_factor(rbg_ctx* ctx, int S);
typedef struct {
    int built;             /* 0 until the first assembly after rbg_set_centres */
    int sub_div;           /* q: sub-tile edge = radius / q (before growth for huge grids) */
    int super_factor;      /* S */
    int n_buckets;         /* launch classes */
    uint64_t n_super;      /* super-tiles */
    uint64_t n_fallback;   /* super-tiles on the slow per-point path */
    uint32_t max_super_centres, max_sub_centres;
    double mean_super_centres, mean_sub_centres;
    double sub_edge;
    double build_ms;       /* host wall time of the layout build */
} rbg_layout_info;
rbg_status rbg_get_layout_info(rbg_ctx* ctx, rbg_layout_info* info);
/* Device time of the last assembly: point binning and tiled numeric phase. */
rbg_status rbg_assembly_times(rbg_ctx* ctx, double* bin_ms, double* tiles_ms);

/* phi(r) exactly as the device computes it (KernelSpec::evaluate, kernel.hpp:42-62). */
rbg_status rbg_kernel_value(int kernel_family, double alpha, double r, double* out);

#ifdef __cplusplus
}
#endif
#endif /* RBG_H */
