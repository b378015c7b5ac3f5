/*
 * rbf_oracle.h -- CPU restatement of the reference (rbfit) CS-RBF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1806_07884_b200/,
 * include/) links, loads or calls this code.  Only tests/, the smoke() check in
 * __graft_entry__.py and the cpu_baseline / --impl reference legs of bench.py
 * may use it, and only as the checker (or the timed CPU baseline), never as the
 * thing measured for the GPU numbers.
 *
 * Every function restates one reference function; the citation is the
 * reference file:line under /root/reference/proj/core.  Compiled with
 * -ffp-contract=off so the arithmetic is the same separate mul/add sequence the
 * reference's x86-64 baseline build performs; the sparse assembly sums every
 * A^T A / A^T h entry in ascending point order, which is the order
 * GramOps::self / CooMatrix::transpose_matvec use, so its results are bitwise
 * equal to the reference's dense build for the same inputs (checked against
 * fixtures produced by the compiled reference itself, tests/golden/).
 *
 * Parity pinning: see DESIGN.md section "Oracle".  The 3-D / wendland-3-2
 * path has no reference counterpart (the reference is 2-D only) and is
 * "restatement-only, parity unpinned by the reference".
 */
#ifndef RBF_ORACLE_H
#define RBF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Kernel family ids; 0..2 are the reference's KernelFamily order
 * (kernel.hpp:21-25), 3 is the BASELINE wendland-3-2 extension. */
enum { ORC_W30 = 0, ORC_W31 = 1, ORC_W33 = 2, ORC_W32 = 3 };

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_RUNTIME = 2, ORC_DOMAIN = 3 };

/* KernelSpec::evaluate (kernel.hpp:42-62): domain_error on negative/non-finite r. */
int orc_phi(int family, double alpha, double r, double* out);

/* radical_inverse (data.cpp:76-87). */
double orc_radical_inverse(unsigned base, uint64_t index);
/* franke (data.cpp:108-116), the code form with the unsquared (9y+1)/10 term. */
double orc_franke(double x, double y);

/* Pattern predicate shared by oracle and GPU: upper-triangle CSR of centre
 * pairs i <= j with dist2(c_i, c_j) < (2*(1/alpha))^2, columns ascending.
 * Call with cols == NULL to get the row pointer (and nnz) only. */
int orc_pattern(int dim, const double* centres, uint64_t m, double alpha,
                uint64_t* row_ptr /* m+1 */, uint32_t* cols /* nullable */);

/* Sparse restatement of build_normal_system for one block
 * (solver.cpp:131-236 with assemble_submatrix coo.cpp:166-192,
 * transpose_matvec coo.cpp:75-82, gram_self coo.cpp:134-151):
 * vals[slot(i,j)] = sum over points p ascending of phi_i(p)*phi_j(p), i <= j;
 * rhs[i] = sum over p ascending of phi_i(p)*h_p; hits[i] = #{p: phi_i(p) != 0}.
 * Outputs are overwritten.  Returns ORC_RUNTIME if an update falls outside the
 * pattern (impossible for a consistent pattern). */
int orc_assemble(int dim, const double* pts, const double* h, uint64_t n,
                 const double* centres, uint64_t m, int family, double alpha,
                 const uint64_t* row_ptr, const uint32_t* cols,
                 double* vals, double* rhs, uint64_t* hits);

/* evaluate_shifted with delta = 0 (model.cpp:50-72): f = sum_j w_j phi_j(q)
 * over the support hits in ascending j, as separate mul/add. */
int orc_evaluate(int dim, const double* centres, uint64_t m, const double* w,
                 int family, double alpha, const double* q, uint64_t nq, double* f);

/* error_report (model.cpp:196-232) plus RMS and max |e| (not in the
 * reference; defined here as sqrt(mean e^2) and max |e|). */
int orc_error_report(const double* f, const double* h, uint64_t n, double* mae,
                     double* deviation, double* rel_pct, double* rms, double* max_abs);

/* solve_weights (solver.cpp:289-330): Cholesky with the ridge ladder
 * lambda in {0,1e-10,...,1e-6} x trace/side.  Eigen's LLT is not available
 * here; this is a textbook right-looking Cholesky (same method, different
 * rounding).  bad_pivot is first_bad_pivot (solver.cpp:56-72) on failure. */
int orc_cholesky_solve(uint64_t side, const double* b_dense, const double* rhs,
                       double* x, double* ridge_lambda, int* attempts, int64_t* bad_pivot);

/* Jacobi-preconditioned CG on the upper-CSR system -- the GPU solve's method
 * and stopping rule (||r||_2 <= tol * ||b||_2, at most max_iter iterations),
 * restated sequentially.  shift is added to every diagonal (ridge). */
int orc_pcg(uint64_t m, const uint64_t* row_ptr, const uint32_t* cols,
            const double* vals, const double* rhs, double shift, double tol,
            int max_iter, double* x, int* iters, double* rel_res);

/* Linear-polynomial border blocks A^T P (T x m, term-major), P^T P (T x T),
 * P^T h (T), T = dim + 1 (solver.cpp:189-207, 238-262). */
int orc_border(int dim, const double* pts, const double* h, uint64_t n, const double* centres,
               uint64_t m, int family, double alpha, double* atp, double* ptp, double* pth);

/* orc_evaluate plus the polynomial term a (T coefficients, model.cpp:65-68). */
int orc_evaluate_poly(int dim, const double* centres, uint64_t m, const double* w, const double* a,
                      int family, double alpha, const double* q, uint64_t nq, double* f);

/* Upper CSR -> dense symmetric row-major (m*m). */
void orc_densify(uint64_t m, const uint64_t* row_ptr, const uint32_t* cols,
                 const double* vals, double* dense);

#ifdef __cplusplus
}
#endif
#endif
