/* rbfit_io.h -- C entry points of the reference's on-disk formats
 * (librbfit_b200.so, implemented in paper_1806_07884_b200/csrc/rbfit_io.cpp).
 *
 * Host-only (no GPU).  Files are byte-identical to the reference's:
 *   rbfit_io_save_model / rbfit_io_load_model  <- rbfit::save_model / load_model
 *                                                 (proj/core/src/model.cpp:76-190)
 *   rbfit_io_save_xyz / rbfit_io_load_records  <- rbfit::save_xyz / load_xyz /
 *                                                 load_eval_points / load_ref_points
 *                                                 (proj/core/src/data.cpp:126-196)
 *   rbfit_io_write_signed_errors               <- rbfit::write_signed_errors (model.cpp:234-256)
 *   rbfit_io_center_cloud                      <- rbfit::center_cloud (data.cpp:198-223)
 * Points are interleaved x, y doubles.  Status: 0 ok, 1 invalid argument
 * (std::invalid_argument), 2 runtime error (I/O, format); the message of the
 * calling thread's last failure is rbfit_io_last_error().  Loads park their
 * result per thread until the matching take call copies it out. */
#ifndef RBFIT_IO_H
#define RBFIT_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* rbfit_io_last_error(void);

/* family: rbg_kernel_family; offset: 2 doubles (NULL = 0, 0); poly: 3 doubles or NULL */
int rbfit_io_save_model(const char* path, int family, double alpha, const double* refs_xy, const double* weights,
                        uint64_t m, const double* offset, const double* poly);
/* scalars6 = {alpha, offset x, offset y, poly[3] (zeros without a polynomial)} */
int rbfit_io_load_model(const char* path, int* family, int* has_poly, uint64_t* m, double* scalars6);
int rbfit_io_take_model(double* refs_xy, double* weights);

int rbfit_io_save_xyz(const char* path, const double* xy, const double* h, uint64_t n);
/* kind: 0 load_xyz (3 columns), 1 load_eval_points (2 or 3), 2 load_ref_points (2) */
int rbfit_io_load_records(const char* path, int kind, uint64_t* n, int* arity);
int rbfit_io_take_records(double* rows /* n * arity doubles */);

int rbfit_io_write_signed_errors(const char* path, const double* xy, const double* h, uint64_t n,
                                 const double* offset, const double* predictions);
int rbfit_io_center_cloud(double* xy, uint64_t n, double* offset);

#ifdef __cplusplus
}
#endif
#endif
