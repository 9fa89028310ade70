/* tgb_host.h — host-side input producers exported by libtgb (C ABI).
 *
 * These are the reference's untimed producers of hot-path inputs, restated
 * with identical floating-point formulas:
 *   tgb_mesh_size        <- tg::make_grid h = 2b/(n+1)          grid.cpp:14
 *   tgb_snap_to_node     <- tg::snap_to_node                     grid.cpp:23-30
 *   tgb_window_offset    <- tg::window_offset                    grid.cpp:32-38
 *   tgb_make_expsum      <- tg::make_expsum (Newton, 2M+1 nodes)  kernel.cpp:71-123
 *   tgb_expsum_for_interval <- tg::expsum_for_interval (Newton)  kernel.cpp:131-165
 *   tgb_reciprocal_expsum <- tg::reciprocal_expsum                kernel.cpp:205-250
 *   tgb_kernel_factors   <- tg::kernel_tensor (one axis)         kernel.cpp:182-203
 *   tgb_gauss_cell_integral <- tg::gauss_cell_integral           kernel.cpp:171-180
 *   tgb_primitive_norm   <- tg::primitive_norm                   basis.cpp:8-14
 *   tgb_gaussian_factor  <- one axis column of tg::discretize_basis basis.cpp:29-41
 * Return codes as in tgb.h; messages via tgb_host_last_error().
 */
#ifndef TGB_HOST_H
#define TGB_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* tgb_host_last_error(void);
double tgb_mesh_size(double b_half, int64_t n);
int tgb_snap_to_node(double b_half, int64_t n, double x, int64_t* node);
int tgb_window_offset(double b_half, int64_t n, double center, int64_t* ofs);
/* nodes/weights: 2m+1 entries each */
int tgb_make_expsum(int64_t m, double c0, double fit_lo, double fit_hi, double* nodes, double* weights,
                    double* scale, double* mesh);
/* factor: (doubled ? 2n : n) x terms, column-major */
int tgb_kernel_factors(double b_half, int64_t n, int64_t terms, const double* nodes, const double* weights,
                       int doubled, double* factor);
/* kernel.cpp:125-165: the reference's M schedule and golden-section C0 for a
 * Newton sum accurate to eps on [r_min, r_max] (m_cap = 2048 in the reference);
 * build it with tgb_make_expsum(m, c0, r_min, r_max, ...). */
int tgb_expsum_for_interval(double r_min, double r_max, double eps, int64_t m_cap, int64_t* m, double* c0);
/* kernel.cpp:205-250 (tg::reciprocal_expsum, term_cap 256 in the reference): rates and
 * weights need term_cap entries; *ok = 0 when the cap is hit. */
int tgb_reciprocal_expsum(double lo, double hi, double eps, int64_t term_cap, int64_t* terms, double* rates,
                          double* weights, double* achieved, int* ok);
double tgb_gauss_cell_integral(double t, double center, double h);
int tgb_primitive_norm(double alpha, int l, double* out);
int tgb_gaussian_factor(double b_half, int64_t n, double center, double alpha, int degree, double* column);

#ifdef __cplusplus
}
#endif

#endif /* TGB_HOST_H */
