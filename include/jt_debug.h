/* jt_debug.h — test hooks exported by libjt.so (not part of the transform API).
 *
 * jt_debug_modified_pq: the modified Jacobi functions of the first and second kind,
 *     P~_k(t) = C_k P_k^{(a,b)}(cos t) sin(t/2)^{a+1/2} cos(t/2)^{b+1/2}     (eq:modifiedjac)
 *     Q~_k(t) = C_k Q_k^{(a,b)}(cos t) sin(t/2)^{a+1/2} cos(t/2)^{b+1/2}     (eq:modifiedjac2)
 * for k = 0..kmax at the host angles t[0..nt-1] in (0, pi), computed by the PLAN's route: the
 * Cauchy transform h0 (tanh-sinh, long double) and the three-term recurrence.  Q~ follows the
 * equal-amplitude normalisation of DESIGN.md reading R8 (P~ + iQ~ = M e^{i psi}, Wronskian
 * (2k+a+b+1)/pi > 0).  Outputs are row-major nt x (kmax+1) host arrays owned by the
 * caller.  Returns JT_ERR_ARG on null pointers / negative sizes, JT_ERR_DOMAIN if a, b are not in (-1,1).
 */
#ifndef JT_DEBUG_H
#define JT_DEBUG_H
#include "jt.h"
#ifdef __cplusplus
extern "C" {
#endif
jt_status jt_debug_modified_pq(double a, double b, int64_t nt, const double *t, int kmax, double *p_out,
                               double *q_out);

/* jt_debug_pair_factors: the plan's SECOND factor set of axis `axis`, used by its forward passes where the axis has
 * one (uniform axes of FFT length 256 / 512 / 2048 / 4096; DESIGN.md §6 "Two real rank terms per FFT"; the method is eq:oneJ,
 * PAPER.md:610, with a factorisation of eq:approxA whose v'_l are REAL, so two terms share one complex FFT):
 *   *r      number of FFTs (pairs) per line, 0 if the axis has no paired set (then nothing else is written)
 *   *rreal  number of real rank terms (2 r or 2 r - 1)
 *   u       n x 2r complex (row-major, interleaved re/im): column 2q = P_q, 2q + 1 = conj(Q_q)
 *   v       r x N complex: (v'_{2q} + i v'_{2q+1})[k] e^{i pi k / N} (zero for k < k0 and k >= n)
 *   phiv    n x k0 (as jt_plan_factors), bins n int32: m_j = floor(t_j N / 2 pi) (the half-integer grid m + 1/2)
 * so that  y_j = (phiv a_V)_j + Re sum_q ( P_q[j] Z_q[m_j] + conj(Q_q)[j] Z_q[N - 1 - m_j] ),
 * Z_q[m] = sum_k v_q[k] a_k e^{+2 pi i k m / N}.  Host arrays owned by the caller (any may be NULL); sizes from
 * jt_plan_info (n, N, k0) and a first call with NULL arrays (*r).  JT_ERR_ARG on a bad plan / axis. */
jt_status jt_debug_pair_factors(jt_plan_t p, int axis, int *r, int *rreal, double *u_host, double *v_host,
                                double *phiv_host, int32_t *bins_host);

/* Virtual ranks on one GPU (tests of the distributed schedule, with only one GPU at hand).
 *
 * jt_debug_vgroup_create makes a group of `nranks` virtual ranks; jt_debug_plan_virtual then builds rank `rank`'s
 * distributed plan exactly as jt_plan_dist_ex does (same n / a / b / eps / opts / flags on every rank, same
 * x-slab / y-slab boxes, same schedule, same kernels, same chunk-major layouts), except that the all-to-all is
 * not NCCL: rank g's exchange copies rows of block g of every member's send buffer into its own receive buffer
 * with one cudaMemcpyAsync per peer on its own stream, ordered by cross-stream CUDA events and a host barrier
 * of the G members (so the G ranks must be driven by G host threads, each calling jt_forward / jt_inverse /
 * jt_*_host* on its own plan and stream, like G processes would).  No kernel waits on another: the copies are
 * ordinary stream work.  A member that does not reach an exchange within `timeout_ms` makes the others' call
 * return JT_ERR_NCCL and marks their plans broken (the communicator-abort path of the NCCL build).
 * All members must use the same device.  Destroy every member plan (jt_destroy) before the group.
 * Errors: JT_ERR_ARG for bad sizes, a NULL group, a rank that already has a plan, or destroying a group that
 * still has plans. */
/* Bounds-check build (libjt_checks.so, compiled with -DJT_CHECKS=1 by build.py): every global index, shared-memory
 * exchange slot, bin index and tensor-memory column the kernels touch is checked; a violation is counted and its
 * access skipped (no fault).  jt_debug_checks synchronises the device and returns whether this build checks
 * (*enabled), the number of violations since the last call (*count) and the kernel source line of the first
 * (*line), then resets both.  JT_ERR_ARG on NULL arguments. */
jt_status jt_debug_checks(int *enabled, unsigned long long *count, int *line);

/* jt_forward_axis / jt_inverse_axis (plain layout, out of place or in place, never term-split) with the input and
 * output extents DECLARED by the caller (elements from the pointers) instead of derived from the geometry: the
 * negative control of the checks build (declaring out_lim smaller than outer * n[axis] * inner must produce
 * violations and leave the elements beyond out_lim untouched). */
jt_status jt_debug_axis_pass_lim(jt_plan_t p, int axis, int inverse, const double *in, double *out, int64_t outer,
                                 int64_t inner, int64_t in_lim, int64_t out_lim, void *cuda_stream);

typedef struct jt_vgroup_s *jt_vgroup_t;
jt_status jt_debug_vgroup_create(jt_vgroup_t *out, int nranks, int timeout_ms);
jt_status jt_debug_vgroup_destroy(jt_vgroup_t group);
jt_status jt_debug_plan_virtual(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[],
                                double eps, const jt_opts *opts, jt_vgroup_t group, int rank, int flags);
#ifdef __cplusplus
}
#endif
#endif
