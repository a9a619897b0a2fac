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
#ifdef __cplusplus
}
#endif
#endif
