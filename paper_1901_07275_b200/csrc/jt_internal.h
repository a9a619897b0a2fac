// Internal declarations shared by the host plan builder (plan.cpp) and the CUDA side (jt_api.cu).
// Nothing here is part of the C ABI (include/jt.h).
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/jt.h"

namespace jt {

using cd = std::complex<double>;

// Host-side plan of one axis.  Notation follows SURVEY.md §8(a) / PAPER.md §3.1:
//   n        axis length; N = FFT length (power of two >= max(n, 16)); for power-of-two n >= 16, N == n
//   k0       degrees 0..k0-1 form the dense block V, k0 = min(opts.k0, n)
//   r        rank of the factorisation of B (eq:approxA)
//   t, w     nodes (ascending) and trigonometric weights (introduction:modrule, reading R2)
//   u        n x r  (u[j*r + l]) : u~_l = W u_l S^{1/2}     (weights folded)
//   v        r x N  (v[l*N + k]) : v_l = S^{1/2} V_l, zero for k < k0 and k >= n
//   phiv     n x k0 (phiv[j*k0 + k]) : sqrt(w_j) P~_k(t_j)
//   bins     n     : m_j = [t_j N / 2 pi]  (eq:B / eq:permuDFT)
//   bstart   N/2+2 : rows of bin m are bstart[m] .. bstart[m+1]-1 (bins are monotone in j)
struct AxisHost {
  int64_t n = 0, N = 0;
  int k0 = 0, r = 0;
  double a = 0, b = 0;
  std::vector<double> t, w;
  std::vector<cd> u, v;
  std::vector<double> phiv;
  std::vector<int32_t> bins, bstart;
  std::vector<double> sigma;  // singular values of Algorithm 1's middle matrix (descending)
  int rmax_used = 0;
  bool uniform = true;  // Gauss-Jacobi nodes, weighted rows (false: caller's points, unweighted)
  int kind = 0;         // 0: P~ (first kind), 1: Q~ (second kind)
  // pair: two REAL rank terms per complex FFT (forward kernels with Cfg::PAIR).  Then bins are
  // m_j = floor(t_j N / 2 pi) (half-integer grid m + 1/2, <= 2 rows per bin), r counts the FFTs (pairs),
  // u is n x 2r: u[j*2r + 2q] = P_q[j], u[j*2r + 2q + 1] = conj(Q_q)[j], v[q*N + k] = (v'_{2q} + i v'_{2q+1})[k]
  // e^{i pi k / N}, and y_j = (W V a_V)_j + Re sum_q (P_q[j] Z_q[m_j] + conj(Q_q)[j] Z_q[N - 1 - m_j]),
  // Z_q = F_N (v_q (.) a).  rreal = the number of real terms (2r or 2r - 1).
  bool pair = false;
  int rreal = 0;
};

// Builds one axis's plan on the host.  Returns JT_OK or an error code with `err` filled.
// points == nullptr: uniform (Gauss-Jacobi nodes); else n caller points in (0, pi), non-decreasing.
// kind 0: P~, 1: Q~.
jt_status build_axis_host(AxisHost &ax, int64_t n, double a, double b, double eps, const jt_opts &opts,
                          std::string &err, const double *points = nullptr, int kind = 0, bool pair = false);

// Debug / test hook: P~_k(t) and Q~_k(t) (PAPER.md eq:modifiedjac, eq:modifiedjac2; reading R8 for Q~)
// for k = 0..kmax at the angles t[0..nt-1], by the plan's own route (Cauchy transform h0 + recurrence).
void modified_pq(double a, double b, int64_t nt, const double *t, int kmax, double *p_out, double *q_out);

// FFT length used for an axis of length n.
int64_t fft_length(int64_t n);

}  // namespace jt
