// Host plan builder ("fac" in the paper's timings): everything the fused CUDA axis
// passes need for one axis, computed once per plan on the host in long double / fp64.
//
//   1. Gauss-Jacobi rule in t (construction deferred by the paper to
//      [Jacobi], PAPER.md:444 -> DESIGN.md reading R3): eigenvalues of the Jacobi matrix by implicit
//      symmetric QR (long double), Newton polish in t on p_n(cos t), weights lambda_j = 1 / sum_{k<n} p_k(x_j)^2.
//   2. Non-oscillatory generator P~_k + i Q~_k = M e^{i psi} at the nodes,
//      by the Cauchy transform h0 (tanh-sinh, long double) + the three-term recurrence
//      (reading R8 / route A5' of SURVEY.md).
//   3. The matrix B of eq:B with the weights folded in (reading R17), factorised by
//      Algorithm 1 with an adaptive rank cap (reading R11) and truncated at
//      sigma_{r+1} <= eps sigma_1.
//   4. The dense low-degree block W V and the bins m_j.
//
// This file shares no code with oracle/ (which is numpy; this is C++ with different algorithms for
// the nodes, weights and entries).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <set>

#include "jt_internal.h"

namespace jt {

using ld = long double;
using cld = std::complex<long double>;

static const ld PI_L = 3.141592653589793238462643383279502884L;

int64_t fft_length(int64_t n) {
  int64_t N = 16;
  while (N < n) N <<= 1;
  return N;
}

// ------------------------------------------------------------------------------------------------
// Recurrence coefficients of the orthonormal Jacobi polynomials for (1-x)^a (1+x)^b:
//   x p_k = beta_{k+1} p_{k+1} + alpha_k p_k + beta_k p_{k-1}.
// ------------------------------------------------------------------------------------------------
struct Recurrence {
  std::vector<ld> alpha, beta;  // alpha[0..K], beta[0..K] (beta[0] = 0)
  ld mu0 = 0;                   // int w = 2^{a+b+1} Gamma(a+1) Gamma(b+1) / Gamma(a+b+2)
};

static Recurrence make_recurrence(int64_t K, ld a, ld b) {
  Recurrence R;
  R.alpha.assign(K + 1, 0);
  R.beta.assign(K + 1, 0);
  for (int64_t k = 0; k <= K; ++k) {
    ld s = 2 * (ld)k + a + b;
    R.alpha[k] = (k == 0) ? (b - a) / (a + b + 2) : (b * b - a * a) / (s * (s + 2));
    if (k == 1) {
      R.beta[1] = sqrtl(4 * (1 + a) * (1 + b) / ((2 + a + b) * (2 + a + b) * (3 + a + b)));
    } else if (k >= 2) {
      ld kk = (ld)k;
      R.beta[k] = sqrtl(4 * kk * (kk + a) * (kk + b) * (kk + a + b) / (s * s * (s + 1) * (s - 1)));
    }
  }
  R.mu0 = powl(2.0L, a + b + 1) * expl(lgammal(a + 1) + lgammal(b + 1) - lgammal(a + b + 2));
  return R;
}

// x - alpha_k with x = cos t, in the cancellation-free t-form (1-x = 2 sin^2(t/2), 1+x = 2 cos^2(t/2)).
struct TForm {
  ld sx, cx;  // 1 - x, 1 + x
  bool low;   // t < pi/2
  explicit TForm(ld t) {
    ld s = sinl(t / 2), c = cosl(t / 2);
    sx = 2 * s * s;
    cx = 2 * c * c;
    low = t < PI_L / 2;
  }
  ld xm(ld alpha_k) const { return low ? (1 - alpha_k) - sx : cx - (1 + alpha_k); }
};

// p_n(cos t), d/dt p_n(cos t) and the Christoffel sum K = sum_{k<n} p_k(cos t)^2 by the (differentiated)
// recurrence.  (The Christoffel-Darboux shortcut 1/(beta_n p_n' p_{n-1}) loses ~1e-11 relative accuracy at
// the extreme nodes for n ~ 1e3 — measured — so the weights use the sum itself.)
static void pn_eval(const Recurrence &R, int64_t n, ld t, ld &pn, ld &dpn, ld &ksum) {
  TForm tf(t);
  const ld st = sinl(t);
  ld pk = 1 / sqrtl(R.mu0), pkm1 = 0, qk = 0, qkm1 = 0;  // p_k, p_{k-1}; q = dp/dt
  ld s = 0;
  for (int64_t k = 0; k < n; ++k) {
    s += pk * pk;
    const ld xm = tf.xm(R.alpha[k]);
    const ld pnew = (xm * pk - R.beta[k] * pkm1) / R.beta[k + 1];
    const ld qnew = (xm * qk - st * pk - R.beta[k] * qkm1) / R.beta[k + 1];
    pkm1 = pk;
    pk = pnew;
    qkm1 = qk;
    qk = qnew;
  }
  pn = pk;
  dpn = qk;
  ksum = s;
}

// Eigenvalues of the symmetric tridiagonal matrix T (diagonal d[0..n-1], off-diagonal e[k] = T[k][k+1])
// by implicit symmetric QR steps with the Wilkinson shift (the textbook method, e.g. Golub & Van Loan,
// "Matrix Computations", symmetric tridiagonal QR): the bottom of the active range shrinks whenever its last
// off-diagonal is negligible; otherwise one shifted step runs on the unreduced block [lo, hi] ending there.
// The step starts with the plane rotation that maps the first column (d[lo] - mu, e[lo]) of T - mu I onto a
// multiple of e_lo, applies it as a similarity, and chases the resulting bulge (the entry T[k-1][k+1])
// down the diagonal with one rotation per row.  Eigenvalues only, O(n^2) overall; the nodes are polished by
// Newton afterwards, so this only has to land each eigenvalue in its root's basin.
static bool tridiag_eigenvalues(std::vector<ld> &d, std::vector<ld> e) {
  const int64_t n = (int64_t)d.size();
  if (n <= 1) return true;
  e.resize(n - 1);
  auto negligible = [&](int64_t k) { return fabsl(e[k]) <= LDBL_EPSILON * (fabsl(d[k]) + fabsl(d[k + 1])); };
  int64_t hi = n - 1;
  int64_t steps = 0;
  while (hi > 0) {
    if (negligible(hi - 1)) {  // T[hi][hi] has decoupled: it is an eigenvalue
      e[hi - 1] = 0;
      --hi;
      continue;
    }
    if (++steps > 40 * n) return false;
    int64_t lo = hi - 1;
    while (lo > 0 && !negligible(lo - 1)) --lo;
    // Wilkinson shift: the eigenvalue of the trailing 2x2 block closer to its last diagonal entry
    const ld half = (d[hi - 1] - d[hi]) / 2, off = e[hi - 1];
    const ld root = hypotl(half, off);
    const ld mu = d[hi] - off * off / (half + (half < 0 ? -root : root));
    ld x = d[lo] - mu, z = e[lo];
    for (int64_t k = lo; k < hi; ++k) {
      // rotation [c s; -s c] in the plane (k, k+1) with [c s; -s c] (x, z)^T = (rho, 0)^T
      const ld rho = hypotl(x, z);
      const ld c = rho == 0 ? 1 : x / rho, s = rho == 0 ? 0 : z / rho;
      if (k > lo) e[k - 1] = rho;  // the bulge T[k-1][k+1] is gone
      const ld dk = d[k], dk1 = d[k + 1], ek = e[k];
      d[k] = c * c * dk + 2 * c * s * ek + s * s * dk1;
      d[k + 1] = s * s * dk - 2 * c * s * ek + c * c * dk1;
      e[k] = c * s * (dk1 - dk) + (c * c - s * s) * ek;
      if (k + 1 < hi) {  // the rotation of row k+1 pushes part of e[k+1] into the new bulge T[k][k+2]
        x = e[k];
        z = s * e[k + 1];
        e[k + 1] *= c;
      }
    }
  }
  return true;
}

// Gauss-Jacobi rule: t ascending, lambda (Christoffel numbers).  Returns false if Newton fails.
static bool gauss_jacobi_t(int64_t n, ld a, ld b, const Recurrence &R, std::vector<ld> &t,
                           std::vector<ld> &lam) {
  std::vector<ld> d(R.alpha.begin(), R.alpha.begin() + n), e(n, 0);
  for (int64_t i = 0; i + 1 < n; ++i) e[i] = R.beta[i + 1];
  if (!tridiag_eigenvalues(d, e)) return false;
  t.resize(n);
  for (int64_t j = 0; j < n; ++j) t[j] = acosl(std::max(-1.0L, std::min(1.0L, d[j])));
  std::sort(t.begin(), t.end());
  lam.assign(n, 0);
  bool ok = true;
#pragma omp parallel for schedule(dynamic, 16) reduction(&& : ok)
  for (int64_t j = 0; j < n; ++j) {
    ld tj = t[j], pn, dpn, ksum;
    int extra = -1;
    for (int it = 0; it < 20; ++it) {
      pn_eval(R, n, tj, pn, dpn, ksum);
      ld dt = pn / dpn;
      tj -= dt;
      if (extra < 0 && fabsl(dt) < 1e-12L) {
        extra = 2;
      } else if (extra > 0) {
        if (--extra == 0) break;
      }
    }
    if (extra != 0) ok = false;
    pn_eval(R, n, tj, pn, dpn, ksum);
    lam[j] = 1 / ksum;  // Christoffel number
    t[j] = tj;
  }
  if (!ok) return false;
  for (int64_t j = 0; j + 1 < n; ++j)
    if (!(t[j] < t[j + 1]) || !(lam[j] > 0)) return false;
  return lam[n - 1] > 0 && t[0] > 0 && t[n - 1] < PI_L;
}

// ------------------------------------------------------------------------------------------------
// Cauchy transform: g(t) := h0(x) / (pi w(x)) with h0(x) = PV int_{-1}^{1} w(y) / (x - y) dy, x = cos t.
//   h0(x) = int_{-1}^{x} (w(y)-w(x))/(x-y) dy + int_{x}^{1} (w(y)-w(x))/(x-y) dy + w(x) log((1+x)/(1-x)).
// Substituting y = -1 + (1+x)(1+s)/2 on [-1,x] and y = x + (1-x)(1+s)/2 on [x,1] (s in (-1,1)):
//   h0 / w(x) = J1 - J2 + log(cx/sx),
//   J1 = int expm1(a log1p(cx(1-s)/(2 sx)) + b log((1+s)/2)) / (1-s) ds,
//   J2 = int expm1(a log((1-s)/2) + b log1p(sx(1+s)/(2 cx))) / (1+s) ds,
// each by tanh-sinh (s = tanh(pi/2 sinh tau)) in long double; 1 -+ s are formed without cancellation,
// so the endpoint singularities of w at y = +-1 are resolved down to ~1e-4900.
// ------------------------------------------------------------------------------------------------
static ld cauchy_g(ld t, ld a, ld b) {
  TForm tf(t);
  const ld sx = tf.sx, cx = tf.cx;
  const ld h = 1.0L / 64, tau_max = 8.5L;
  const int K = (int)(tau_max / h);
  ld J1 = 0, J2 = 0;
  for (int k = -K; k <= K; ++k) {
    ld tau = k * h;
    ld u = (PI_L / 2) * sinhl(tau);
    ld em = expl(-2 * fabsl(u));
    ld one_m_s, one_p_s;  // 1 - s, 1 + s
    if (u >= 0) {
      one_m_s = 2 * em / (1 + em);
      one_p_s = 2 / (1 + em);
    } else {
      one_p_s = 2 * em / (1 + em);
      one_m_s = 2 / (1 + em);
    }
    ld jac = (PI_L / 2) * coshl(tau);  // ds/dtau = jac (1-s)(1+s)
    ld E1 = a * log1pl(cx * one_m_s / (2 * sx)) + b * logl(one_p_s / 2);
    ld E2 = a * logl(one_m_s / 2) + b * log1pl(sx * one_p_s / (2 * cx));
    J1 += expm1l(E1) * jac * one_p_s;
    J2 += expm1l(E2) * jac * one_m_s;
  }
  J1 *= h;
  J2 *= h;
  return (J1 - J2 + logl(cx / sx)) / PI_L;
}

// z_k(t) = p_k(x) - i H_k(x) / (pi w(x)) for k = 0..kmax, H_k the Cauchy transform of w p_k.
// H_k obeys the p-recurrence for k >= 1 and H_1 = ((x - alpha_0) H_0 - sqrt(mu0)) / beta_1, so
//   z_0 = p_0 (1 - i g),  z_1 = ((x - alpha_0) z_0 + i sqrt(mu0)/(pi w)) / beta_1,
//   z_{k+1} = ((x - alpha_k) z_k - beta_k z_{k-1}) / beta_{k+1}.
// Then P~_k(t) = sqrt(w(x) sin t) Re z_k and Q~_k(t) = sqrt(w(x) sin t) Im z_k (reading R8), and
// sqrt(lambda_j) z_k(t_j) = sqrt(w_j) (P~_k + i Q~_k)(t_j).
template <class Sink>
static void z_sweep(const Recurrence &R, ld t, ld a, ld b, int64_t kmax, Sink &&sink) {
  TForm tf(t);
  ld wx = powl(tf.sx, a) * powl(tf.cx, b);
  ld g = cauchy_g(t, a, b);
  ld p0 = 1 / sqrtl(R.mu0);
  ld zr = p0, zi = -p0 * g;  // z_0
  sink(0, zr, zi);
  if (kmax == 0) return;
  ld xm = tf.xm(R.alpha[0]);
  ld z1r = xm * zr / R.beta[1];
  ld z1i = (xm * zi + sqrtl(R.mu0) / (PI_L * wx)) / R.beta[1];
  sink(1, z1r, z1i);
  ld pr = zr, pi_ = zi, cr = z1r, ci = z1i;
  for (int64_t k = 1; k < kmax; ++k) {
    ld x_m = tf.xm(R.alpha[k]);
    ld nr = (x_m * cr - R.beta[k] * pr) / R.beta[k + 1];
    ld ni = (x_m * ci - R.beta[k] * pi_) / R.beta[k + 1];
    pr = cr;
    pi_ = ci;
    cr = nr;
    ci = ni;
    sink(k + 1, cr, ci);
  }
}

void modified_pq(double a, double b, int64_t nt, const double *t, int kmax, double *p_out, double *q_out) {
  Recurrence R = make_recurrence(kmax + 2, a, b);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t j = 0; j < nt; ++j) {
    ld tj = t[j];
    TForm tf(tj);
    ld scale = sqrtl(powl(tf.sx, (ld)a) * powl(tf.cx, (ld)b) * sinl(tj));
    z_sweep(R, tj, a, b, kmax, [&](int64_t k, ld zr, ld zi) {
      p_out[j * (kmax + 1) + k] = (double)(scale * zr);
      q_out[j * (kmax + 1) + k] = (double)(scale * zi);
    });
  }
}

// ------------------------------------------------------------------------------------------------
// Dense complex linear algebra for Algorithm 1 (column-major matrices).
// ------------------------------------------------------------------------------------------------
struct CMat {
  int m = 0, n = 0;
  std::vector<cd> a;
  CMat() = default;
  CMat(int m_, int n_) : m(m_), n(n_), a((size_t)m_ * n_, cd(0, 0)) {}
  cd &operator()(int i, int j) { return a[(size_t)j * m + i]; }
  const cd &operator()(int i, int j) const { return a[(size_t)j * m + i]; }
};

struct QRResult {
  std::vector<int> perm;           // column permutation (perm[k] = original column at position k)
  std::vector<std::vector<cd>> v;  // Householder vectors (v[k] has length m - k), normalised to |v|^2 = 2
  std::vector<cd> rdiag;
};

// Householder QR with column pivoting (largest remaining column norm first), `steps` steps.
static QRResult pivoted_qr(CMat A, int steps, bool pivot = true) {
  const int m = A.m, n = A.n;
  steps = std::min(steps, std::min(m, n));
  QRResult res;
  res.perm.resize(n);
  std::iota(res.perm.begin(), res.perm.end(), 0);
  for (int k = 0; k < steps; ++k) {
    if (pivot) {
      int best = k;
      double bestn = -1;
      for (int j = k; j < n; ++j) {
        double s = 0;
        for (int i = k; i < m; ++i) s += std::norm(A(i, j));
        if (s > bestn) {
          bestn = s;
          best = j;
        }
      }
      if (best != k) {
        for (int i = 0; i < m; ++i) std::swap(A(i, k), A(i, best));
        std::swap(res.perm[k], res.perm[best]);
      }
    }
    double nx = 0;
    for (int i = k; i < m; ++i) nx += std::norm(A(i, k));
    nx = std::sqrt(nx);
    std::vector<cd> v(m - k);
    cd alpha = 0;
    if (nx > 0) {
      cd x0 = A(k, k);
      cd ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : cd(1, 0);
      alpha = -ph * nx;
      for (int i = k; i < m; ++i) v[i - k] = A(i, k);
      v[0] -= alpha;
      double vn = 0;
      for (auto &z : v) vn += std::norm(z);
      double sc = std::sqrt(2.0 / vn);
      for (auto &z : v) z *= sc;  // H = I - v v^*
      for (int j = k; j < n; ++j) {
        cd dot = 0;
        for (int i = k; i < m; ++i) dot += std::conj(v[i - k]) * A(i, j);
        for (int i = k; i < m; ++i) A(i, j) -= v[i - k] * dot;
      }
    }
    res.v.push_back(v);
    res.rdiag.push_back(nx > 0 ? alpha : cd(0, 0));
  }
  return res;
}

// First `cols` columns of Q = H_0 ... H_{s-1} (m x cols).
static CMat form_q(const QRResult &qr, int m, int cols) {
  CMat Q(m, cols);
  for (int j = 0; j < cols; ++j) Q(j, j) = 1;
  for (int k = (int)qr.v.size() - 1; k >= 0; --k) {
    const auto &v = qr.v[k];
    if (v.empty()) continue;
    bool nz = false;
    for (auto &z : v) nz |= (z != cd(0, 0));
    if (!nz) continue;
    for (int j = 0; j < cols; ++j) {
      cd dot = 0;
      for (int i = k; i < m; ++i) dot += std::conj(v[i - k]) * Q(i, j);
      for (int i = k; i < m; ++i) Q(i, j) -= v[i - k] * dot;
    }
  }
  return Q;
}

// Least squares X = pinv(A) C for tall A (m x r, m >= r) via unpivoted Householder QR; columns of R
// with |R_ii| below 1e-14 |R_00| are treated as zero (minimum-norm in that direction).
static CMat lstsq(const CMat &A, const CMat &C) {
  const int m = A.m, r = A.n, nc = C.n;
  QRResult qr = pivoted_qr(A, r, false);
  // apply Q^* to C
  CMat QC = C;
  for (int k = 0; k < (int)qr.v.size(); ++k) {
    const auto &v = qr.v[k];
    if (v.empty()) continue;
    for (int j = 0; j < nc; ++j) {
      cd dot = 0;
      for (int i = k; i < m; ++i) dot += std::conj(v[i - k]) * QC(i, j);
      for (int i = k; i < m; ++i) QC(i, j) -= v[i - k] * dot;
    }
  }
  // R = upper triangle of Q^* A (recompute by applying reflectors to A)
  CMat RA = A;
  for (int k = 0; k < (int)qr.v.size(); ++k) {
    const auto &v = qr.v[k];
    if (v.empty()) continue;
    for (int j = 0; j < r; ++j) {
      cd dot = 0;
      for (int i = k; i < m; ++i) dot += std::conj(v[i - k]) * RA(i, j);
      for (int i = k; i < m; ++i) RA(i, j) -= v[i - k] * dot;
    }
  }
  double r00 = std::abs(RA(0, 0));
  CMat X(r, nc);
  for (int j = 0; j < nc; ++j) {
    for (int i = r - 1; i >= 0; --i) {
      if (std::abs(RA(i, i)) <= 1e-14 * r00) {
        X(i, j) = 0;
        continue;
      }
      cd s = QC(i, j);
      for (int kk = i + 1; kk < r; ++kk) s -= RA(i, kk) * X(kk, j);
      X(i, j) = s / RA(i, i);
    }
  }
  return X;
}

static CMat adjoint(const CMat &A) {
  CMat B(A.n, A.m);
  for (int j = 0; j < A.n; ++j)
    for (int i = 0; i < A.m; ++i) B(j, i) = std::conj(A(i, j));
  return B;
}

static CMat matmul(const CMat &A, const CMat &B) {
  CMat C(A.m, B.n);
  for (int j = 0; j < B.n; ++j)
    for (int k = 0; k < A.n; ++k) {
      cd bkj = B(k, j);
      if (bkj == cd(0, 0)) continue;
      for (int i = 0; i < A.m; ++i) C(i, j) += A(i, k) * bkj;
    }
  return C;
}

// One-sided (Hestenes) Jacobi SVD of a small complex square matrix: M = U diag(s) V^*, s descending.
static void jacobi_svd(const CMat &M, CMat &U, std::vector<double> &s, CMat &V) {
  const int n = M.n, m = M.m;
  CMat A = M;
  V = CMat(n, n);
  for (int i = 0; i < n; ++i) V(i, i) = 1;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0, be = 0;
        cd ga = 0;
        for (int i = 0; i < m; ++i) {
          al += std::norm(A(i, p));
          be += std::norm(A(i, q));
          ga += std::conj(A(i, p)) * A(i, q);
        }
        double ag = std::abs(ga);
        if (ag == 0 || ag <= 1e-17 * std::sqrt(al * be)) continue;
        off = std::max(off, ag / std::sqrt(al * be));
        cd ph = ga / ag;  // a_q' = conj(ph) a_q makes the Gram entry real
        double zeta = (be - al) / (2 * ag);
        double tt = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1 + zeta * zeta));
        double c = 1 / std::sqrt(1 + tt * tt), sn = c * tt;
        for (int i = 0; i < m; ++i) {
          cd xp = A(i, p), xq = std::conj(ph) * A(i, q);
          A(i, p) = c * xp - sn * xq;
          A(i, q) = sn * xp + c * xq;
        }
        for (int i = 0; i < n; ++i) {
          cd xp = V(i, p), xq = std::conj(ph) * V(i, q);
          V(i, p) = c * xp - sn * xq;
          V(i, q) = sn * xp + c * xq;
        }
      }
    if (off < 1e-16) break;
  }
  std::vector<double> nrm(n);
  for (int j = 0; j < n; ++j) {
    double sj = 0;
    for (int i = 0; i < m; ++i) sj += std::norm(A(i, j));
    nrm[j] = std::sqrt(sj);
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
  U = CMat(m, n);
  CMat V2(n, n);
  s.assign(n, 0);
  for (int jj = 0; jj < n; ++jj) {
    int j = ord[jj];
    s[jj] = nrm[j];
    for (int i = 0; i < m; ++i) U(i, jj) = nrm[j] > 0 ? A(i, j) / nrm[j] : cd(0, 0);
    for (int i = 0; i < n; ++i) V2(i, jj) = V(i, j);
  }
  V = V2;
}

// Random sample of `count` indices from [0, total) excluding `exclude`, from the seeded generator.
static std::vector<int> sample(std::mt19937_64 &rng, int total, int count, const std::vector<int> &exclude) {
  std::vector<char> used(total, 0);
  for (int e : exclude) used[e] = 1;
  std::vector<int> pool;
  pool.reserve(total);
  for (int i = 0; i < total; ++i)
    if (!used[i]) pool.push_back(i);
  count = std::min<int>(count, (int)pool.size());
  for (int i = 0; i < count; ++i) {
    std::uniform_int_distribution<int> dist(i, (int)pool.size() - 1);
    std::swap(pool[i], pool[dist(rng)]);
  }
  pool.resize(count);
  return pool;
}

static std::vector<int> merge_unique(const std::vector<int> &x, const std::vector<int> &y) {
  std::vector<int> out = x;
  std::set<int> seen(x.begin(), x.end());
  for (int v : y)
    if (seen.insert(v).second) out.push_back(v);
  return out;
}

// Z is n x nc row-major (Z[j*nc + c]).
struct ZView {
  const cd *z;
  int n, nc;
  cd operator()(int j, int c) const { return z[(size_t)j * nc + c]; }
};

static CMat gather(const ZView &Z, const std::vector<int> &rows, const std::vector<int> &cols) {
  CMat A((int)rows.size(), (int)cols.size());
  for (int jc = 0; jc < (int)cols.size(); ++jc)
    for (int ir = 0; ir < (int)rows.size(); ++ir) A(ir, jc) = Z(rows[ir], cols[jc]);
  return A;
}

static std::vector<int> iota_vec(int n) {
  std::vector<int> v(n);
  std::iota(v.begin(), v.end(), 0);
  return v;
}

// Algorithm 1 at rank parameter r; returns U0 (n x r), sigma (r), V0h (r x nc).
static void algorithm1(const ZView &Z, int r, int q, int sweeps, std::mt19937_64 &rng, CMat &U0,
                       std::vector<double> &sigma, CMat &V0h) {
  const int n = Z.n, nc = Z.nc;
  const std::vector<int> all_rows = iota_vec(n), all_cols = iota_vec(nc);
  std::vector<int> Pi_row, Pi_col;                 // Step 1: empty
  for (int sw = 0; sw < sweeps; ++sw) {            // Step 4: repeat steps 2-3
    // Step 2: sample rq rows, I = S_row u Pi_row, pivoted QR of Z_{I,:} -> Pi_col = first r pivots
    std::vector<int> I = merge_unique(Pi_row, sample(rng, n, r * q, Pi_row));
    QRResult qr = pivoted_qr(gather(Z, I, all_cols), r);
    Pi_col.assign(qr.perm.begin(), qr.perm.begin() + std::min<int>(r, (int)qr.perm.size()));
    // Step 3: sample rq columns, J = S_col u Pi_col, pivoted LQ of Z_{:,J} (= pivoted QR of Z_{:,J}^*)
    std::vector<int> J = merge_unique(Pi_col, sample(rng, nc, r * q, Pi_col));
    QRResult lq = pivoted_qr(adjoint(gather(Z, all_rows, J)), r);
    Pi_row.assign(lq.perm.begin(), lq.perm.begin() + std::min<int>(r, (int)lq.perm.size()));
  }
  // Step 5: Q_col from pivoted QR of Z_{:,Pi_col}; Q_row from pivoted QR of Z_{Pi_row,:}^*
  const int rc = (int)Pi_col.size(), rr = (int)Pi_row.size();
  CMat Zc = gather(Z, all_rows, Pi_col);
  CMat Qcol = form_q(pivoted_qr(Zc, rc), n, rc);
  CMat Zr = adjoint(gather(Z, Pi_row, all_cols));  // nc x rr
  CMat Qrow = form_q(pivoted_qr(Zr, rr), nc, rr);
  // Step 6: fresh samples; M = (Q_col)_{I,:}^+ Z_{I,J} ((Q_row^*)_{:,J})^+
  std::vector<int> I = merge_unique(Pi_row, sample(rng, n, r * q, Pi_row));
  std::vector<int> J = merge_unique(Pi_col, sample(rng, nc, r * q, Pi_col));
  CMat QcI((int)I.size(), rc);
  for (int c = 0; c < rc; ++c)
    for (int i = 0; i < (int)I.size(); ++i) QcI(i, c) = Qcol(I[i], c);
  CMat QrJ((int)J.size(), rr);  // rows J of Q_row  == ((Q_row^*)_{:,J})^*
  for (int c = 0; c < rr; ++c)
    for (int i = 0; i < (int)J.size(); ++i) QrJ(i, c) = Qrow(J[i], c);
  CMat X = lstsq(QcI, gather(Z, I, J));           // rc x |J|
  // M = X pinv(QrJ^*) = (pinv(QrJ) X^*)^*
  CMat M = adjoint(lstsq(QrJ, adjoint(X)));       // rc x rr
  // Step 7: SVD of M (square when rc == rr; pad otherwise)
  int ms = std::max(rc, rr);
  CMat Ms(ms, ms);
  for (int j = 0; j < rr; ++j)
    for (int i = 0; i < rc; ++i) Ms(i, j) = M(i, j);
  CMat UM, VM;
  jacobi_svd(Ms, UM, sigma, VM);
  CMat UMr(rc, ms), VMr(rr, ms);
  for (int j = 0; j < ms; ++j) {
    for (int i = 0; i < rc; ++i) UMr(i, j) = UM(i, j);
    for (int i = 0; i < rr; ++i) VMr(i, j) = VM(i, j);
  }
  U0 = matmul(Qcol, UMr);                 // n x ms
  V0h = adjoint(matmul(Qrow, VMr));       // ms x nc  (= V_M^* Q_row^*)
}

jt_status build_axis_host(AxisHost &ax, int64_t n, double a, double b, double eps, const jt_opts &opts,
                          std::string &err, const double *points, int kind, bool pair) {
  ax = AxisHost();
  ax.pair = pair;
  ax.n = n;
  ax.N = fft_length(n);
  ax.a = a;
  ax.b = b;
  ax.kind = kind;
  ax.uniform = points == nullptr;
  ax.k0 = (int)std::min<int64_t>(std::max(opts.k0, 0), n);
  const int k0 = ax.k0;
  Recurrence R = make_recurrence(n + 1, a, b);
  // Row scale s_j of the entries s_j z_k(t_j) (z_k = p_k - i H_k / (pi w), see z_sweep):
  //   uniform (Gauss-Jacobi nodes):  s_j = sqrt(lambda_j)  -> sqrt(w_j) (P~ + iQ~)_k(t_j)  (the weighted W J_n)
  //   nonuniform (given points):     s_j = sqrt(w(x_j) sin t_j) -> (P~ + iQ~)_k(t_j)      (J_n itself, W = I:
  //                                  "does not require ... quadrature nodes and weights")
  std::vector<ld> t, scale(n);
  if (ax.uniform) {
    std::vector<ld> lam;
    if (!gauss_jacobi_t(n, a, b, R, t, lam)) {
      err = "Gauss-Jacobi Newton iteration did not converge";
      return JT_ERR_NUMERIC;
    }
    for (int64_t j = 0; j < n; ++j) scale[j] = sqrtl(lam[j]);
    ax.t.resize(n);
    ax.w.resize(n);
    for (int64_t j = 0; j < n; ++j) {
      ax.t[j] = (double)t[j];
      TForm tf(t[j]);
      // w_j = lambda_j / (2^{a+b+1} sin^{2a+1}(t/2) cos^{2b+1}(t/2)) = lambda_j / (sx^{a+1/2} cx^{b+1/2})
      ax.w[j] = (double)(lam[j] / (powl(tf.sx, (ld)a + 0.5L) * powl(tf.cx, (ld)b + 0.5L)));
    }
  } else {
    t.resize(n);
    ax.t.assign(points, points + n);
    ax.w.assign(n, 1.0);
    for (int64_t j = 0; j < n; ++j) {
      if (!(points[j] > 0 && points[j] < 3.141592653589793) || (j > 0 && points[j] < points[j - 1])) {
        err = "nonuniform points must lie in (0, pi) in non-decreasing order";
        return JT_ERR_ARG;
      }
      t[j] = points[j];
      TForm tf(t[j]);
      scale[j] = sqrtl(powl(tf.sx, (ld)a) * powl(tf.cx, (ld)b) * sinl(t[j]));
    }
  }
  // Bins m_j = [t_j N / 2 pi] (eq:B) hold at most 4 rows each (the kernels' MAXR).  Gauss-Jacobi
  // nodes never exceed it.  Clustered nonuniform points are spread greedily to the next bins (m_j stays
  // non-decreasing in j; the factorisation absorbs the larger residual t_j - 2 pi m_j / N as extra rank),
  // displacing no point by more than 2 bins; if that fails the FFT length doubles (up to the kernels' 4096).
  // Spreading (reading R21): each point takes the first bin >= max([t_j N / 2 pi], previous point's bin) with room
  // (bins stay non-decreasing, rows of a bin contiguous), at most 2 bins right of its rounded bin, under a cap of 3
  // rows per bin (the kernels' MAXR = 3 instantiation: a quarter less row work than MAXR = 4), else 4; failing both,
  // the FFT length doubles.  Gauss-Jacobi nodes (<= 2 per bin) are never moved.
  if (pair) {
    // Paired real terms (DESIGN.md §6 "Two real rank terms per FFT"): half-integer bins m_j + 1/2 = t_j N / 2 pi
    // rounded to the nearest half-integer, i.e. m_j = floor(t_j N / 2 pi) in [0, N/2), so that bin m and its
    // conjugate mirror N - 1 - m pair up uniformly; at most 2 rows per bin (no spreading: the caller falls back)
    ax.bins.assign(n, 0);
    ax.bstart.assign(ax.N / 2 + 2, 0);
    // (where the nodes drift across a bin boundary -- a + b far from 0 -- a bin would take 3: the node moves to the
    // next bin, at most one bin right of its own, bins staying non-decreasing in j; the factorisation absorbs the
    // larger residual as in reading R21; failing that the caller keeps the unpaired set)
    int32_t prev = 0;
    for (int64_t j = 0; j < n; ++j) {
      const int32_t m0 = (int32_t)floorl(t[j] * (ld)ax.N / (2 * PI_L));
      int32_t m = std::max(m0, prev);
      while (m >= 0 && m < ax.N / 2 && ax.bstart[m + 1] >= 2) ++m;
      if (m0 < 0 || m >= ax.N / 2 || m - m0 > 1) {
        err = "pair: more than 2 nodes in a half-integer FFT bin";
        return JT_ERR_NUMERIC;
      }
      ax.bins[j] = prev = m;
      ax.bstart[m + 1]++;
    }
  } else
  for (;;) {
    bool ok = false;
    for (int cap : {3, 4}) {
      ax.bins.assign(n, 0);
      ax.bstart.assign(ax.N / 2 + 2, 0);
      ok = true;
      int32_t prev = 0;
      for (int64_t j = 0; j < n && ok; ++j) {
        const int32_t m0 = (int32_t)nearbyintl(t[j] * (ld)ax.N / (2 * PI_L));
        int32_t m = std::max(m0, prev);
        while (m <= ax.N / 2 && ax.bstart[m + 1] >= cap) ++m;
        if (m > ax.N / 2 || m - m0 > 2) ok = false;
        else {
          ax.bins[j] = prev = m;
          ax.bstart[m + 1]++;
        }
      }
      if (ok) break;
    }
    if (ok) break;
    if (ax.N >= 4096) {
      err = "points too clustered: more than 4 per FFT bin within 2 bins even at FFT length 4096";
      return JT_ERR_NUMERIC;
    }
    ax.N *= 2;
  }
  const int64_t N = ax.N;
  for (int64_t m = 0; m < N / 2 + 1; ++m) ax.bstart[m + 1] += ax.bstart[m];

  // Entries: phiv (k < k0) and Z = W B (k >= k0), row by row in long double.
  const int nc = (int)(n - k0);
  // (pair: e^{-2 pi i (m_j + 1/2) k / N} = e^{-2 pi i ((2 m_j + 1) k mod 2N) / 2N})
  const int64_t NT = pair ? 2 * N : N;
  std::vector<cld> twl(NT);
  for (int64_t q = 0; q < NT; ++q) twl[q] = cld(cosl(2 * PI_L * q / NT), -sinl(2 * PI_L * q / NT));
  ax.phiv.assign((size_t)n * k0, 0.0);
  std::vector<cd> Z((size_t)n * std::max(nc, 0));
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t j = 0; j < n; ++j) {
    ld sl = scale[j];
    int64_t mj = ax.bins[j];
    z_sweep(R, t[j], a, b, n - 1, [&](int64_t k, ld zr, ld zi) {
      if (kind == 1) {  // second kind: Q~ = Im z = Re(-i z) (NEXT-3, "the transform for Q~ is similar")
        const ld tr = zr;
        zr = zi;
        zi = -tr;
      }
      if (k < k0) {
        ax.phiv[(size_t)j * k0 + k] = (double)(sl * zr);
      } else {
        cld z(sl * zr, sl * zi);
        z *= pair ? twl[((2 * mj + 1) * k) % NT] : twl[(mj * k) % N];  // e^{-2 pi i m_j k / N}
        Z[(size_t)j * nc + (k - k0)] = cd((double)z.real(), (double)z.imag());
      }
    });
  }
  if (nc <= 0) {
    ax.r = 0;
    ax.v.assign(0, cd(0, 0));
    return JT_OK;
  }
  // Algorithm 1 with the adaptive cap (reading R11): accept when sigma_{rmax-1} <= 0.1 eps sigma_0.
  ZView zv{Z.data(), (int)n, nc};
  int cap = (int)std::min<int64_t>(n, nc);
  int rmax = opts.rmax_init > 0 ? opts.rmax_init
                                : std::max(32, (int)std::ceil(2 * std::log2((double)std::max<int64_t>(n, 2))));
  rmax = std::min(rmax, cap);
  // Growth cap ("growth cap (r > min(m,n)/4) aborts"; reading R25): the doubling may
  // raise rmax beyond its start value only up to min(n, n - k0) / 4; a factorisation still unconverged there
  // is JT_ERR_NUMERIC (the factored form would no longer be cheaper than the dense product).  A start value at
  // the full size (small n: B is factored exactly) never grows and never fails.
  const int grow_cap = std::max(rmax, cap / 4);
  std::mt19937_64 rng(opts.seed ^ 0x9E3779B97F4A7C15ULL);
  CMat U0, V0h;
  std::vector<double> sig;
  for (;;) {
    algorithm1(zv, rmax, std::max(opts.q, 1), std::max(opts.sweeps, 1), rng, U0, sig, V0h);
    double s0 = sig.empty() ? 0 : sig[0];
    bool converged = sig.size() < (size_t)rmax || sig.back() <= 0.1 * eps * s0;
    if (converged || rmax >= cap) break;
    if (rmax >= grow_cap) {
      err = "adaptive rank exceeded its growth cap min(n, n-k0)/4 = " + std::to_string(cap / 4) +
            " (rmax " + std::to_string(rmax) + " not converged at eps)";
      return JT_ERR_NUMERIC;
    }
    rmax = std::min(grow_cap, 2 * rmax);
  }
  ax.rmax_used = rmax;
  ax.sigma = sig;
  const double s0 = sig.empty() ? 0 : sig[0];
  int r = 0;
  while (r < (int)sig.size() && sig[r] > eps * s0) ++r;
  ax.r = r;
  ax.u.assign((size_t)n * r, cd(0, 0));
  ax.v.assign((size_t)r * N, cd(0, 0));
  for (int l = 0; l < r; ++l) {
    double sq = std::sqrt(sig[l]);
    for (int64_t j = 0; j < n; ++j) ax.u[(size_t)j * r + l] = U0(j, l) * sq;
    for (int c = 0; c < nc; ++c) ax.v[(size_t)l * N + k0 + c] = V0h(l, c) * sq;
  }
  if (pair) {
    // Two real rank terms per FFT.  Z ~ U0 diag(sig) V0h (complex rank r); the real row space of [Re Z; Im Z] has
    // dimension r' in [r, 2r] (measured r' <= r + 1 for the Jacobi kernels): with T = diag(sig) V0h (U0 has
    // orthonormal columns, so [Re Z; Im Z] and M = [Re T; Im T] have the same singular values and right singular
    // vectors), the right singular vectors V' (real, orthonormal) of M above eps sigma_0 span it, and Z ~ (Z V') V'^T
    // with REAL v'_l.  For real x = v'_l (.) alpha the FFT is conjugate-symmetric, so two terms (l, l') share one
    // complex FFT of (v'_l + i v'_l') e^{i pi k / N} (.) alpha (half-integer bins): with P = (u_l - i u_l') / 2 and
    // Q = (u_l + i u_l') / 2,  Re(u_l X_l[m] + u_l' X_l'[m]) = Re(P Z[m]) + Re(conj(Q) Z[N - 1 - m]).
    int r2 = 0;
    while (r2 < (int)sig.size() && sig[r2] > 0.01 * eps * s0) ++r2;
    CMat Mt(nc, 2 * r2);
    for (int l = 0; l < r2; ++l)
      for (int c = 0; c < nc; ++c) {
        const cd tv = V0h(l, c) * sig[l];
        Mt(c, l) = tv.real();
        Mt(c, r2 + l) = tv.imag();
      }
    CMat Us, Vs;
    std::vector<double> ss;
    jacobi_svd(Mt, Us, ss, Vs);
    int rp = 0;
    while (rp < (int)ss.size() && ss[rp] > eps * ss[0]) ++rp;
    const int np = (rp + 1) / 2;
    // u'_l = Z v'_l (complex), balanced like the unpaired factors: u' / sqrt(s), v' sqrt(s)
    std::vector<cd> up((size_t)n * 2 * np, cd(0, 0));
    std::vector<double> vp((size_t)2 * np * nc, 0.0);
    for (int l = 0; l < rp; ++l) {
      const double sq = std::sqrt(ss[l]);
      for (int c = 0; c < nc; ++c) vp[(size_t)l * nc + c] = Us(c, l).real() * sq;
#pragma omp parallel for
      for (int64_t j = 0; j < n; ++j) {
        cd acc(0, 0);
        for (int c = 0; c < nc; ++c) acc += Z[(size_t)j * nc + c] * Us(c, l).real();
        up[(size_t)j * 2 * np + l] = acc / sq;
      }
    }
    ax.r = np;
    ax.rreal = rp;
    ax.u.assign((size_t)n * 2 * np, cd(0, 0));
    ax.v.assign((size_t)np * N, cd(0, 0));
    for (int q = 0; q < np; ++q) {
      for (int64_t j = 0; j < n; ++j) {
        const cd ua = up[(size_t)j * 2 * np + 2 * q], ub = up[(size_t)j * 2 * np + 2 * q + 1];
        ax.u[(size_t)j * 2 * np + 2 * q] = 0.5 * (ua - cd(0, 1) * ub);                 // P
        ax.u[(size_t)j * 2 * np + 2 * q + 1] = std::conj(0.5 * (ua + cd(0, 1) * ub));  // conj(Q)
      }
      for (int c = 0; c < nc; ++c) {
        const int64_t k = k0 + c;
        const cld ph(cosl(PI_L * k / N), sinl(PI_L * k / N));
        const cld z = cld(vp[(size_t)(2 * q) * nc + c], vp[(size_t)(2 * q + 1) * nc + c]) * ph;
        ax.v[(size_t)q * N + k] = cd((double)z.real(), (double)z.imag());
      }
    }
    return JT_OK;
  }
  return JT_OK;
}

}  // namespace jt
