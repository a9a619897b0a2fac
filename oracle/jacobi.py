"""ORACLE for the d-dimensional uniform discrete Jacobi transform (arXiv 1901.07275).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
The product path (`paper_1901_07275_b200/`) never imports, links or executes
anything under `oracle/`, and this module imports nothing from the product
path: the two share no code (the seeded inputs come from `seeded_inputs.py`,
which holds none of the method's arithmetic).

What it computes is the PLAIN DEFINITION that the paper's fast method reaches
to within ~eps:

  * p_k, the orthonormal Jacobi polynomials for the weight (1-x)^a (1+x)^b on
    [-1, 1] (PAPER.md:54-61 eq:GJquadrule with reading R1 of DESIGN.md), by
    their three-term recurrence (§2.2 and PAPER.md:526, "three-term
    recurrence relations");
  * the n-point Gauss-Jacobi rule: nodes x_j = cos t_j (zeros of p_n), t_j
    ascending (reading R5), Christoffel numbers lambda_j = 1 / sum_{k<n} p_k(x_j)^2
    (construction deferred by the paper to [Jacobi],
    PAPER.md:444 -> reading R3: Golub-Welsch start, Newton in t);
  * Phi[j, k] = sqrt(lambda_j) p_k(x_j) = sqrt(w_j) P~_k(t_j), the orthogonal
    matrix W J_n of PAPER.md:495-509 (readings R1, R2);
  * forward: values = (Phi_0 (x) Phi_1 (x) ... ) coeffs  (eq:2Djac PAPER.md:659-662,
    eq:3Djac PAPER.md:698-701, weighted per eq:TJ / eq:TJ3pre PAPER.md:669-706),
    inverse: the transpose in every axis (eq:oneJinv PAPER.md:621-630,
    eq:invTJ PAPER.md:683-687, eq:invTJ3 PAPER.md:731-735).

Precision: nodes and Phi entries in numpy longdouble (80-bit x87 extended,
eps 1.08e-19), rounded once to float64; the separable apply runs in float64
with numpy's BLAS (a library matmul serves as the mode-product step).  The
literal O(n^{2d}) Kronecker sum is `kron_matrix` (small sizes only).

Every function here is pinned by `tests/test_oracle.py` and (the NEXT-row functions:
phi_points, cauchy_h0 / modified_q_all, phi_q_uniform, forward_ex, adjoint_ex,
forward_axes) `tests/test_next.py` against things other than itself (DCT-II/III,
DST-I and DST-III closed forms via scipy, trigonometric closed forms summed
literally, gamma-function endpoint values, Beta-function moments via mpmath,
40-digit mpmath Golub-Welsch + hypergeometric Jacobi values, scipy Jacobi
polynomials, mpmath Ferrers Q, the Wronskian, orthogonality and the adjoint
identity).  No function is "parity unpinned".
"""
from __future__ import annotations

import functools

import mpmath
import numpy as np

LD = np.longdouble


def _ld(x) -> np.longdouble:
    """Exact conversion of a Python/mpmath number to longdouble via a 30-digit string."""
    return LD(mpmath.nstr(mpmath.mpf(x), 30, strip_zeros=False))


def recurrence_coefficients(n: int, a: float, b: float):
    """alpha_k (k = 0..n) and beta_k (k = 0..n, beta_0 := 0) of the orthonormal Jacobi family.

    x p_k = beta_{k+1} p_{k+1} + alpha_k p_k + beta_k p_{k-1}   (the
    standard Jacobi-matrix coefficients; "three-term recurrence").
      alpha_0 = (b - a) / (a + b + 2)
      alpha_k = (b^2 - a^2) / ((2k+a+b)(2k+a+b+2))                      k >= 1
      beta_1^2 = 4 (1+a)(1+b) / ((2+a+b)^2 (3+a+b))
      beta_k^2 = 4k(k+a)(k+b)(k+a+b) / ((2k+a+b)^2 (2k+a+b+1)(2k+a+b-1))  k >= 2
    Computed in longdouble.
    """
    a = _ld(a)
    b = _ld(b)
    alpha = np.zeros(n + 1, dtype=LD)
    beta = np.zeros(n + 1, dtype=LD)
    alpha[0] = (b - a) / (a + b + 2)
    for k in range(1, n + 1):
        s = 2 * k + a + b
        alpha[k] = (b * b - a * a) / (s * (s + 2))
    if n >= 1:
        beta[1] = np.sqrt(4 * (1 + a) * (1 + b) / ((2 + a + b) ** 2 * (3 + a + b)))
    for k in range(2, n + 1):
        s = 2 * k + a + b
        beta[k] = np.sqrt(4 * k * (k + a) * (k + b) * (k + a + b) / (s * s * (s + 1) * (s - 1)))
    return alpha, beta


def mu0(a: float, b: float) -> np.longdouble:
    """mu_0 = int_{-1}^{1} (1-x)^a (1+x)^b dx = 2^{a+b+1} Gamma(a+1) Gamma(b+1) / Gamma(a+b+2)."""
    with mpmath.workdps(40):
        v = mpmath.power(2, a + b + 1) * mpmath.gamma(a + 1) * mpmath.gamma(b + 1) / mpmath.gamma(a + b + 2)
        return _ld(v)


def _x_minus_alpha_factory(t):
    """x - alpha_k with x = cos t, written in t to avoid cancellation near x = +-1 (reading R3).

    t < pi/2: (1 - alpha_k) - 2 sin^2(t/2);  t >= pi/2: 2 cos^2(t/2) - (1 + alpha_k).
    Returns a function of alpha_k (the t-dependent parts are computed once).
    """
    s2 = 2 * np.sin(t / 2) ** 2
    c2 = 2 * np.cos(t / 2) ** 2
    low = t < LD(np.pi) / 2
    return lambda alpha_k: np.where(low, (1 - alpha_k) - s2, c2 - (1 + alpha_k))


def p_all(t, kmax: int, a: float, b: float, with_dt: bool = False):
    """p_k(cos t) for k = 0..kmax (rows) at the angles t (columns), longdouble.

    Forward three-term recurrence.  With `with_dt`, also the
    t-derivatives d/dt p_k(cos t) from the differentiated recurrence
      q_{k+1} = ((x - alpha_k) q_k - sin(t) p_k - beta_k q_{k-1}) / beta_{k+1}.
    """
    t = np.asarray(t, dtype=LD)
    alpha, beta = recurrence_coefficients(kmax + 1, a, b)
    P = np.zeros((kmax + 1,) + t.shape, dtype=LD)
    Q = np.zeros_like(P) if with_dt else None
    P[0] = 1 / np.sqrt(mu0(a, b))
    sint = np.sin(t)
    x_minus = _x_minus_alpha_factory(t)
    for k in range(kmax):
        xm = x_minus(alpha[k])
        prev = P[k - 1] if k >= 1 else 0
        P[k + 1] = (xm * P[k] - beta[k] * prev) / beta[k + 1]
        if with_dt:
            qprev = Q[k - 1] if k >= 1 else 0
            Q[k + 1] = (xm * Q[k] - sint * P[k] - beta[k] * qprev) / beta[k + 1]
    return (P, Q) if with_dt else P


@functools.lru_cache(maxsize=64)
def gauss_jacobi(n: int, a: float, b: float):
    """n-point Gauss-Jacobi rule in the trigonometric variable.

    Returns (t, lam, w) in longdouble with t ascending in (0, pi):
      t      nodes, x_j = cos t_j the zeros of p_n;
      lam    Christoffel numbers lambda_j = 1 / sum_{k<n} p_k(x_j)^2 (weights of eq:GJquadrule);
      w      trigonometric weights of introduction:modrule with reading R2:
             w_j = lambda_j / (2^{a+b+1} sin^{2a+1}(t_j/2) cos^{2b+1}(t_j/2)).
    Construction (reading R3; the paper defers it to [Jacobi]):
    Golub-Welsch eigenvalues of the Jacobi matrix (float64 LAPACK) as starting
    points, then Newton in t on p_n(cos t) in longdouble: iterate until
    max |dt| < 1e-12, then two more steps (quadratic convergence takes the error
    to the longdouble noise floor, ~1e-18; a final step above 1e-15 is an error).
    """
    alpha, beta = recurrence_coefficients(n, a, b)
    J = np.diag(alpha[:n].astype(np.float64))
    if n > 1:
        off = beta[1:n].astype(np.float64)
        J += np.diag(off, 1) + np.diag(off, -1)
    x0 = np.linalg.eigvalsh(J)
    t = np.sort(np.arccos(np.clip(x0, -1.0, 1.0))).astype(LD)
    extra = None
    for it in range(16):
        P, Q = p_all(t, n, a, b, with_dt=True)
        dt = P[n] / Q[n]
        t = t - dt
        step = float(np.max(np.abs(dt)))
        if extra is None and step < 1e-12:
            extra = 2
        elif extra is not None:
            extra -= 1
            if extra == 0:
                break
    if extra != 0 or step > 1e-15:
        raise RuntimeError("oracle Newton did not converge")
    order = np.argsort(t)
    t = t[order]
    P = p_all(t, n - 1, a, b)
    lam = 1 / np.sum(P * P, axis=0)
    aa, bb = _ld(a), _ld(b)
    w = lam / (LD(2) ** (aa + bb + 1) * np.sin(t / 2) ** (2 * aa + 1) * np.cos(t / 2) ** (2 * bb + 1))
    return t, lam, w


@functools.lru_cache(maxsize=64)
def phi(n: int, a: float, b: float) -> np.ndarray:
    """The orthogonal n x n matrix W J_n: Phi[j,k] = sqrt(lambda_j) p_k(x_j).

    Row j = node t_j (ascending), column k = degree k.  Entries in longdouble,
    rounded once to float64.  Equal to sqrt(w_j) P~_k(t_j) of eq:modifiedjac / tf:transout
    (reading R2).  Returned read-only.
    """
    t, lam, _ = gauss_jacobi(n, a, b)
    P = p_all(t, n - 1, a, b)           # (k, j)
    M = (np.sqrt(lam)[None, :] * P).T    # (j, k)
    out = np.ascontiguousarray(M.astype(np.float64))
    out.setflags(write=False)
    return out


def _mode_product(M: np.ndarray, X: np.ndarray, axis: int) -> np.ndarray:
    """Y = X x_axis M, i.e. Y[..., i, ...] = sum_k M[i, k] X[..., k, ...] (fp64 BLAS)."""
    return np.moveaxis(np.tensordot(M, X, axes=([1], [axis])), 0, axis)


def _params(shape, a, b):
    d = len(shape)
    a = tuple(float(v) for v in np.broadcast_to(np.asarray(a, dtype=np.float64), (d,)))
    b = tuple(float(v) for v in np.broadcast_to(np.asarray(b, dtype=np.float64), (d,)))
    return a, b


def forward(coeffs: np.ndarray, a, b) -> np.ndarray:
    """Weighted values (W_0 (x) ... (x) W_{d-1}) f = (Phi_0 (x) ... (x) Phi_{d-1}) coeffs.

    coeffs: float64 array, C-order, shape (n_0, ..., n_{d-1}), axis i uses (a[i], b[i])
    (reading R5/R7).  Axis i's coefficient index is the degree, the value index the node.
    Separable mode products (the Kronecker identity of eq:TJ / eq:TJ3).
    """
    X = np.asarray(coeffs, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    for ax in range(X.ndim):
        X = _mode_product(phi(X.shape[ax], a[ax], b[ax]), X, ax)
    return np.ascontiguousarray(X)


def inverse(values: np.ndarray, a, b) -> np.ndarray:
    """Coefficients = (Phi_0^T (x) ... (x) Phi_{d-1}^T) values (eq:oneJinv, eq:invTJ, eq:invTJ3)."""
    X = np.asarray(values, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    for ax in range(X.ndim):
        X = _mode_product(phi(X.shape[ax], a[ax], b[ax]).T, X, ax)
    return np.ascontiguousarray(X)


def forward_axes(coeffs: np.ndarray, a, b, axes, points=None, kind: int = 0) -> np.ndarray:
    """Apply the axis matrices along the listed axes only (bench's bounded CPU samples; slab host tests).
    points / kind as in `forward_ex` (default: the uniform first-kind Phi)."""
    X = np.asarray(coeffs, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    for ax in axes:
        pts = None if points is None else points[ax]
        M = phi(X.shape[ax], a[ax], b[ax]) if (pts is None and kind == 0) else axis_matrix(X.shape[ax], a[ax], b[ax],
                                                                                            pts, kind)
        X = _mode_product(M, X, ax)
    return np.ascontiguousarray(X)


def forward_at(coeffs: np.ndarray, a, b, idx: np.ndarray, full_shape=None) -> np.ndarray:
    """Forward-transform values at the multi-indices `idx` (k x d), one by one.

    Y[i_0..i_{d-1}] = sum_{k_0..k_{d-1}} Phi_0[i_0,k_0] ... Phi_{d-1}[i_{d-1},k_{d-1}] coeffs[k_0..]
    (eq:2Djac / eq:3Djac as a single sum), evaluated by contracting the last axis first.
    """
    X = np.asarray(coeffs, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    mats = [phi(X.shape[ax], a[ax], b[ax]) for ax in range(X.ndim)]
    out = np.empty(len(idx), dtype=np.float64)
    for s, ii in enumerate(np.asarray(idx)):
        v = X
        for ax in range(X.ndim - 1, -1, -1):
            v = v @ mats[ax][ii[ax]]
        out[s] = v
    return out


def inverse_at(values: np.ndarray, a, b, idx: np.ndarray) -> np.ndarray:
    """Inverse-transform coefficients at the multi-indices `idx` (transpose of forward_at)."""
    X = np.asarray(values, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    mats = [phi(X.shape[ax], a[ax], b[ax]) for ax in range(X.ndim)]
    out = np.empty(len(idx), dtype=np.float64)
    for s, kk in enumerate(np.asarray(idx)):
        v = X
        for ax in range(X.ndim - 1, -1, -1):
            v = v @ mats[ax][:, kk[ax]]
        out[s] = v
    return out


def kron_matrix(shape, a, b) -> np.ndarray:
    """The literal (prod n) x (prod n) Kronecker matrix Phi_0 (x) ... (x) Phi_{d-1} (small sizes).

    vec in C-order, so forward(coeffs).ravel() == kron_matrix(...) @ coeffs.ravel().
    """
    a, b = _params(shape, a, b)
    K = np.ones((1, 1))
    for ax, n in enumerate(shape):
        K = np.kron(K, phi(int(n), a[ax], b[ax]))
    return K


# ---------------------------------------------------------------------------------------------------
# SURVEY.md §8(f) NEXT-1 (nonuniform forward) and NEXT-3 (second-kind Q~ transforms): the same plain
# definitions at arbitrary angles.  PAPER.md:491 ("the nonuniform forward Jacobi transform does not require
# trigonometric Gauss-Jacobi quadrature nodes and weights": the matrix is J itself, W = I), PAPER.md:457 and
# 646 ("the transform for Q~ is similar"), eq:modifiedjac / eq:modifiedjac2.
# ---------------------------------------------------------------------------------------------------
def _trig_scale(t, a: float, b: float):
    """sqrt(2^{a+b+1}) sin(t/2)^{a+1/2} cos(t/2)^{b+1/2} in longdouble (eq:modifiedjac)."""
    t = np.asarray(t, dtype=LD)
    aa, bb = _ld(a), _ld(b)
    return np.sqrt(LD(2) ** (aa + bb + 1)) * np.sin(t / 2) ** (aa + LD(0.5)) * np.cos(t / 2) ** (bb + LD(0.5))


def cauchy_h0(t, a: float, b: float):
    """H_0(x) = PV int_{-1}^{1} w(y) / (x - y) dy, w(y) = (1-y)^a (1+y)^b, x = cos t, for each angle (float64
    array in, longdouble out).  The principal value written as the plain integral of (w(y) - w(x))/(x - y)
    (a removable singularity at y = x) plus w(x) log((1+x)/(1-x)), by mpmath tanh-sinh quadrature at 60 digits
    split at y = x, in the variables 1 + y and 1 - y (exact near the singular ends).  (reading R8; the definition of the second-kind functions via the Cauchy
    transform.)"""
    out = np.empty(len(t), dtype=LD)
    with mpmath.workdps(60):  # 60 digits: the (w(y) - w(x)) / (x - y) cancellation at nodes next to y = x
        A, B = mpmath.mpf(a), mpmath.mpf(b)
        for j, tj in enumerate(np.asarray(t, dtype=np.float64)):
            th = mpmath.mpf(float(tj))
            omx = 2 * mpmath.sin(th / 2) ** 2      # 1 - x, no cancellation
            opx = 2 * mpmath.cos(th / 2) ** 2      # 1 + x
            x = 1 - omx
            wx = omx ** A * opx ** B

            # substitute s = 1 + y on [-1, x] and s = 1 - y on [x, 1] so that the endpoint factors (1 +- y)
            # are the quadrature variable itself (exact near the singular ends of w)
            def f_lo(s_):  # y = -1 + s
                return ((2 - s_) ** A * s_ ** B - wx) / (opx - s_)

            def f_hi(s_):  # y = 1 - s
                return (s_ ** A * (2 - s_) ** B - wx) / (s_ - omx)

            def integral(f, e, c):
                # int_0^c f(s) ds with f ~ s^e at 0: for e < 0 substitute s = u^p, p = 1/(1+e), which makes the
                # integrand bounded (a truncated tanh-sinh tail of s^e would cost c_min^{1+e}, ~1e-6 at e = -0.9)
                if e >= 0:
                    return mpmath.quad(f, [0, c])
                p_ = 1 / (1 + e)
                return mpmath.quad(lambda u: f(u ** p_) * p_ * u ** (p_ - 1), [0, c ** (1 + e)])
            v = integral(f_lo, B, opx) + integral(f_hi, A, omx) + wx * mpmath.log(opx / omx)
            out[j] = _ld(v)
    return out


def modified_q_all(t, kmax: int, a: float, b: float):
    """Q~_k(t) for k = 0..kmax (rows) at the angles t (columns), longdouble, by the definition of reading R8:
        Q~_k(t) = -sqrt(sin t / w(x)) H_k(x) / pi,  H_k(x) = PV int w(y) p_k(y) / (x - y) dy,
    with H_0 from `cauchy_h0` and the three-term recurrence of the p_k carried over to H_k: for k >= 1,
    H_{k+1} = ((x - alpha_k) H_k - beta_k H_{k-1}) / beta_{k+1}, and H_1 = ((x - alpha_0) H_0 - sqrt(mu0)) / beta_1
    (the k = 0 moment term: int w p_0 = sqrt(mu0); it vanishes for k >= 1 by orthogonality)."""
    t = np.asarray(t, dtype=LD)
    alpha, beta = recurrence_coefficients(kmax + 1, a, b)
    H = np.zeros((kmax + 1,) + t.shape, dtype=LD)
    H[0] = cauchy_h0(t.astype(np.float64), a, b) / np.sqrt(mu0(a, b))   # H for p_0 = mu0^{-1/2}
    x_minus = _x_minus_alpha_factory(t)
    if kmax >= 1:
        H[1] = (x_minus(alpha[0]) * H[0] - np.sqrt(mu0(a, b))) / beta[1]
    for k in range(1, kmax):
        H[k + 1] = (x_minus(alpha[k]) * H[k] - beta[k] * H[k - 1]) / beta[k + 1]
    aa, bb = _ld(a), _ld(b)
    w = (2 * np.sin(t / 2) ** 2) ** aa * (2 * np.cos(t / 2) ** 2) ** bb
    return -np.sqrt(np.sin(t) / w) * H / LD(np.pi)


def phi_points(t, n: int, a: float, b: float, kind: int = 0) -> np.ndarray:
    """The m x n matrix J[j, k] = P~_k(t_j) (kind 0) or Q~_k(t_j) (kind 1) at arbitrary angles t_j in (0, pi)
    (unweighted: the nonuniform transform's matrix).  longdouble entries rounded once."""
    t = np.asarray(t, dtype=np.float64)
    if kind == 0:
        M = (_trig_scale(t, a, b)[None, :] * p_all(t, n - 1, a, b)).T
    else:
        M = modified_q_all(t, n - 1, a, b).T
    return np.ascontiguousarray(M.astype(np.float64))


@functools.lru_cache(maxsize=32)
def phi_q_uniform(n: int, a: float, b: float) -> np.ndarray:
    """Uniform second-kind matrix sqrt(w_j) Q~_k(t_j) at the Gauss-Jacobi nodes (rows weighted as W J_n)."""
    t, _, w = gauss_jacobi(n, a, b)
    M = np.sqrt(w)[:, None] * modified_q_all(t, n - 1, a, b).T
    out = np.ascontiguousarray(M.astype(np.float64))
    out.setflags(write=False)
    return out


def axis_matrix(n: int, a: float, b: float, points=None, kind: int = 0) -> np.ndarray:
    """Axis matrix of a plan: uniform weighted (points None) or nonuniform unweighted; first or second kind."""
    if points is None:
        return phi(n, a, b) if kind == 0 else phi_q_uniform(n, a, b)
    return phi_points(points, n, a, b, kind)


def forward_ex(coeffs: np.ndarray, a, b, points=None, kind: int = 0) -> np.ndarray:
    """values = (M_0 (x) ... (x) M_{d-1}) coeffs with the per-axis matrices of `axis_matrix`
    (points: None, or one entry per axis, None = uniform)."""
    X = np.asarray(coeffs, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    for ax in range(X.ndim):
        pts = None if points is None else points[ax]
        X = _mode_product(axis_matrix(X.shape[ax], a[ax], b[ax], pts, kind), X, ax)
    return np.ascontiguousarray(X)


def adjoint_ex(values: np.ndarray, a, b, points=None, kind: int = 0) -> np.ndarray:
    """coeffs = (M_0^T (x) ... (x) M_{d-1}^T) values (the transpose; the inverse only when orthogonal)."""
    X = np.asarray(values, dtype=np.float64)
    a, b = _params(X.shape, a, b)
    for ax in range(X.ndim):
        pts = None if points is None else points[ax]
        X = _mode_product(axis_matrix(X.shape[ax], a[ax], b[ax], pts, kind).T, X, ax)
    return np.ascontiguousarray(X)
