"""SURVEY.md §8(f) NEXT-1 (nonuniform forward transform) and NEXT-3 (second-kind Q~ transforms), CPU part.

* The oracle's new definitions (oracle.phi_points, oracle.modified_q_all, oracle.phi_q_uniform) are pinned
  against things other than themselves: trigonometric closed forms (a = b = -1/2, 1/2), scipy's Legendre
  and Jacobi polynomials, mpmath's Ferrers Q and Szego's hypergeometric second-kind function, the uniform
  oracle at the Gauss-Jacobi nodes, and the Wronskian (2k + a + b + 1)/pi of P~ and Q~ (reading R9).
* The host plan's factored operator for nonuniform / second-kind plans (numpy FFT apply of the plan's
  factors, as in tests/test_plan.py) is checked against those oracles to ~eps.
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.special as sp

import oracle
import paper_1901_07275_b200 as jt
from test_plan import fast_apply_np, fast_apply_T_np

T_EDGE = np.array([2e-4, 1e-2, 0.3, 1.2, 1.5707, 2.5, 3.1, 3.1414])


# ---------------------------------------------------------------------------------------------------
# oracle pins: P~ at arbitrary angles
# ---------------------------------------------------------------------------------------------------
def test_phi_points_chebyshev_closed_forms():
    k = np.arange(40)
    M = oracle.phi_points(T_EDGE, 40, -0.5, -0.5)
    np.testing.assert_allclose(M[:, 1:], np.sqrt(2 / np.pi) * np.cos(np.outer(T_EDGE, k[1:])), atol=2e-14)
    np.testing.assert_allclose(M[:, 0], 1 / np.sqrt(np.pi), atol=1e-15)
    M = oracle.phi_points(T_EDGE, 40, 0.5, 0.5)
    np.testing.assert_allclose(M, np.sqrt(2 / np.pi) * np.sin(np.outer(T_EDGE, k + 1)), atol=2e-14)


@pytest.mark.parametrize("a,b", [(0.0, 0.0), (0.25, -0.3), (-0.75, 0.6), (0.9, 0.2)])
def test_phi_points_scipy_jacobi(a, b):
    """P~_k(t) = sqrt(2^{a+b+1}) P_k^{(a,b)}(cos t) / sqrt(h_k) sin(t/2)^{a+1/2} cos(t/2)^{b+1/2} (eq:modifiedjac,
    eq:C PAPER.md:111-128), with scipy's eval_jacobi and the closed-form norm h_k."""
    n = 30
    M = oracle.phi_points(T_EDGE, n, a, b)
    k = np.arange(n)
    lh = ((a + b + 1) * math.log(2) - np.log(2 * k + a + b + 1) + sp.gammaln(k + a + 1) + sp.gammaln(k + b + 1)
          - sp.gammaln(k + a + b + 1) - sp.gammaln(k + 1))
    lh[0] = (a + b + 1) * math.log(2) + sp.gammaln(a + 1) + sp.gammaln(b + 1) - sp.gammaln(a + b + 2)
    scale = math.sqrt(2 ** (a + b + 1)) * np.sin(T_EDGE / 2) ** (a + 0.5) * np.cos(T_EDGE / 2) ** (b + 0.5)
    ref = scale[:, None] * sp.eval_jacobi(k[None, :], a, b, np.cos(T_EDGE)[:, None]) * np.exp(-0.5 * lh)[None, :]
    np.testing.assert_allclose(M, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("n,a,b", [(16, 0.25, -0.3), (100, -0.6, 0.45), (257, 0.1, 0.9)])
def test_phi_points_at_gauss_nodes_is_uniform_unweighted(n, a, b):
    """At the Gauss-Jacobi nodes the nonuniform matrix times sqrt(w_j) is the uniform W J_n."""
    t, _, w = oracle.gauss_jacobi(n, a, b)
    M = oracle.phi_points(t.astype(np.float64), n, a, b)
    np.testing.assert_allclose(np.sqrt(w.astype(np.float64))[:, None] * M, oracle.phi(n, a, b), atol=5e-14)


# ---------------------------------------------------------------------------------------------------
# oracle pins: Q~
# ---------------------------------------------------------------------------------------------------
def test_q_chebyshev_closed_forms():
    k = np.arange(41)
    Q = oracle.modified_q_all(T_EDGE, 40, -0.5, -0.5).astype(np.float64).T
    np.testing.assert_allclose(Q[:, 1:], np.sqrt(2 / np.pi) * np.sin(np.outer(T_EDGE, k[1:])), atol=2e-14)
    np.testing.assert_allclose(Q[:, 0], 0, atol=1e-15)
    Q = oracle.modified_q_all(T_EDGE, 40, 0.5, 0.5).astype(np.float64).T
    np.testing.assert_allclose(Q, -np.sqrt(2 / np.pi) * np.cos(np.outer(T_EDGE, k + 1)), atol=2e-14)


def test_q_legendre_ferrers():
    """a = b = 0: Q~_k(t) = -(2/pi) sqrt(sin t) sqrt((2k+1)/2) Q_k(cos t), Ferrers' Q_k from mpmath.legenq."""
    Q = oracle.modified_q_all(T_EDGE, 40, 0.0, 0.0).astype(np.float64).T
    mpmath.mp.dps = 30
    for i, ti in enumerate(T_EDGE):
        x = mpmath.cos(mpmath.mpf(ti))
        st = mpmath.sqrt(mpmath.sin(mpmath.mpf(ti)))
        for k in [0, 1, 3, 17, 40]:
            ref = float(-2 / mpmath.pi * st * mpmath.sqrt(mpmath.mpf(2 * k + 1) / 2) * mpmath.legenq(k, 0, x, type=2))
            assert abs(Q[i, k] - ref) <= 2e-14 * max(1.0, abs(ref)), (ti, k, Q[i, k], ref)


@pytest.mark.parametrize("a,b,tol", [(0.45, -0.45, 1e-13), (-0.75, 0.3, 1e-13), (0.9, -0.9, 2e-12)])
def test_q_hypergeometric(a, b, tol):
    """General (a,b): Szego's Q_k^{(a,b)} through mpmath.hyp2f1 at z = x + 1e-45 i (see tests/test_plan.py)."""
    mpmath.mp.dps = 50
    A, B = mpmath.mpf(a), mpmath.mpf(b)

    def h_k(k):
        if k == 0:
            return 2 ** (A + B + 1) * mpmath.gamma(A + 1) * mpmath.gamma(B + 1) / mpmath.gamma(A + B + 2)
        return (2 ** (A + B + 1) / (2 * k + A + B + 1) * mpmath.gamma(k + A + 1) * mpmath.gamma(k + B + 1)
                / (mpmath.gamma(k + A + B + 1) * mpmath.gamma(k + 1)))

    def cauchy(k, x):
        z = mpmath.mpc(x, mpmath.mpf("1e-45"))
        Qk = (2 ** (k + A + B) * mpmath.gamma(k + A + 1) * mpmath.gamma(k + B + 1) / mpmath.gamma(2 * k + A + B + 2)
              * (z - 1) ** (-k - A - 1) * (z + 1) ** (-B) * mpmath.hyp2f1(k + 1, k + A + 1, 2 * k + A + B + 2, 2 / (1 - z)))
        return mpmath.re(2 * (z - 1) ** A * (z + 1) ** B * Qk / mpmath.sqrt(h_k(k)))

    ts = np.array([1e-3, 0.7, 2.2, 3.14])
    Q = oracle.modified_q_all(ts, 12, a, b).astype(np.float64).T
    for i, ti in enumerate(ts):
        T = mpmath.mpf(ti)
        x = mpmath.cos(T)
        w = (1 - x) ** A * (1 + x) ** B
        for k in [0, 1, 4, 12]:
            ref = float(-mpmath.sqrt(mpmath.sin(T) / w) * cauchy(k, x) / mpmath.pi)
            assert abs(Q[i, k] - ref) <= tol * max(1.0, abs(ref)), (ti, k, Q[i, k], ref)


@pytest.mark.parametrize("a,b", [(0.3, -0.2), (-0.6, 0.1)])
def test_q_wronskian(a, b):
    """P~ Q~' - P~' Q~ = (2k+a+b+1)/pi > 0 (reading R9), central differences of the oracle."""
    h = 1e-5
    t = np.array([0.2, 1.1, 2.8])
    n = 25
    P0, Q0 = oracle.phi_points(t, n, a, b), oracle.phi_points(t, n, a, b, kind=1)
    Pp, Qp = oracle.phi_points(t + h, n, a, b), oracle.phi_points(t + h, n, a, b, kind=1)
    Pm, Qm = oracle.phi_points(t - h, n, a, b), oracle.phi_points(t - h, n, a, b, kind=1)
    W = P0 * (Qp - Qm) / (2 * h) - (Pp - Pm) / (2 * h) * Q0
    np.testing.assert_allclose(W, np.broadcast_to((2 * np.arange(n) + a + b + 1) / np.pi, W.shape), rtol=1e-6)


def test_q_uniform_weighted_rows():
    n, a, b = 24, 0.2, -0.35
    t, _, w = oracle.gauss_jacobi(n, a, b)
    np.testing.assert_allclose(oracle.phi_q_uniform(n, a, b),
                               np.sqrt(w.astype(np.float64))[:, None] * oracle.phi_points(t.astype(np.float64), n, a, b, 1),
                               atol=1e-14)


# ---------------------------------------------------------------------------------------------------
# host plan: nonuniform and second-kind factorisations against the oracle
# ---------------------------------------------------------------------------------------------------
def random_points(n, seed, clustered=False):
    rng = np.random.default_rng(seed)
    u = np.sort(rng.uniform(0, 1, n))
    if clustered:  # 4x denser than uniform at both ends: t(u) = pi (u - 0.12 sin(2 pi u))
        return np.pi * (u - 0.12 * np.sin(2 * np.pi * u)) * (1 - 2e-6) + 1e-6
    return np.pi * u * (1 - 2e-6) + 1e-6


@pytest.mark.parametrize("n,a,b,clustered", [(64, 0.25, -0.3, False), (300, 0.4, 0.4, False), (512, -0.6, 0.2, True),
                                             (1000, 0.0, 0.0, True), (40, 0.9, -0.9, False)])
def test_nonuniform_plan_vs_oracle(n, a, b, clustered):
    t = random_points(n, n, clustered)
    p = jt.Plan(n, a, b, 1e-12, device=-2, points=[t])
    assert p.kind() == (False, 0)
    tt, w = p.nodes()
    np.testing.assert_array_equal(tt, t)
    np.testing.assert_array_equal(w, np.ones(n))
    M = oracle.phi_points(t, n, a, b)
    rng = np.random.default_rng(1)
    alpha = rng.standard_normal(n)
    ref = M @ alpha
    assert np.linalg.norm(fast_apply_np(p, alpha) - ref) / np.linalg.norm(ref) <= 1e-11
    z = rng.standard_normal(n)
    ref_t = M.T @ z
    assert np.linalg.norm(fast_apply_T_np(p, z) - ref_t) / np.linalg.norm(ref_t) <= 1e-11


@pytest.mark.parametrize("n,a,b", [(48, 0.25, -0.3), (96, -0.4, 0.1)])
def test_second_kind_plan_vs_oracle(n, a, b):
    p = jt.Plan(n, a, b, 1e-12, device=-2, kind=jt.JT_KIND_Q)
    assert p.kind() == (True, 1)
    M = oracle.phi_q_uniform(n, a, b)
    alpha = np.random.default_rng(2).standard_normal(n)
    ref = M @ alpha
    assert np.linalg.norm(fast_apply_np(p, alpha) - ref) / np.linalg.norm(ref) <= 1e-11
    t = random_points(n, 7)
    q = jt.Plan(n, a, b, 1e-12, device=-2, points=[t], kind=jt.JT_KIND_Q)
    M = oracle.phi_points(t, n, a, b, kind=1)
    ref = M @ alpha
    assert np.linalg.norm(fast_apply_np(q, alpha) - ref) / np.linalg.norm(ref) <= 1e-11


def test_nonuniform_plan_argument_errors():
    with pytest.raises(jt.JTError) as ei:
        jt.Plan(8, 0.1, 0.1, 1e-12, device=-2, points=[np.linspace(0.5, 0.1, 8)])  # decreasing
    assert ei.value.status == jt.JT_ERR_ARG
    with pytest.raises(jt.JTError) as ei:
        jt.Plan(8, 0.1, 0.1, 1e-12, device=-2, points=[np.linspace(0.0, 1.0, 8)])  # t = 0 not in (0, pi)
    assert ei.value.status == jt.JT_ERR_ARG
    with pytest.raises(jt.JTError) as ei:
        jt.Plan(64, 0.1, 0.1, 1e-12, device=-2, points=[np.full(64, 1.0)])  # 64 points in one bin
    assert ei.value.status == jt.JT_ERR_NUMERIC


def test_random_points_take_the_cap3_bins():
    """Uniformly random points (the NEXT-1 bench config's recipe): the plan's spreading finds a cap-3 assignment
    (the kernels' MAXR = 3 instantiation) at the natural FFT length where one exists within 2 bins, bins non-decreasing, every point at most 2 bins
    right of its rounded bin (reading R21)."""
    import seeded_inputs as si
    caps = []
    for i in range(3):
        t = si.points(256, 100 + i)
        p = jt.Plan(256, 0.4, 0.4, 1e-12, device=-2, points=[t])
        _, _, _, bins = p.factors()
        N = p.info()["N"]
        disp = bins - np.rint(t * N / (2 * np.pi))
        assert N == 256 and np.all(np.diff(bins) >= 0)
        caps.append(int(np.bincount(bins).max()))
        assert np.min(disp) >= 0 and np.max(disp) <= 2
        p.close()
    assert caps == [3, 4, 3]  # axis 1's points have a run that fits 3 per bin only beyond 2 bins: cap 4 there


def test_clustered_points_spread_over_bins():
    """Clustered points: at most 4 rows per FFT bin, bins non-decreasing, and no point more than 2 bins from
    its rounded bin [t_j N / 2 pi] (the spreading of DESIGN.md reading R21)."""
    n = 512
    t = random_points(n, 3, clustered=True)
    p = jt.Plan(n, 0.2, 0.2, 1e-12, device=-2, points=[t])
    _, _, _, bins = p.factors()
    N = p.info()["N"]
    assert np.all(np.diff(bins) >= 0)
    assert np.bincount(bins).max() <= 4
    assert np.max(np.abs(bins - np.rint(t * N / (2 * np.pi)))) <= 2


# ---------------------------------------------------------------------------------------------------
# oracle pins: the composed nonuniform / second-kind transforms (forward_ex, adjoint_ex, forward_axes)
# ---------------------------------------------------------------------------------------------------
def _cheb_matrix(t, n, kind):
    """a = b = -1/2 closed forms: P~_k(t) = sqrt(2/pi) cos(k t) (k >= 1), 1/sqrt(pi) (k = 0); Q~_k(t) =
    sqrt(2/pi) sin(k t) (pinned above against the oracle's own P~ / Q~ generators)."""
    k = np.arange(n)
    if kind == 0:
        M = np.sqrt(2 / np.pi) * np.cos(np.outer(t, k))
        M[:, 0] = 1 / np.sqrt(np.pi)
    else:
        M = np.sqrt(2 / np.pi) * np.sin(np.outer(t, k))
    return M


@pytest.mark.parametrize("kind", [0, 1])
def test_forward_ex_literal_double_sum(kind):
    """forward_ex / adjoint_ex at random angles (values f(t_i, s_j) = sum_{k,l}
    J_k(t_i) J_l(s_j) alpha_{kl}) against the literal double sum of the closed-form entries."""
    rng = np.random.default_rng(11)
    n0, n1 = 7, 9
    t0, t1 = np.sort(rng.uniform(0.01, np.pi - 0.01, n0)), np.sort(rng.uniform(0.01, np.pi - 0.01, n1))
    A, B = _cheb_matrix(t0, n0, kind), _cheb_matrix(t1, n1, kind)
    x = rng.standard_normal((n0, n1))
    ref = np.zeros((n0, n1))
    for i in range(n0):
        for j in range(n1):
            ref[i, j] = sum(A[i, k] * B[j, l] * x[k, l] for k in range(n0) for l in range(n1))
    ab = (-0.5, -0.5)
    np.testing.assert_allclose(oracle.forward_ex(x, ab, ab, [t0, t1], kind), ref, atol=1e-13)
    refT = np.zeros((n0, n1))
    for k in range(n0):
        for l in range(n1):
            refT[k, l] = sum(A[i, k] * B[j, l] * x[i, j] for i in range(n0) for j in range(n1))
    np.testing.assert_allclose(oracle.adjoint_ex(x, ab, ab, [t0, t1], kind), refT, atol=1e-13)


def test_forward_ex_second_kind_uniform_is_a_sine_transform():
    """Uniform second kind at a = b = -1/2: nodes t_j = (2j+1) pi / (2n), w_j = pi / n, so the weighted matrix is
    sqrt(2/n) sin(k t_j) -- for k = 1..n-1 the orthonormal DST-II basis (scipy DST-III of the shifted vector)."""
    import scipy.fft as sfft
    n = 12
    x = np.random.default_rng(3).standard_normal(n)
    x[0] = 0.0  # Q~_0 = 0: the k = 0 column is zero
    got = oracle.forward_ex(x, (-0.5,), (-0.5,), None, 1)
    # sum_{k=1}^{n-1} sqrt(2/n) sin(pi k (2j+1) / (2n)) x_k = DST-III (orthonormal) of (x_1, ..., x_{n-1}, 0)
    y = np.append(x[1:], 0.0)
    np.testing.assert_allclose(got, sfft.dst(y, type=3, norm="ortho"), atol=1e-13)


@pytest.mark.parametrize("kind", [0, 1])
def test_adjoint_ex_is_the_transpose(kind):
    """<forward_ex(x), y> = <x, adjoint_ex(y)> for general (a, b), 3D, mixed uniform / nonuniform axes."""
    rng = np.random.default_rng(17)
    shape = (6, 5, 7)
    a, b = (0.3, -0.6, 0.1), (-0.2, 0.45, 0.7)
    pts = [np.sort(rng.uniform(0.05, 3.0, 6)), None, np.sort(rng.uniform(0.05, 3.0, 7))]
    x, y = rng.standard_normal(shape), rng.standard_normal(shape)
    lhs = float(np.sum(oracle.forward_ex(x, a, b, pts, kind) * y))
    rhs = float(np.sum(x * oracle.adjoint_ex(y, a, b, pts, kind)))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_forward_axes_composes_to_the_full_transform():
    """Axis passes in any order and grouping give the full transform (the operator is a Kronecker product)."""
    rng = np.random.default_rng(19)
    shape, a, b = (5, 6, 4), (0.2, -0.3, 0.5), (0.1, 0.4, -0.6)
    x = rng.standard_normal(shape)
    full = oracle.forward(x, a, b)
    np.testing.assert_allclose(oracle.forward_axes(oracle.forward_axes(x, a, b, [2]), a, b, [0, 1]), full, atol=1e-14)
    np.testing.assert_allclose(oracle.forward_axes(x, a, b, [1, 0, 2]), full, atol=1e-14)
