"""Pins for the CPU oracle (oracle/jacobi.py) against things other than itself.

Each test names the passage / closed form it pins.  None of them re-types the
oracle's own formula: they use scipy's DCT/DST, gamma-function closed forms,
Beta-function moments and 40-digit mpmath (hypergeometric Jacobi values and an
independent Golub-Welsch eigen-solve).  All CPU-only (-m "not gpu").
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.fft as sfft

import oracle

PAIRS = [(0.25, -0.3), (0.1, -0.4), (-0.25, 0.35), (0.45, -0.45), (0.0, 0.0), (0.2, -0.2),
         (-0.4, 0.3), (0.35, 0.1), (0.25, -0.25), (-0.75, -0.75), (0.75, 0.9), (-0.9, 0.6)]


# ---------------------------------------------------------------------------------------------
# Textbook reductions (SURVEY.md §8(c) "What pins each part"): a=b=-1/2 is the Chebyshev
# (first kind) case -> Phi = orthonormal DCT-III, Phi^T = DCT-II; a=b=+1/2 is Chebyshev second
# kind -> Phi = orthonormal DST-I.  A dropped sqrt(weight), a wrong node order, a sign or a
# transposed Phi fails these.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 7, 64, 300])
def test_chebyshev_first_kind_is_dct(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n)
    P = oracle.phi(n, -0.5, -0.5)
    np.testing.assert_allclose(P @ x, sfft.dct(x, type=3, norm="ortho"), atol=2e-14 * math.sqrt(n), rtol=0)
    np.testing.assert_allclose(P.T @ x, sfft.dct(x, type=2, norm="ortho"), atol=2e-14 * math.sqrt(n), rtol=0)
    t, lam, w = oracle.gauss_jacobi(n, -0.5, -0.5)
    j = np.arange(n)
    np.testing.assert_allclose(t.astype(float), (2 * j + 1) * np.pi / (2 * n), rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(lam.astype(float), np.pi / n, rtol=1e-14)
    np.testing.assert_allclose(w.astype(float), np.pi / n, rtol=1e-14)


@pytest.mark.parametrize("n", [1, 3, 16, 129])
def test_chebyshev_second_kind_is_dst1(n):
    rng = np.random.default_rng(100 + n)
    x = rng.standard_normal(n)
    P = oracle.phi(n, 0.5, 0.5)
    np.testing.assert_allclose(P @ x, sfft.dst(x, type=1, norm="ortho"), atol=2e-14 * math.sqrt(n), rtol=0)
    t, _, _ = oracle.gauss_jacobi(n, 0.5, 0.5)
    np.testing.assert_allclose(t.astype(float), np.arange(1, n + 1) * np.pi / (n + 1), rtol=1e-15)


def test_axis_association_2d_3d():
    """Axis i uses (a[i], b[i]) and C-order (readings R5/R7): mixed DCT-III / DST-I per axis."""
    rng = np.random.default_rng(7)
    X = rng.standard_normal((7, 12))
    Y = oracle.forward(X, a=(-0.5, 0.5), b=(-0.5, 0.5))
    ref = sfft.dst(sfft.dct(X, type=3, norm="ortho", axis=0), type=1, norm="ortho", axis=1)
    np.testing.assert_allclose(Y, ref, atol=1e-13, rtol=0)
    Z = oracle.inverse(Y, a=(-0.5, 0.5), b=(-0.5, 0.5))
    np.testing.assert_allclose(Z, X, atol=1e-13, rtol=0)
    X3 = rng.standard_normal((5, 6, 9))
    Y3 = oracle.forward(X3, a=(0.5, -0.5, -0.5), b=(0.5, -0.5, -0.5))
    ref3 = sfft.dst(X3, type=1, norm="ortho", axis=0)
    ref3 = sfft.dct(sfft.dct(ref3, type=3, norm="ortho", axis=1), type=3, norm="ortho", axis=2)
    np.testing.assert_allclose(Y3, ref3, atol=1e-13, rtol=0)
    inv3 = sfft.dct(sfft.dct(sfft.dst(Y3, type=1, norm="ortho", axis=0), type=2, norm="ortho", axis=1),
                    type=2, norm="ortho", axis=2)
    np.testing.assert_allclose(oracle.inverse(Y3, a=(0.5, -0.5, -0.5), b=(0.5, -0.5, -0.5)), inv3, atol=1e-13)


# ---------------------------------------------------------------------------------------------
# Endpoint closed forms: P_k^{(a,b)}(1) = Gamma(k+a+1)/(Gamma(k+1)Gamma(a+1)),
# P_k^{(a,b)}(-1) = (-1)^k Gamma(k+b+1)/(Gamma(k+1)Gamma(b+1)), norm h_k.  Pins the recurrence
# coefficients alpha_k, beta_k, p_0 = mu_0^{-1/2} and the t-form of x - alpha_k (t = 0, pi).
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("a,b", [(0.0, 0.0), (0.25, -0.3), (-0.6, 0.45), (0.9, 0.2)])
def test_endpoint_values(a, b):
    K = 400
    P = oracle.p_all(np.array([0.0, np.pi]), K, a, b).astype(float)
    mpmath.mp.dps = 30
    a, b = mpmath.mpf(a), mpmath.mpf(b)  # exact binary values; no float rounding of k+a+1 etc.
    for k in [0, 1, 2, 3, 10, 57, 200, 400]:
        hk = (mpmath.power(2, a + b + 1) / (2 * k + a + b + 1) * mpmath.gamma(k + a + 1) * mpmath.gamma(k + b + 1)
              / (mpmath.gamma(k + a + b + 1) * mpmath.gamma(k + 1)))
        p1 = mpmath.gamma(k + a + 1) / (mpmath.gamma(k + 1) * mpmath.gamma(a + 1)) / mpmath.sqrt(hk)
        pm1 = (-1) ** k * mpmath.gamma(k + b + 1) / (mpmath.gamma(k + 1) * mpmath.gamma(b + 1)) / mpmath.sqrt(hk)
        assert abs(P[k, 0] - float(p1)) <= 1e-14 * abs(float(p1)), (k, P[k, 0], p1)
        assert abs(P[k, 1] - float(pm1)) <= 1e-14 * abs(float(pm1)), (k, P[k, 1], pm1)


def test_legendre_endpoints():
    """Legendre: p_k(+-1) = (+-1)^k sqrt((2k+1)/2)."""
    P = oracle.p_all(np.array([0.0, np.pi]), 1000, 0.0, 0.0).astype(float)
    k = np.arange(1001)
    np.testing.assert_allclose(P[:, 0], np.sqrt((2 * k + 1) / 2), rtol=2e-14)
    np.testing.assert_allclose(P[:, 1], (-1.0) ** k * np.sqrt((2 * k + 1) / 2), rtol=2e-14)


# ---------------------------------------------------------------------------------------------
# Quadrature exactness ("exact when p is a polynomial of degree <= 2n-1"):
# sum_j lambda_j x_j^m = int x^m (1-x)^a (1+x)^b dx, the right side from Beta functions at 50 digits.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,a,b", [(1, 0.3, -0.2), (5, 0.25, -0.3), (10, -0.75, 0.5), (12, 0.45, -0.45),
                                   (9, 0.0, 0.0)])
def test_quadrature_moments(n, a, b):
    t, lam, _ = oracle.gauss_jacobi(n, a, b)
    x = np.cos(t)
    mpmath.mp.dps = 50
    mu = float(oracle.mu0(a, b))
    a, b = mpmath.mpf(a), mpmath.mpf(b)
    for m in range(0, 2 * n):
        exact = mpmath.power(2, a + b + 1) * mpmath.fsum(
            mpmath.binomial(m, i) * mpmath.power(2, i) * (-1) ** (m - i) * mpmath.beta(b + i + 1, a + 1)
            for i in range(m + 1))
        got = np.sum(lam * x ** m)
        assert abs(float(got) - float(exact)) <= 2e-15 * mu, (m, got, exact)


# ---------------------------------------------------------------------------------------------
# Brute force, n <= 32 (north star: "brute-force high-precision sums for n <= 32"):
# 40-digit mpmath Golub-Welsch (eigsy: nodes = eigenvalues, lambda_j = mu_0 v_{0j}^2) and
# hypergeometric mpmath.jacobi values normalised by h_k.  Independent of the recurrence, the
# Newton iteration and the Christoffel sum used by the oracle.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,a,b", [(8, 0.25, -0.3), (17, -0.4, 0.3), (32, 0.45, -0.45), (32, 0.0, 0.0)])
def test_phi_bruteforce_mpmath(n, a, b):
    mpmath.mp.dps = 40
    a_ = mpmath.mpf(a)
    b_ = mpmath.mpf(b)
    A = mpmath.zeros(n, n)
    for k in range(n):
        s = 2 * k + a_ + b_
        A[k, k] = (b_ - a_) / (a_ + b_ + 2) if k == 0 else (b_ ** 2 - a_ ** 2) / (s * (s + 2))
    for k in range(1, n):
        s = 2 * k + a_ + b_
        if k == 1:
            bk2 = 4 * (1 + a_) * (1 + b_) / ((2 + a_ + b_) ** 2 * (3 + a_ + b_))
        else:
            bk2 = 4 * k * (k + a_) * (k + b_) * (k + a_ + b_) / (s ** 2 * (s + 1) * (s - 1))
        A[k, k - 1] = A[k - 1, k] = mpmath.sqrt(bk2)
    E, Q = mpmath.eigsy(A)
    mu = mpmath.power(2, a_ + b_ + 1) * mpmath.gamma(a_ + 1) * mpmath.gamma(b_ + 1) / mpmath.gamma(a_ + b_ + 2)
    order = sorted(range(n), key=lambda j: -E[j])  # t ascending <=> x descending
    # the eigenvalues are the zeros of the (hypergeometric) P_n^{(a,b)}: the matrix is right
    Pn_scale = max(abs(mpmath.jacobi(n, a_, b_, 1)), abs(mpmath.jacobi(n, a_, b_, -1)))
    assert max(abs(mpmath.jacobi(n, a_, b_, E[j])) for j in range(n)) < mpmath.mpf(10) ** -30 * Pn_scale
    Phi_ref = np.zeros((n, n))
    for jj, j in enumerate(order):
        x = E[j]
        lam = mu * Q[0, j] ** 2
        for k in range(n):
            hk = (mpmath.power(2, a_ + b_ + 1) / (2 * k + a_ + b_ + 1) * mpmath.gamma(k + a_ + 1)
                  * mpmath.gamma(k + b_ + 1) / (mpmath.gamma(k + a_ + b_ + 1) * mpmath.gamma(k + 1)))
            Phi_ref[jj, k] = float(mpmath.sqrt(lam) * mpmath.jacobi(k, a_, b_, x) / mpmath.sqrt(hk))
    np.testing.assert_allclose(oracle.phi(n, a, b), Phi_ref, atol=3e-15, rtol=0)


def test_modified_jacobi_normalisation():
    """eq:C and eq:modifiedjac with reading R2: sqrt(w_j) P~_k(t_j) == Phi[j,k],
    P~ built from mpmath.jacobi and the paper's C_nu; w_j the oracle's trigonometric weights."""
    n, a, b = 24, 0.35, -0.6
    t, _, w = oracle.gauss_jacobi(n, a, b)
    P = oracle.phi(n, a, b)
    mpmath.mp.dps = 30
    a, b = mpmath.mpf(a), mpmath.mpf(b)
    for j in [0, 5, 11, 23]:
        tj = mpmath.mpf(str(t[j]))
        for k in [0, 1, 7, 23]:
            C = mpmath.sqrt((2 * k + a + b + 1) * mpmath.gamma(1 + k) * mpmath.gamma(1 + k + a + b)
                            / (mpmath.gamma(1 + k + a) * mpmath.gamma(1 + k + b)))
            Pt = (C * mpmath.jacobi(k, a, b, mpmath.cos(tj)) * mpmath.sin(tj / 2) ** (a + 0.5)
                  * mpmath.cos(tj / 2) ** (b + 0.5))
            ref = float(mpmath.sqrt(mpmath.mpf(str(w[j]))) * Pt)
            assert abs(P[j, k] - ref) <= 1e-14, (j, k, P[j, k], ref)


def test_modified_jacobi_l2_normalised():
    """{P~_nu} is orthonormal in L^2(0, pi); spot-check nu = 0, 3 with mpmath.quad."""
    a, b = 0.25, -0.3
    mpmath.mp.dps = 20

    def Pt(k, t):
        C = mpmath.sqrt((2 * k + a + b + 1) * mpmath.gamma(1 + k) * mpmath.gamma(1 + k + a + b)
                        / (mpmath.gamma(1 + k + a) * mpmath.gamma(1 + k + b)))
        return C * mpmath.jacobi(k, a, b, mpmath.cos(t)) * mpmath.sin(t / 2) ** (a + 0.5) * mpmath.cos(t / 2) ** (b + 0.5)

    assert abs(mpmath.quad(lambda t: Pt(0, t) ** 2, [0, mpmath.pi]) - 1) < 1e-12
    assert abs(mpmath.quad(lambda t: Pt(3, t) ** 2, [0, mpmath.pi]) - 1) < 1e-12
    # and the oracle's quadrature reproduces it: sum_j w_j P~_3(t_j)^2 = sum_j Phi[j,3]^2 = 1
    P = oracle.phi(16, a, b)
    assert abs(np.sum(P[:, 3] ** 2) - 1) < 1e-14


# ---------------------------------------------------------------------------------------------
# Orthogonality of W J — north star: "discrete orthonormality of the weighted
# matrix to 1e-13".
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,a,b", [(1024, 0.25, -0.3), (256, 0.1, -0.4), (256, -0.25, 0.35), (512, 0.25, -0.25),
                                   (333, -0.9, 0.75)])
def test_orthogonality(n, a, b):
    P = oracle.phi(n, a, b)
    E = P.T @ P - np.eye(n)
    assert np.abs(E).max() <= 1e-13
    assert np.linalg.norm(E, 2) <= 1e-12


def test_orthogonality_4096():
    P = oracle.phi(4096, 0.45, -0.45)
    E = P.T @ P - np.eye(4096)
    assert np.abs(E).max() <= 1e-13
    assert np.linalg.norm(E, 2) <= 1e-12


def test_symmetric_nodes():
    t, lam, _ = oracle.gauss_jacobi(101, 0.4, 0.4)
    np.testing.assert_allclose((t + t[::-1]).astype(float), np.pi, atol=1e-15)
    np.testing.assert_allclose(lam.astype(float), lam[::-1].astype(float), rtol=1e-14)


# ---------------------------------------------------------------------------------------------
# Separable apply == literal Kronecker sum (eq:TJ PAPER.md:669-674, eq:TJ3 PAPER.md:718-722) on
# ragged shapes with a different (a, b) per axis; rank-1 inputs give outer products.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("shape", [(9, 13), (4, 6, 5), (16, 16), (8, 3, 11)])
def test_kronecker_literal(shape):
    rng = np.random.default_rng(len(shape) * 31 + shape[0])
    a = [PAIRS[i][0] for i in range(len(shape))]
    b = [PAIRS[i][1] for i in range(len(shape))]
    X = rng.standard_normal(shape)
    K = oracle.kron_matrix(shape, a, b)
    Y = oracle.forward(X, a, b)
    np.testing.assert_allclose(Y.ravel(), K @ X.ravel(), atol=1e-13, rtol=0)
    np.testing.assert_allclose(oracle.inverse(Y, a, b).ravel(), K.T @ Y.ravel(), atol=1e-13, rtol=0)
    np.testing.assert_allclose(oracle.inverse(Y, a, b), X, atol=1e-13, rtol=0)
    idx = np.array([[rng.integers(0, s) for s in shape] for _ in range(5)])
    np.testing.assert_allclose(oracle.forward_at(X, a, b, idx), Y[tuple(idx.T)], atol=1e-13)
    np.testing.assert_allclose(oracle.inverse_at(Y, a, b, idx), X[tuple(idx.T)], atol=1e-13)


def test_rank_one_separability():
    rng = np.random.default_rng(3)
    n = (20, 24, 18)
    a, b = (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)
    vs = [rng.standard_normal(m) for m in n]
    X = np.einsum("i,j,k->ijk", *vs)
    Y = oracle.forward(X, a, b)
    outs = [oracle.phi(n[i], a[i], b[i]) @ vs[i] for i in range(3)]
    np.testing.assert_allclose(Y, np.einsum("i,j,k->ijk", *outs), atol=1e-13)
