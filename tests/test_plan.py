"""CPU checks of the library's host plan (opts.device = -2, no GPU): quadrature, the low-degree block,
the bins, the non-oscillatory generator P~ + iQ~ and Algorithm 1's factors.

The factored operator is applied here with numpy's FFT (test-only code; the product path runs it in
the CUDA kernels) and compared with the oracle: this pins every plan output at once against the
independent definition, separately from the kernels.
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
import paper_1901_07275_b200 as jt
import seeded_inputs as si

CFG_PAIRS = [(0.25, -0.3), (0.1, -0.4), (-0.25, 0.35), (0.45, -0.45), (0.0, 0.0), (0.2, -0.2), (-0.4, 0.3),
             (0.35, 0.1), (0.25, -0.25)]


def fast_apply_np(plan, alpha, axis=0):
    """eq:oneJ with the plan's factors: y = phiv a_V + Re sum_l u_l (.) F_N (v_l (.) a)[m]."""
    u, v, phiv, bins = plan.factors(axis)
    n, k0 = phiv.shape
    N = v.shape[1]
    y = phiv @ alpha[:k0]
    for l in range(u.shape[1]):
        x = np.zeros(N, complex)
        x[:n] = v[l, :n] * alpha
        X = np.fft.ifft(x) * N  # positive exponent, unnormalised
        y = y + (u[:, l] * X[bins]).real
    return y


def fast_apply_T_np(plan, y, axis=0):
    """eq:oneJinv: a_V = phiv^T y, a_G = Re sum_l v_l (.) F_N^T (u_l (.) y)."""
    u, v, phiv, bins = plan.factors(axis)
    n, k0 = phiv.shape
    N = v.shape[1]
    a = np.zeros(n)
    a[:k0] = phiv.T @ y
    for l in range(u.shape[1]):
        b = np.zeros(N, complex)
        np.add.at(b, bins, u[:, l] * y)
        B = np.fft.ifft(b) * N
        a = a + (v[l, :n] * B[:n]).real
    return a


@pytest.mark.parametrize("n,a,b", [(64, 0.25, -0.3), (256, 0.1, -0.4), (1000, -0.75, 0.6), (1024, 0.25, -0.3),
                                   (4096, 0.45, -0.45)])
def test_nodes_weights_vs_oracle(n, a, b):
    p = jt.Plan(n, a, b, 1e-12, device=-2)
    t, w = p.nodes()
    to, lo, wo = oracle.gauss_jacobi(n, a, b)
    np.testing.assert_allclose(t, to.astype(float), rtol=0, atol=4e-16 * math.pi)
    np.testing.assert_allclose(w, wo.astype(float), rtol=1e-13, atol=0)
    assert np.all(np.diff(t) > 0) and t[0] > 0 and t[-1] < math.pi


@pytest.mark.parametrize("n,a,b,eps", [(64, 0.25, -0.3, 1e-12), (100, 0.3, 0.3, 1e-12), (256, 0.1, -0.4, 1e-12),
                                       (256, -0.25, 0.35, 1e-12), (300, -0.9, 0.9, 1e-12),
                                       (512, 0.25, -0.25, 1e-12), (1024, 0.25, -0.3, 1e-12),
                                       (1024, 0.25, -0.3, 1e-8), (777, 0.75, -0.75, 1e-10), (30, 0.2, 0.1, 1e-12)])
def test_factored_operator_vs_oracle(n, a, b, eps):
    """The plan's factored W J (eq:lastJ / eq:oneJ) matches the dense definition within ~eps."""
    p = jt.Plan(n, a, b, eps, device=-2)
    P = oracle.phi(n, a, b)
    rng = np.random.default_rng(n)
    alpha = rng.standard_normal(n)
    y = fast_apply_np(p, alpha)
    ref = P @ alpha
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 10 * eps
    z = rng.standard_normal(n)
    at = fast_apply_T_np(p, z)
    ref_t = P.T @ z
    assert np.linalg.norm(at - ref_t) / np.linalg.norm(ref_t) <= 10 * eps
    # low-degree block = first k0 columns of Phi
    u, v, phiv, bins = p.factors()
    np.testing.assert_allclose(phiv, P[:, :phiv.shape[1]], atol=2e-15, rtol=0)


def test_factored_operator_4096():
    p = jt.Plan(4096, 0.0, 0.0, 1e-12, device=-2)
    P = oracle.phi(4096, 0.0, 0.0)
    alpha = np.random.default_rng(5).standard_normal(4096)
    y = fast_apply_np(p, alpha)
    ref = P @ alpha
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-11


@pytest.mark.parametrize("n,a,b", [(256, 0.1, -0.4), (1000, 0.45, -0.45), (33, -0.6, 0.2)])
def test_bins(n, a, b):
    """m_j = [t_j N / 2pi] (eq:B): residual |t_j - 2 pi m_j / N| <= pi / N, so that the
    phase difference k |t_j - 2 pi m_j/N| between A and B is at most pi."""
    p = jt.Plan(n, a, b, 1e-12, device=-2)
    t, _ = p.nodes()
    _, _, _, bins = p.factors()
    N = p.info()["N"]
    assert np.all(np.diff(bins) >= 0) and bins.min() >= 0 and bins.max() <= N // 2
    assert np.max(np.abs(t - 2 * np.pi * bins / N)) <= np.pi / N * (1 + 1e-12)
    np.testing.assert_array_equal(bins, np.rint(t * N / (2 * np.pi)).astype(np.int32))


# ---------------------------------------------------------------------------------------------
# Ranks (Algorithm 1 + truncation at eps): closed-form and paper-printed pins.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [64, 256, 1024])
def test_rank_chebyshev_first_kind_is_two(n):
    """a=b=-1/2: P~ + iQ~ = sqrt(2/pi) e^{ikt} and t_j - 2 pi m_j/n = +-pi/(2n), so B has exactly two
    distinct row patterns e^{+-ik pi/2n}: rank 2 (paper Table 1 row -0.5 prints 2-4)."""
    p = jt.Plan(n, -0.5, -0.5, 1e-12, device=-2)
    assert p.rank() == 2


@pytest.mark.parametrize("n", [512, 4096])
def test_rank_chebyshev_second_kind_table1(n):
    """a=b=1/2: B_jk = -i sqrt(2/pi) e^{it_j} e^{ik(t_j - 2 pi m_j/n)}: its rank depends only on the
    distribution of k (t_j - 2 pi m_j / n) in [-pi, pi], not on n.  Table 1 prints RS rank
    9 at eps = 1e-8 for every n = 2^14..2^19."""
    p = jt.Plan(n, 0.5, 0.5, 1e-8, device=-2)
    assert 8 <= p.rank() <= 10


@pytest.mark.parametrize("a", [0.0, 0.2, -0.3, 0.4])
def test_rank_band_vs_table1(a):
    """Table 1: RS ranks 17-19 at eps=1e-8 for n = 2^14 and |a| <= 0.4, growing like
    O(log n).  At n = 4096 = 2^12 the rank must not exceed the 2^14 value and be at
    least ~2/3 of it."""
    p = jt.Plan(4096, a, a, 1e-8, device=-2)
    assert 11 <= p.rank() <= 19


def test_config_ranks_regression():
    """Ranks at eps = 1e-12, k0 = 27 for the BASELINE configs; SURVEY.md App. A measured the optimal
    (dense SVD) ranks 15 (n=256), 17 (n=512), 18 (n=1024), 21 / 22 (n=4096) independently."""
    assert jt.Plan(256, 0.1, -0.4, 1e-12, device=-2).rank() <= 16
    assert jt.Plan(512, 0.25, -0.25, 1e-12, device=-2).rank() <= 18
    assert jt.Plan(1024, 0.25, -0.3, 1e-12, device=-2).rank() <= 19


def test_plan_deterministic_given_seed():
    p1 = jt.Plan(300, 0.3, -0.1, 1e-12, device=-2, seed=7)
    p2 = jt.Plan(300, 0.3, -0.1, 1e-12, device=-2, seed=7)
    for x, y in zip(p1.factors(), p2.factors()):
        np.testing.assert_array_equal(x, y)


def test_rank_changes_little_with_seed():
    ranks = {jt.Plan(512, 0.2, -0.2, 1e-12, device=-2, seed=s).rank() for s in range(4)}
    assert max(ranks) - min(ranks) <= 1


# ---------------------------------------------------------------------------------------------
# The non-oscillatory generator P~ + iQ~ (eq:modifiedjac / eq:modifiedjac2, PAPER.md:97-122;
# DESIGN.md reading R8) by the plan's route (Cauchy transform + recurrence).
# ---------------------------------------------------------------------------------------------
def test_pq_chebyshev_closed_forms():
    t = np.array([1e-3, 0.3, 1.2, 2.5, 3.14])
    P, Q = jt.jt_debug_modified_pq(-0.5, -0.5, t, 40)
    k = np.arange(41)
    np.testing.assert_allclose(P[:, 1:], np.sqrt(2 / np.pi) * np.cos(np.outer(t, k[1:])), atol=1e-14)
    np.testing.assert_allclose(Q[:, 1:], np.sqrt(2 / np.pi) * np.sin(np.outer(t, k[1:])), atol=1e-14)
    np.testing.assert_allclose(P[:, 0], 1 / np.sqrt(np.pi), atol=1e-15)
    np.testing.assert_allclose(Q[:, 0], 0, atol=1e-15)
    P, Q = jt.jt_debug_modified_pq(0.5, 0.5, t, 40)
    th = np.outer(t, k + 1)
    np.testing.assert_allclose(P, np.sqrt(2 / np.pi) * np.sin(th), atol=1e-14)
    np.testing.assert_allclose(Q, -np.sqrt(2 / np.pi) * np.cos(th), atol=1e-14)


def test_pq_legendre_ferrers():
    """a=b=0: Q~_k(t) = -(2/pi) sqrt(sin t) sqrt((2k+1)/2) Q_k(cos t), Q_k Ferrers' second kind
    (Neumann: Q_k(x) = 1/2 PV int P_k(y)/(x-y) dy), from mpmath.legenq."""
    t = np.array([2e-4, 0.01, 0.7, 1.5707, 2.9, 3.1415])
    P, Q = jt.jt_debug_modified_pq(0.0, 0.0, t, 60)
    mpmath.mp.dps = 30
    for i, ti in enumerate(t):
        x = mpmath.cos(mpmath.mpf(ti))
        st = mpmath.sqrt(mpmath.sin(mpmath.mpf(ti)))
        for k in [0, 1, 2, 7, 27, 60]:
            c = mpmath.sqrt(mpmath.mpf(2 * k + 1) / 2)
            q_ref = -2 / mpmath.pi * st * c * mpmath.legenq(k, 0, x, type=2)
            p_ref = st * c * mpmath.legendre(k, x)
            scale = max(1.0, abs(float(q_ref)))
            assert abs(Q[i, k] - float(q_ref)) <= 2e-14 * scale, (ti, k, Q[i, k], q_ref)
            assert abs(P[i, k] - float(p_ref)) <= 2e-14, (ti, k)


@pytest.mark.parametrize("a,b", [(0.45, -0.45), (-0.75, 0.3), (0.25, -0.3), (0.9, 0.6)])
def test_pq_cauchy_transform_hypergeometric(a, b):
    """General (a,b): the Cauchy transform H_k(x) = PV int w(y) p_k(y)/(x-y) dy is the boundary value of
    2 (z-1)^a (z+1)^b Q_k^{(a,b)}(z) / sqrt(h_k), with Szego's hypergeometric Jacobi function of the
    second kind Q_k^{(a,b)}(z) = 2^{k+a+b} G(k+a+1)G(k+b+1)/G(2k+a+b+2) (z-1)^{-k-a-1}(z+1)^{-b}
    2F1(k+1, k+a+1; 2k+a+b+2; 2/(1-z)), evaluated by mpmath at z = x + 1e-35 i (50 digits); the PV is its
    real part.  Q~_k = -sqrt(sin t / w(x)) H_k(x) / pi (reading R8).  Independent of the plan's tanh-sinh
    h0 and recurrence; extreme angles included."""
    mpmath.mp.dps = 50
    A, B = mpmath.mpf(a), mpmath.mpf(b)

    def cauchy_pk(k, x):
        if k > 0:
            hk = (2 ** (A + B + 1) / (2 * k + A + B + 1) * mpmath.gamma(k + A + 1) * mpmath.gamma(k + B + 1)
                  / (mpmath.gamma(k + A + B + 1) * mpmath.gamma(k + 1)))
        else:
            hk = 2 ** (A + B + 1) * mpmath.gamma(A + 1) * mpmath.gamma(B + 1) / mpmath.gamma(A + B + 2)
        z = mpmath.mpc(x, mpmath.mpf("1e-35"))
        Qk = (2 ** (k + A + B) * mpmath.gamma(k + A + 1) * mpmath.gamma(k + B + 1) / mpmath.gamma(2 * k + A + B + 2)
              * (z - 1) ** (-k - A - 1) * (z + 1) ** (-B) * mpmath.hyp2f1(k + 1, k + A + 1, 2 * k + A + B + 2, 2 / (1 - z)))
        return mpmath.re(2 * (z - 1) ** A * (z + 1) ** B * Qk / mpmath.sqrt(hk))

    ts = [1e-4, 0.002, 1.1, 3.13, 3.1415]
    P, Q = jt.jt_debug_modified_pq(a, b, np.array(ts), 60)
    for i, ti in enumerate(ts):
        T = mpmath.mpf(ti)
        x = mpmath.cos(T)
        w = (1 - x) ** A * (1 + x) ** B
        for k in [0, 1, 2, 5, 27, 60]:
            q_ref = float(-mpmath.sqrt(mpmath.sin(T) / w) * cauchy_pk(k, x) / mpmath.pi)
            assert abs(Q[i, k] - q_ref) <= 2e-15 * max(1.0, abs(q_ref)), (ti, k, Q[i, k], q_ref)


@pytest.mark.parametrize("a,b", [(0.45, -0.45), (0.0, 0.0), (-0.4, 0.3), (0.9, -0.9)])
def test_wronskian(a, b):
    """P~ Q~' - P~' Q~ = W = (2k+a+b+1)/pi > 0 (value: reading R9), central differences."""
    h = 1e-5
    t = np.array([0.05, 0.9, 1.6, 2.7, 3.1])
    k = np.arange(41)
    P0, Q0 = jt.jt_debug_modified_pq(a, b, t, 40)
    Pp, Qp = jt.jt_debug_modified_pq(a, b, t + h, 40)
    Pm, Qm = jt.jt_debug_modified_pq(a, b, t - h, 40)
    W = P0 * (Qp - Qm) / (2 * h) - (Pp - Pm) / (2 * h) * Q0
    np.testing.assert_allclose(W, np.broadcast_to((2 * k + a + b + 1) / np.pi, W.shape), rtol=2e-6)


def test_amplitude_non_oscillatory():
    """M^2 = P~^2 + Q~^2 is non-oscillatory and tends to 2/pi in the interior for large nu (reading R9):
    M^2 psi' = W with psi' -> nu + (a+b+1)/2."""
    t = np.concatenate([np.linspace(0.3, 2.8, 50), 1.0 + 1e-4 * np.arange(100)])
    P, Q = jt.jt_debug_modified_pq(0.3, -0.2, t, 2000)
    M2 = P[:, 2000] ** 2 + Q[:, 2000] ** 2
    assert np.max(np.abs(M2 - 2 / np.pi)) < 2e-3
    M2, P = M2[50:], P[50:]  # fine grid resolving the oscillation (period 2 pi / 2000)
    # no oscillation: second differences tiny compared with those of P~^2
    assert np.max(np.abs(np.diff(M2, 2))) < 1e-3 * np.max(np.abs(np.diff(P[:, 2000] ** 2, 2)))


def test_auto_k0():
    """k0 = -1 (default, R24): the paper's 27, or 32 when that lowers the rank for FFT lengths
    <= 512, or the narrower 20 (FFT length 4096) / 24 (2048) when that keeps the rank; explicit k0 values are kept."""
    p = jt.Plan(512, 0.25, -0.25, 1e-12, device=-2)
    r27 = jt.Plan(512, 0.25, -0.25, 1e-12, device=-2, k0=27).rank()
    r32 = jt.Plan(512, 0.25, -0.25, 1e-12, device=-2, k0=32).rank()
    assert p.info()["k0"] == (32 if r32 < r27 else 27) and p.rank() == min(r27, r32)
    assert jt.Plan(1024, 0.25, -0.3, 1e-12, device=-2).info()["k0"] == 27  # FFT length 1024: the paper's 27
    for n, kn in ((2048, 24), (4096, 20)):
        p = jt.Plan(n, 0.45, -0.45, 1e-12, device=-2)
        r27 = jt.Plan(n, 0.45, -0.45, 1e-12, device=-2, k0=27).rank()
        rn = jt.Plan(n, 0.45, -0.45, 1e-12, device=-2, k0=kn).rank()
        assert p.info()["k0"] == (kn if rn <= r27 else 27) and p.rank() == min(r27, rn)
    assert jt.Plan(512, 0.25, -0.25, 1e-12, device=-2, k0=20).info()["k0"] == 20


def pair_apply_np(plan, alpha, axis=0):
    """The paired forward (include/jt_debug.h jt_debug_pair_factors): y = phiv a_V + Re sum_q (P_q (.) Z_q[m] +
    conj(Q_q) (.) Z_q[N - 1 - m]), Z_q = F_N (v_q (.) a) with numpy's FFT (test-only code; the product path runs it
    in the Cfg::PAIR kernels)."""
    u, v, phiv, bins, rreal = jt.jt_debug_pair_factors(plan.handle, axis)
    n, k0 = phiv.shape
    N = v.shape[1]
    y = phiv @ alpha[:k0]
    for q in range(v.shape[0]):
        x = np.zeros(N, complex)
        x[:n] = v[q, :n] * alpha
        Z = np.fft.ifft(x) * N
        y = y + (u[:, 2 * q] * Z[bins]).real + (u[:, 2 * q + 1] * Z[N - 1 - bins]).real
    return y


@pytest.mark.parametrize("a,b", [(0.25, -0.25), (0.1, -0.4), (-0.45, 0.45), (0.0, 0.0)])
def test_paired_factors_vs_oracle(a, b):
    """Two real rank terms per FFT (eq:oneJ, with real v'_l): the plan's second factor set
    of an N = 512 axis reproduces the oracle's matrix-vector product to the plan's eps with about half the FFTs, its v
    is a real vector times e^{i pi k / N} pairwise, and its bins are the half-integer grid (2 nodes per bin)."""
    n = 512
    p = jt.Plan(n, a, b, 1e-12, device=-2)
    got = jt.jt_debug_pair_factors(p.handle, 0)
    assert got is not None
    u, v, phiv, bins, rreal = got
    r = p.rank()
    assert v.shape[0] == (rreal + 1) // 2 and r <= rreal <= r + 2 and v.shape[0] < r
    t, _ = p.nodes()
    assert np.array_equal(bins, np.floor(t * n / (2 * np.pi)).astype(np.int32))
    assert np.bincount(bins, minlength=n // 2).max() <= 2 and bins.max() < n // 2
    k = np.arange(n)
    vr = v * np.exp(-1j * np.pi * k / n)  # (v'_{2q} + i v'_{2q+1}): both parts real vectors, zero below k0
    k0 = p.info()["k0"]
    assert np.all(vr[:, :k0] == 0)
    x = si.gaussian((n,), seed=5)
    ref = oracle.phi(n, a, b) @ x
    y = pair_apply_np(p, x)
    assert np.linalg.norm(y - ref) <= 1e-11 * np.linalg.norm(ref)
    # the unit vectors of a few degrees: column by column against the oracle's matrix
    Phi = oracle.phi(n, a, b)
    for kk in (0, k0 - 1, k0, k0 + 1, 100, n - 1):
        e = np.zeros(n)
        e[kk] = 1.0
        assert np.linalg.norm(pair_apply_np(p, e) - Phi[:, kk]) <= 2e-11 * np.linalg.norm(Phi[:, kk])
    p.close()


def test_pair_env_off(monkeypatch):
    """JT_PAIR=0 at plan time: no paired set; FFT lengths without paired kernels (1024: one last-pass butterfly per
    thread) never have one; 256 / 2048 / 4096 do (csrc/launch.cuh pair_length)."""
    monkeypatch.setenv("JT_PAIR", "0")
    p = jt.Plan(512, 0.25, -0.25, 1e-12, device=-2)
    assert jt.jt_debug_pair_factors(p.handle, 0) is None
    p.close()
    monkeypatch.delenv("JT_PAIR")
    q = jt.Plan(1024, 0.25, -0.3, 1e-12, device=-2)
    assert jt.jt_debug_pair_factors(q.handle, 0) is None
    q.close()
    for n in (256, 200, 2048):
        q = jt.Plan(n, 0.1, -0.2, 1e-12, device=-2)
        got = jt.jt_debug_pair_factors(q.handle, 0)
        assert got is not None and got[1].shape[0] < q.rank()
        x = si.gaussian((n,), seed=n)
        ref = oracle.phi(n, 0.1, -0.2) @ x
        assert np.linalg.norm(pair_apply_np(q, x) - ref) <= 1e-11 * np.linalg.norm(ref)
        q.close()


@pytest.mark.parametrize("n,a,b", [(512, -0.3, 0.6), (2048, -0.3, 0.6), (512, 0.7, 0.6)])
def test_paired_bins_spill(n, a, b):
    """(a, b) whose nodes drift across a half-integer bin boundary (a + b far from 0): a third node of a bin moves to
    the next bin (plan.cpp, pair bins); the paired set still reproduces the oracle's product, or the plan falls back
    to the unpaired set (None)."""
    p = jt.Plan(n, a, b, 1e-12, device=-2)
    got = jt.jt_debug_pair_factors(p.handle, 0)
    if got is not None:
        u, v, phiv, bins, rreal = got
        t, _ = p.nodes()
        d = bins - np.floor(t * n / (2 * np.pi)).astype(np.int32)
        assert d.min() >= 0 and d.max() <= 1 and np.all(np.diff(bins) >= 0)
        assert np.bincount(bins, minlength=n // 2).max() <= 2 and bins.max() < n // 2
        assert v.shape[0] < p.rank()
        x = si.gaussian((n,), seed=n + 1)
        ref = oracle.phi(n, a, b) @ x
        assert np.linalg.norm(pair_apply_np(p, x) - ref) <= 1e-11 * np.linalg.norm(ref)
    p.close()
