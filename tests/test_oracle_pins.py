"""Pins for the CPU oracle (oracle/fabf_oracle.c) -- CPU only, no GPU.

Each test checks an oracle routine against something other than itself: exact
rational arithmetic, mpmath quadrature, closed forms printed in the paper or
following from it, scipy/numpy library routines, limits and symmetries.
P:<n> = /root/reference/PAPER.md line (the reference itself is not read here).
"""
from fractions import Fraction
from math import comb

import mpmath as mp
import numpy as np
import pytest
from scipy import ndimage

import workloads

mp.mp.dps = 40


# ---------------------------------------------------------------- Theorem 1
def _hilbert_inverse_exact(N):
    """Gauss-Jordan inverse of the (N+1)x(N+1) Hilbert matrix, eq.(18) P:284-288,
    in exact rationals -- independent of the closed form eq.(19)."""
    n = N + 1
    A = [[Fraction(1, i + j + 1) for j in range(n)] + [Fraction(int(i == j)) for j in range(n)]
         for i in range(n)]
    for c in range(n):
        piv = next(r for r in range(c, n) if A[r][c] != 0)
        A[c], A[piv] = A[piv], A[c]
        pv = A[c][c]
        A[c] = [v / pv for v in A[c]]
        for r in range(n):
            if r != c and A[r][c] != 0:
                fac = A[r][c]
                A[r] = [a - fac * b for a, b in zip(A[r], A[c])]
    return [[A[i][n + j] for j in range(n)] for i in range(n)]


@pytest.mark.parametrize("N", list(range(0, 13)))
def test_hilbert_inverse_matches_exact_rational_inverse(orc, N):
    exact = _hilbert_inverse_exact(N)
    got = orc.hilbert_inverse(N)
    for i in range(N + 1):
        for j in range(N + 1):
            e = exact[i][j]
            assert e.denominator == 1
            if abs(e.numerator) < 2 ** 53:
                assert got[i, j] == float(e.numerator), (i, j)
            else:
                assert abs(got[i, j] - e.numerator) <= 2 ** -52 * abs(e.numerator)


def test_hilbert_inverse_small_examples(orc):
    # the 1x1 Hilbert matrix is [1]; 2x2 and 3x3 inverses by hand
    assert orc.hilbert_inverse(0).tolist() == [[1.0]]
    assert orc.hilbert_inverse(1).tolist() == [[4, -6], [-6, 12]]
    assert orc.hilbert_inverse(2).tolist() == [[9, -36, 30], [-36, 192, -180], [30, -180, 180]]


# ---------------------------------------------------------------- fit
@pytest.mark.parametrize("N", [0, 1, 2, 5, 8, 10])
def test_fit_reproduces_moments(orc, N):
    """c = A^{-1} mu must satisfy the moment-matching equations eq.(14)/(17):
    int_0^1 t^k p(t) dt = sum_n c_n/(k+n+1) = mu_k, checked in 40-digit mpmath."""
    rng = np.random.default_rng(N)
    t = rng.beta(0.7, 1.3, 200)  # moments of a genuine histogram on [0,1]
    mu = np.array([np.sum(t ** k) for k in range(N + 1)])
    c = orc.fit(mu, N)
    cm = [mp.mpf(x) for x in c]
    for k in range(N + 1):
        lhs = mp.fsum(cm[n] / (k + n + 1) for n in range(N + 1))
        assert abs(lhs - mu[k]) <= 1e-9 * mu[0], (k, float(lhs), mu[k])


def test_fit_known_polynomials(orc):
    # moments of p(t)=1 on [0,1] are 1/(k+1) -> c = e_1
    for N in range(0, 9):
        mu = np.array([1.0 / (k + 1) for k in range(N + 1)])
        c = orc.fit(mu, N)
        # mu is rounded to double (rel. 1.1e-16); A^{-1} amplifies that by its row sums
        amp = max(sum(abs(float(v)) for v in row) for row in _hilbert_inverse_exact(N))
        assert np.allclose(c, np.eye(N + 1)[0], rtol=0, atol=2.3e-16 * amp)
    # moments of p(t)=t are 1/(k+2) -> c = e_2
    c = orc.fit(np.array([1 / 2, 1 / 3, 1 / 4]), 2)
    assert np.allclose(c, [0, 1, 0], atol=1e-12)


# ---------------------------------------------------------------- Prop.3 eq.(24)
@pytest.mark.parametrize("seed", range(5))
def test_stretch_equals_direct_stretched_moments(orc, seed):
    """eq.(24) applied to raw moments m_r = sum f_j^r must equal the moments of
    the explicitly remapped values ((f_j-alpha)/(beta-alpha))^k (App.B);
    exact rational reference."""
    rng = np.random.default_rng(seed)
    f = rng.integers(0, 21, 49)  # small integers: m_r exact in double
    if f.min() == f.max():
        f[0] += 1
    N = 8
    a, b = int(f.min()), int(f.max())
    m = np.array([float(sum(int(v) ** r for v in f)) for r in range(N + 1)])
    mu = orc.stretch(m, N, a, b)
    for k in range(N + 1):
        exact = sum(Fraction(int(v) - a, b - a) ** k for v in f)
        assert abs(mu[k] - float(exact)) <= 1e-13 * max(1.0, float(exact)), k


def test_stretch_special_cases(orc):
    m = np.array([5.0, 2.0, 1.5, 1.25])
    assert np.allclose(orc.stretch(m, 3, 0.0, 1.0), m, rtol=0, atol=1e-15)  # alpha=0,beta=1
    # all mass at alpha: m_k = W alpha^k -> mu = (W, 0, 0, ...)
    alpha, W = 0.3, 7.0
    m = np.array([W * alpha ** k for k in range(6)])
    mu = orc.stretch(m, 5, alpha, 0.9)
    assert mu[0] == pytest.approx(W) and np.all(np.abs(mu[1:]) < 1e-13)


# ---------------------------------------------------------------- integrals eq.(28)-(32)
def _I_mp(lam, t0, k):
    # mpmath's quad stops on an absolute tolerance: integrate the integrand
    # scaled to O(1) (factor exp(lam d^2), d = distance of t0 from [0,1]) and
    # undo the factor afterwards
    c = min(max(t0, mp.mpf(0)), mp.mpf(1))
    d2 = (t0 - c) ** 2
    f = lambda t: t ** k * mp.e ** (-lam * ((t - t0) ** 2 - d2))
    return mp.e ** (-lam * d2) * _quad_peaked(f, lam, t0, c)


def _quad_peaked(f, lam, t0, c):
    # breakpoints at multiples of the integrand's decay length around the peak
    scales = [1 / mp.sqrt(lam)]
    if abs(t0 - c) > 0:
        scales.append(1 / (2 * lam * abs(t0 - c)))
    pts = {mp.mpf(0), mp.mpf(1), c}
    for s in scales:
        for j in (0.25, 0.5, 1, 2, 4, 8, 16):
            for p in (c - j * s, c + j * s):
                if 0 < p < 1:
                    pts.add(p)
    return mp.quad(f, sorted(pts))


LAMS = [1e-6, 1e-3, 0.05, 0.3, 1.0, 2.0, 8.0, 50.0, 400.0, 3000.0]
T0S = [-1.5, -0.3, 0.0, 0.21, 0.5, 0.97, 1.0, 1.4, 2.5]


@pytest.mark.parametrize("lam", LAMS)
def test_integrals_against_mpmath(orc, lam):
    K = 11
    for t0 in T0S:
        I, used = orc.integrals(lam, t0, K)
        ref = [_I_mp(mp.mpf(lam), mp.mpf(t0), k) for k in range(K + 1)]
        scale = float(max(abs(r) for r in ref))
        for k in range(K + 1):
            assert abs(I[k] - float(ref[k])) <= 1e-14 * scale + 1e-300, (lam, t0, k, used)


def test_integral_recursion_and_quadrature_agree(orc):
    """eqs.(30)-(32) and direct quadrature of eq.(28) are two routes to the same
    numbers; where both are accurate they must agree."""
    for lam in [0.5, 0.8, 1.0]:
        for t0 in [-0.4, 0.0, 0.3, 0.5, 1.2]:
            I1, u1 = orc.integrals(lam, t0, 11, method=1)
            I2, u2 = orc.integrals(lam, t0, 11, method=2)
            assert (u1, u2) == (1, 2)
            assert np.max(np.abs(I1 - I2)) <= 1e-15 * I2[0]


def test_integral_closed_forms(orc):
    # I_0(lambda=1, t0=0) = int_0^1 exp(-t^2) dt = sqrt(pi)/2 erf(1)
    I, _ = orc.integrals(1.0, 0.0, 2, method=1)
    assert I[0] == pytest.approx(0.7468241328124270, abs=1e-15)
    for method in (1, 2):
        # symmetric integrand about t = 1/2 -> I_1 = I_0 / 2
        for lam in [0.7, 3.0, 100.0]:
            I, _ = orc.integrals(lam, 0.5, 2, method=method)
            assert I[1] == pytest.approx(I[0] / 2, rel=1e-14)
        # t0 = 0: I_2 = (I_0 - e^{-lambda}) / (2 lambda)  (integration by parts)
        lam = 0.9
        I, _ = orc.integrals(lam, 0.0, 2, method=method)
        assert I[2] == pytest.approx((I[0] - np.exp(-lam)) / (2 * lam), rel=1e-13)
    # lambda -> 0: I_k -> 1/(k+1)
    I, _ = orc.integrals(1e-12, 0.3, 8)
    assert np.allclose(I, [1 / (k + 1) for k in range(9)], rtol=1e-10)
    # lambda = 100, t0 = 1/2: almost all mass inside -> I_0 ~ sqrt(pi/100)
    I, _ = orc.integrals(100.0, 0.5, 0)
    assert I[0] == pytest.approx(np.sqrt(np.pi / 100), rel=1e-10)


# ---------------------------------------------------------------- whole g-hat (eq.(29))
def _ghat_projection_mp(vals, theta, sigma, N):
    """Independent evaluation of eq.(29) through the projection identity:
    sum_k c_k I_k = sum_j (Pi_N psi)(t_j), with Pi_N the L2[0,1] projection onto
    polynomials of degree <= N (follows from eq.(14) + eq.(28)); no Hilbert
    matrix, no recursion.  Legendre coefficients by mpmath quadrature."""
    a, b = mp.mpf(float(min(vals))), mp.mpf(float(max(vals)))
    d = b - a
    lam = d ** 2 / (2 * mp.mpf(float(sigma)) ** 2)
    t0 = (mp.mpf(float(theta)) - a) / d
    psi = lambda t: mp.e ** (-lam * (t - t0) ** 2)
    P = lambda k, t: mp.legendre(k, 2 * t - 1)
    pts = sorted({mp.mpf(0), min(max(t0, mp.mpf(0)), mp.mpf(1)), mp.mpf(1)})
    J = [mp.quad(lambda t: P(k, t) * psi(t), pts) for k in range(N + 1)]
    Jt = [mp.quad(lambda t: t * P(k, t) * psi(t), pts) for k in range(N + 1)]
    ts = [(mp.mpf(float(v)) - a) / d for v in vals]
    num = den = mp.mpf(0)
    absum = mp.mpf(0)
    for k in range(N + 1):
        nu = mp.fsum(P(k, t) for t in ts)
        den += (2 * k + 1) * nu * J[k]
        num += (2 * k + 1) * nu * Jt[k]
        absum += abs((2 * k + 1) * nu * J[k])
    return float(a + d * num / den), float(absum / den) if den > 0 else float("inf")


@pytest.mark.parametrize("N", [0, 1, 2, 5, 8, 10])
def test_window_ghat_projection_identity(orc, N):
    rng = np.random.default_rng(100 + N)
    for trial in range(3):
        n = 25 if trial < 2 else 49
        vals = np.rint(rng.normal(120, 30, n)).clip(0, 255).astype(np.float32)
        if trial == 1:
            vals[: n // 3] = rng.integers(200, 255, n // 3)  # bimodal window
        theta = float(np.float32(vals[n // 2] + rng.uniform(-15, 15)))  # the API is float32
        sigma = float(np.float32(rng.uniform(8, 50)))
        o = orc.fast_window(vals, vals[n // 2], theta, sigma, N)
        ref, kap = _ghat_projection_mp(vals, theta, sigma, N)
        span = float(vals.max() - vals.min())
        assert abs(o["g_lit"] - ref) <= 1e-9 * span, (trial, o["g_lit"], ref)
        assert o["kappa"] == pytest.approx(kap, rel=1e-8)


def test_window_limits(orc):
    rng = np.random.default_rng(7)
    vals = np.rint(rng.uniform(0, 255, 49)).astype(np.float32)
    # constant window: identity
    c = np.full(49, 77.0, np.float32)
    o = orc.fast_window(c, 77.0, 90.0, 10.0, 5)
    assert o["g_lit"] == 77.0 and o["code"] & orc.CODE_IDENTITY
    # sigma -> inf: psi == 1, so g-hat is the box mean for N >= 1 (the fitted p
    # reproduces mu_1) and the midrange for N = 0 (constant p on [alpha, beta])
    for N in (1, 3, 6, 9):
        o = orc.fast_window(vals, vals[24], 100.0, 1e7, N)
        assert o["g_lit"] == pytest.approx(float(np.mean(vals.astype(np.float64))), abs=1e-6)
    o = orc.fast_window(vals, vals[24], 100.0, 1e7, 0)
    assert o["g_lit"] == pytest.approx((float(vals.min()) + float(vals.max())) / 2, abs=1e-6)


def test_window_symmetries(orc):
    rng = np.random.default_rng(11)
    vals = np.rint(rng.normal(100, 40, 81)).clip(0, 255).astype(np.float32)
    theta, sigma, N = float(vals[40] + 6), 21.0, 6
    o = orc.fast_window(vals, vals[40], theta, sigma, N)
    # affine equivariance: f -> a f + b, theta -> a theta + b, sigma -> |a| sigma
    a, b = 0.5, -3.0  # exact in float32 for these integers
    o2 = orc.fast_window(a * vals + b, a * vals[40] + b, a * theta + b, abs(a) * sigma, N)
    assert o2["g_lit"] == pytest.approx(a * o["g_lit"] + b, abs=1e-9)
    # reflection f -> 255 - f
    o3 = orc.fast_window(255 - vals, 255 - vals[40], 255 - theta, sigma, N)
    assert o3["g_lit"] == pytest.approx(255 - o["g_lit"], abs=1e-9)


def test_ghat_converges_to_brute_force_with_N(orc):
    """eq.(29) is the brute force eq.(1) with the range kernel replaced by its
    degree-N projection; the mean error over windows falls with N and is tiny
    at N=16 (Table I's trend)."""
    rng = np.random.default_rng(3)
    errs = []
    for _ in range(20):
        vals = np.rint(rng.normal(120, 25, 25)).clip(0, 255).astype(np.float32)
        theta, sigma = float(vals[12]), 30.0
        w = np.exp(-((vals.astype(np.float64) - theta) ** 2) / (2 * sigma ** 2))
        g = float(np.sum(w * vals) / np.sum(w))
        errs.append([abs(orc.fast_window(vals, vals[12], theta, sigma, N)["g_lit"] - g)
                     for N in (0, 2, 6, 10, 16)])
    m = np.mean(errs, axis=0)
    assert m[0] > m[1] > m[2] > m[3] > m[4]
    assert np.max(errs, axis=0)[4] < 1e-4


def test_guard_semantics(orc):
    rng = np.random.default_rng(5)
    for _ in range(40):
        vals = np.rint(rng.normal(120, 50, 49)).clip(0, 255).astype(np.float32)
        theta, sigma = float(rng.uniform(0, 255)), float(rng.uniform(2, 30))
        o = orc.fast_window(vals, vals[24], theta, sigma, 8)
        o0 = orc.fast_window(vals, vals[24], theta, sigma, 0)
        if o["t2n"] > 0 and o["kappa"] <= orc.KAPPA_MAX:
            assert o["g_guard"] == o["g_lit"] and not (o["code"] & orc.CODE_GUARD)
        else:
            assert o["code"] & orc.CODE_GUARD
            assert o["g_guard"] == pytest.approx(o0["g_lit"], abs=1e-9)
        assert o0["kappa"] == pytest.approx(1.0)


# ---------------------------------------------------------------- image level
def _windows_numpy(img, rho):
    p = np.pad(img, rho, mode="symmetric")  # half-sample symmetric (reading R2)
    H, W = img.shape
    k = 2 * rho + 1
    return np.lib.stride_tricks.sliding_window_view(p, (k, k)).reshape(H, W, k * k)


@pytest.mark.parametrize("shape,rho", [((7, 9), 3), ((16, 16), 0), ((20, 33), 5), ((11, 40), 2)])
def test_bounds_against_scipy(orc, shape, rho):
    rng = np.random.default_rng(sum(shape) + rho)
    f = np.rint(rng.uniform(0, 255, shape)).astype(np.float32)
    a, b = orc.bounds(f, rho)
    k = 2 * rho + 1
    assert np.array_equal(a, ndimage.minimum_filter(f, size=k, mode="reflect"))
    assert np.array_equal(b, ndimage.maximum_filter(f, size=k, mode="reflect"))
    assert np.all(a <= f) and np.all(f <= b)


def test_bounds_1d_example(orc):
    row = np.array([1, 5, 2, 4, 3], np.float32)
    a, b = orc.bounds(np.stack([row] * 3), 1)
    assert (a[1, 2], b[1, 2]) == (2.0, 5.0)


def test_brute_against_numpy(orc):
    rng = np.random.default_rng(9)
    f = np.rint(rng.uniform(0, 255, (13, 17))).astype(np.float32)
    th = (f + rng.uniform(-10, 10, f.shape)).astype(np.float32)
    sg = rng.uniform(5, 40, f.shape).astype(np.float32)
    rho = 3
    win = _windows_numpy(f.astype(np.float64), rho)
    w = np.exp(-((win - th[..., None].astype(np.float64)) ** 2) / (2 * sg[..., None].astype(np.float64) ** 2))
    ref = np.sum(w * win, -1) / np.sum(w, -1)
    assert np.allclose(orc.brute(f, th, sg, rho), ref, rtol=0, atol=1e-9)


def test_brute_limits(orc):
    rng = np.random.default_rng(2)
    f = np.rint(rng.uniform(0, 255, (12, 12))).astype(np.float32)
    big = np.full_like(f, 1e8)
    g = orc.brute(f, f, big, 2)
    assert np.allclose(g, ndimage.uniform_filter(f.astype(np.float64), 5, mode="reflect"), atol=1e-6)
    c = np.full((9, 9), 42.0, np.float32)
    assert np.all(orc.brute(c, c + 3, np.full_like(c, 5.0), 2) == 42.0)
    # step edge with small sigma is preserved
    s = np.zeros((9, 12), np.float32)
    s[:, 6:] = 200
    g = orc.brute(s, s, np.full_like(s, 10.0), 2)
    assert np.allclose(g, s, atol=1e-6)


def test_brute_underflow_shift(orc):
    # sigma tiny and theta away from every sample: unshifted weights would all
    # underflow; eq.(1) still has a well-defined value (nearest-to-theta samples)
    f = np.array([[10, 20, 30], [10, 20, 30], [10, 20, 30]], np.float32)
    g = orc.brute(f, np.full_like(f, 24.0), np.full_like(f, 0.01), 1)
    assert np.all(np.isfinite(g)) and g[1, 1] == pytest.approx(20.0)


def test_fast_image_equals_window_route(orc):
    w = workloads.random_case(2, 13, 19, seed=4, rho=3, N=5)
    o = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N)
    for b in range(2):
        win = _windows_numpy(w.img[b], w.rho)
        for (y, x) in [(0, 0), (6, 9), (12, 18), (0, 18), (5, 0)]:
            r = orc.fast_window(win[y, x], w.img[b, y, x], w.theta[b, y, x], w.sigma[b, y, x], w.N)
            assert o["g_lit"][b, y, x] == r["g_lit"]
            assert o["g_guard"][b, y, x] == r["g_guard"]
    # pixel-list route returns the same values
    idx = np.array([0, 5, 200, 13 * 19 + 7, 2 * 13 * 19 - 1])
    ol = orc.fast(w.img, w.theta, w.sigma, w.rho, w.N, pixels=idx)
    assert np.array_equal(ol["g_guard"], o["g_guard"].ravel()[idx])


def test_fast_rho0_is_identity(orc):
    w = workloads.random_case(1, 8, 8, seed=1, rho=0, N=3)
    o = orc.fast(w.img, w.theta, w.sigma, 0, 3)
    assert np.array_equal(o["g_guard"], w.img.astype(np.float64))


def test_psnr_trend_with_N(orc):
    """Table I's trend: PSNR(fast, brute) rises with N (synthetic)."""
    w = workloads.config(1, scale=0.25)
    g = orc.brute(w.img, w.theta, w.sigma, w.rho)
    ps = []
    for N in (0, 2, 5):
        o = orc.fast(w.img, w.theta, w.sigma, w.rho, N)
        mse = np.mean((o["g_guard"] - g) ** 2)
        ps.append(10 * np.log10(255 ** 2 / mse))
    assert ps[0] < ps[1] < ps[2] and ps[2] > 40.0


@pytest.mark.parametrize("kind", ["integer", "float", "wide_integer"])
def test_histogram_route_equals_sample_sums(orc, kind):
    """eq.(22) summed over the distinct values t of the window weighted by the
    histogram H_i(t) of eq.(5)/(21) (the oracle's route) equals the same sum taken
    sample by sample: the two differ only in the order of __float128 additions."""
    rng = np.random.default_rng({"integer": 1, "float": 2, "wide_integer": 3}[kind])
    for trial in range(40):
        n = int(rng.choice([9, 49, 121, 1681]))
        if kind == "integer":  # the workloads: 0..255 levels, many repeats
            vals = np.rint(np.clip(rng.normal(120, 25, n), 0, 255)).astype(np.float32)
        elif kind == "float":  # non-integer: the sorted-copy route
            vals = rng.normal(0.3, 2.0, n).astype(np.float32)
            vals[: n // 3] = vals[0]  # repeated values too
        else:  # integers spanning more than the counting table: sorted route
            vals = rng.integers(-30000, 30000, n).astype(np.float32)
        N = int(rng.integers(0, 11))
        theta = float(vals.mean() + rng.normal(0, 5))
        sigma = float(rng.uniform(2, 60))
        a = orc.fast_window(vals, vals[n // 2], theta, sigma, N, route=0)
        b = orc.fast_window(vals, vals[n // 2], theta, sigma, N, route=1)
        for k in ("g_lit", "g_guard", "kappa", "t2n"):
            assert a[k] == pytest.approx(b[k], rel=1e-13, abs=1e-13), (trial, k)


def test_literal_o3_matches_reference_when_well_conditioned(orc):
    """O3 (Algorithm 1 as printed, fp64, context only) equals the __float128
    reference where the paper's numerics are safe: small N, lambda >= 2 (forward
    recursion stable), no guard firing.  A dropped term in eq.(24), eq.(19),
    eq.(30)-(32) or the [0,1] scaling would show up here."""
    w = workloads.random_case(1, 40, 48, seed=21, kind="rect", rho=3, N=3)
    sg = np.full_like(w.sigma, 12.0)
    lit = orc.literal(w.img, w.theta, sg, 3, 3)
    o = orc.fast(w.img, w.theta, sg, 3, 3)
    ok = (o["kappa"] < 50) & (o["code"] & orc.CODE_QUAD == 0)
    assert ok.mean() > 0.5
    assert np.max(np.abs(lit[ok] - o["g_lit"][ok])) < 1e-6
    ident = (o["code"] & orc.CODE_IDENTITY) > 0
    assert np.array_equal(lit[ident], w.img[ident].astype(np.float64))


def test_mozerov_against_quadrature_and_limits(orc):
    """The Mozerov baseline: the range-kernel-weighted mean of a uniform
    density on [f, 2 fbar - f], evaluated here by mpmath quadrature of that ratio
    (no erf, no recursion); sigma -> inf gives the interval's midpoint = fbar; a
    constant image maps to itself."""
    import mpmath as mp

    w = workloads.random_case(1, 15, 17, seed=33, kind="rect", rho=2, N=0)
    g = orc.mozerov(w.img, w.theta, w.sigma, 2)
    f = w.img[0]
    pad = np.pad(f.astype(np.float64), 2, mode="symmetric")
    for (y, x) in [(0, 0), (7, 8), (14, 16), (3, 12), (10, 1)]:
        fbar = pad[y:y + 5, x:x + 5].mean()
        a, b = sorted((float(f[y, x]), 2 * fbar - float(f[y, x])))
        th, s = float(w.theta[0, y, x]), float(w.sigma[0, y, x])
        if b - a < 1e-9:
            assert g[0, y, x] == f[y, x]
            continue
        k = lambda t: mp.exp(-(t - th) ** 2 / (2 * s * s))
        ref = mp.quad(lambda t: t * k(t), [a, b]) / mp.quad(k, [a, b])
        assert g[0, y, x] == pytest.approx(float(ref), abs=1e-9)
    big = orc.mozerov(w.img, w.theta, np.full_like(w.sigma, 1e7), 2)
    box = np.array([[pad[y:y + 5, x:x + 5].mean() for x in range(17)] for y in range(15)])
    assert np.max(np.abs(big[0] - box)) < 1e-6
    c = np.full((1, 9, 9), 77.0, np.float32)
    assert np.all(orc.mozerov(c, c + 3, np.full_like(c, 10.0), 2) == 77.0)


@pytest.mark.parametrize("rho,s", [(5, 1.0), (2, 0.7), (3, 2.0)])
def test_sharpen_maps_against_scipy(orc, rho, s):
    """P:620-630 maps: fbar equals scipy's uniform_filter and the LoG equals
    scipy's gaussian_laplace (reflect borders, truncate 4) -- independent
    library routines; sigma is the stated affine map of |LoG|, clipped."""
    from scipy import ndimage

    w = workloads.random_case(1, 33, 41, seed=61, kind="texture", rho=rho, N=0)
    f = w.img[0].astype(np.float64)
    th, sg = orc.sharpen_maps(w.img, rho, log_scale=s, sigma_lo=8.0, sigma_hi=35.0, log_sat=12.0)
    fbar = ndimage.uniform_filter(f, size=2 * rho + 1, mode="reflect")
    assert np.max(np.abs(th[0] - (2 * f - fbar))) < 1e-9
    L = ndimage.gaussian_laplace(f, s, mode="reflect", truncate=4.0)
    ref = 35.0 - (35.0 - 8.0) * np.minimum(np.abs(L) / 12.0, 1.0)
    assert np.max(np.abs(sg[0] - ref)) < 1e-9
    assert sg.min() >= 8.0 and sg.max() <= 35.0


# ---------------------------------------------------------------- NEXT-2: texture maps (mRTV)
@pytest.mark.parametrize("patch", [1, 3, 5])
def test_texture_maps_against_scipy(orc, patch):
    """mRTV of P:835-842 (reading R19): the window max / min / sum come from
    scipy's maximum_filter / minimum_filter / uniform_filter (reflect borders,
    independent library routines) applied to f and to numpy's forward-difference
    gradient magnitude; sigma is the stated affine map, clipped."""
    w = workloads.random_case(2, 37, 45, seed=71, kind="texture", rho=2, N=0)
    eps, m_sat = 1e-3, 9.0
    m, sg = orc.texture_maps(w.img, patch=patch, sigma_lo=6.0, sigma_hi=44.0, mrtv_sat=m_sat, eps=eps)
    for b in range(2):
        f = w.img[b].astype(np.float64)
        gx = np.diff(f, axis=1, append=f[:, -1:])
        gy = np.diff(f, axis=0, append=f[-1:, :])
        G = np.hypot(gx, gy)
        k = 2 * patch + 1
        delta = ndimage.maximum_filter(f, size=k, mode="reflect") - ndimage.minimum_filter(f, size=k, mode="reflect")
        gmax = ndimage.maximum_filter(G, size=k, mode="reflect")
        gsum = ndimage.uniform_filter(G, size=k, mode="reflect") * k * k
        ref = delta * gmax / (gsum + eps)
        assert np.max(np.abs(m[b] - ref)) < 1e-9 * max(1.0, ref.max())
        rs = 44.0 - (44.0 - 6.0) * np.minimum(ref / m_sat, 1.0)
        assert np.max(np.abs(sg[b] - rs)) < 1e-8
    assert sg.min() >= 6.0 and sg.max() <= 44.0


def test_texture_maps_closed_forms(orc):
    """Closed forms that follow from the definition: a constant image
    has mRTV = 0 (sigma = sigma_hi); a vertical step edge of height A has
    mRTV = A * A / ((2p+1) A + eps) at every pixel whose window meets the edge
    (Delta = A, one gradient sample of size A per window row); one-pixel vertical
    stripes 0 / A have mRTV = A * A / (n A + eps) in the interior -- the texture
    scores below the edge ("high near sharp edges and low in textured
    regions"); mRTV is invariant to an intensity offset and, as eps -> 0,
    proportional to an intensity scale."""
    p, A, eps = 3, 60.0, 1e-6
    n = (2 * p + 1) ** 2
    c = np.full((1, 20, 24), 91.0, np.float32)
    m, sg = orc.texture_maps(c, patch=p, sigma_lo=5.0, sigma_hi=33.0, mrtv_sat=4.0, eps=eps)
    assert np.all(m == 0.0) and np.all(sg == 33.0)
    e = np.zeros((1, 20, 24), np.float32)
    e[:, :, 12:] = A
    m, _ = orc.texture_maps(e, patch=p, eps=eps)
    edge = A * A / ((2 * p + 1) * A + eps)
    # forward difference: the gradient sample sits at column 11; windows of columns 8..14 contain it,
    # of which columns 9..14 also see both levels (column 8's window is columns 5..11: flat, Delta = 0)
    assert np.allclose(m[0, :, 9:15], edge, rtol=1e-12)
    assert np.all(m[0, :, :9] == 0.0) and np.all(m[0, :, 15:] == 0.0)
    s = np.zeros((1, 20, 24), np.float32)
    s[:, :, 1::2] = A
    m, _ = orc.texture_maps(s, patch=p, eps=eps)
    tex = A * A / (n * A + eps)
    assert np.allclose(m[0, 4:-4, 4:-5], tex, rtol=1e-12)
    assert tex < edge
    w = workloads.random_case(1, 25, 31, seed=72, kind="rect", rho=2, N=0)
    m0, _ = orc.texture_maps(w.img, patch=2, eps=1e-12)
    m1, _ = orc.texture_maps(w.img + 17.0, patch=2, eps=1e-12)
    m2, _ = orc.texture_maps(w.img * 0.5, patch=2, eps=1e-12)
    assert np.allclose(m1, m0, rtol=1e-9, atol=1e-9) and np.allclose(m2, 0.5 * m0, rtol=1e-9, atol=1e-9)


def test_texture_pipeline_composition(orc):
    """the pipeline is three applications of Algorithm 1 -- checked
    here against the three oracle calls made one by one (theta = f, sigma; then
    theta = g1, 0.8 sigma with the same map; then the sharpening maps of g2),
    and on a constant image every pass is the identity."""
    w = workloads.random_case(1, 30, 34, seed=73, kind="texture", rho=3, N=3)
    tp = dict(patch=2, sigma_lo=7.0, sigma_hi=30.0, mrtv_sat=10.0, eps=1e-3, second_scale=0.8)
    sp = dict(log_scale=1.0, sigma_lo=9.0, sigma_hi=25.0, log_sat=15.0)
    r = orc.texture_pipeline(w.img, 3, 3, texture=tp, sharpen=sp, rho_sharpen=2)
    sg = orc.texture_maps(w.img, **tp)[1].astype(np.float32)
    g1 = orc.fast(w.img, w.img, sg, 3, 3)["g_guard"].astype(np.float32)
    g2 = orc.fast(g1, g1, (np.float32(0.8) * sg).astype(np.float32), 3, 3)["g_guard"].astype(np.float32)
    th3, sg3 = orc.sharpen_maps(g2, 2, **sp)
    out = orc.fast(g2, th3.astype(np.float32), sg3.astype(np.float32), 2, 3)["g_guard"]
    assert np.array_equal(r["pass1"], g1) and np.array_equal(r["pass2"], g2) and np.array_equal(r["out"], out)
    # smoothing passes shrink the texture's variance, the structure survives (mean level kept)
    assert r["pass2"].std() < w.img.std() and abs(float(r["pass2"].mean() - w.img.mean())) < 2.0
    c = np.full((1, 16, 18), 40.0, np.float32)
    rc = orc.texture_pipeline(c, 2, 2)
    assert np.all(rc["out"] == 40.0)


# ---------------------------------------------------------------- NEXT-1: Gaussian omega, eq.(4)
def _gauss_w(rho):
    R = 3 * rho
    d = np.arange(-R, R + 1)
    return np.exp(-(d[:, None] ** 2 + d[None, :] ** 2) / (2.0 * rho * rho))


def _ghat_projection_mp_w(vals, wts, theta, sigma, N):
    """eq.(29) with the weighted histogram of eq.(5): the projection identity
    with weights, sum_k c_k I_k = sum_j w_j (Pi_N psi)(t_j); mpmath, no Hilbert
    matrix, no recursion."""
    a, b = mp.mpf(float(min(vals))), mp.mpf(float(max(vals)))
    d = b - a
    lam = d ** 2 / (2 * mp.mpf(float(sigma)) ** 2)
    t0 = (mp.mpf(float(theta)) - a) / d
    psi = lambda t: mp.e ** (-lam * (t - t0) ** 2)
    P = lambda k, t: mp.legendre(k, 2 * t - 1)
    pts = sorted({mp.mpf(0), min(max(t0, mp.mpf(0)), mp.mpf(1)), mp.mpf(1)})
    J = [mp.quad(lambda t: P(k, t) * psi(t), pts) for k in range(N + 1)]
    Jt = [mp.quad(lambda t: t * P(k, t) * psi(t), pts) for k in range(N + 1)]
    ts = [(mp.mpf(float(v)) - a) / d for v in vals]
    ws = [mp.mpf(float(x)) for x in wts]
    num = den = mp.mpf(0)
    for k in range(N + 1):
        nu = mp.fsum(wj * P(k, t) for wj, t in zip(ws, ts))
        den += (2 * k + 1) * nu * J[k]
        num += (2 * k + 1) * nu * Jt[k]
    return float(a + d * num / den)


@pytest.mark.parametrize("N", [0, 2, 5, 8])
def test_gauss_window_projection_identity_and_routes(orc, N):
    rng = np.random.default_rng(500 + N)
    wts = _gauss_w(2).ravel()  # 13 x 13
    for trial in range(2):
        vals = np.rint(rng.normal(110, 35, wts.size)).clip(0, 255).astype(np.float32)
        if trial:
            vals[::3] = rng.integers(200, 255, vals[::3].size)
        theta = float(np.float32(vals[wts.size // 2] + rng.uniform(-10, 10)))
        sigma = float(np.float32(rng.uniform(10, 50)))
        o = orc.fast_window(vals, vals[wts.size // 2], theta, sigma, N, weights=wts)
        o1 = orc.fast_window(vals, vals[wts.size // 2], theta, sigma, N, route=1, weights=wts)
        ref = _ghat_projection_mp_w(vals, wts, theta, sigma, N)
        span = float(vals.max() - vals.min())
        assert abs(o["g_lit"] - ref) <= 1e-9 * span, (trial, o["g_lit"], ref)
        assert o["g_lit"] == pytest.approx(o1["g_lit"], rel=1e-13, abs=1e-13)
        # the weighted and the unweighted filters differ (the weights matter)
        if N >= 2:
            ob = orc.fast_window(vals, vals[wts.size // 2], theta, sigma, N)
            assert abs(ob["g_lit"] - o["g_lit"]) > 1e-6


def test_gauss_image_routes_limits_and_brute(orc):
    """fast(spatial="gauss") equals the weighted window route pixel by pixel;
    sigma -> inf gives the Gaussian-weighted mean (N >= 1); brute force with the
    Gaussian omega equals an independent numpy implementation."""
    rho = 2
    w = workloads.random_case(1, 19, 23, seed=9, kind="rect", rho=rho, N=4)
    R = 3 * rho
    W2 = _gauss_w(rho)
    pad = np.pad(w.img[0].astype(np.float64), R, mode="symmetric")
    o = orc.fast(w.img, w.theta, w.sigma, rho, 4, spatial="gauss")
    for (y, x) in [(0, 0), (9, 11), (18, 22), (4, 20)]:
        win = pad[y:y + 2 * R + 1, x:x + 2 * R + 1].astype(np.float32)
        r = orc.fast_window(win, w.img[0, y, x], w.theta[0, y, x], w.sigma[0, y, x], 4, weights=W2)
        assert o["g_lit"][0, y, x] == r["g_lit"] and o["g_guard"][0, y, x] == r["g_guard"]
    big = orc.fast(w.img, w.theta, np.full_like(w.sigma, 1e7), rho, 3, spatial="gauss")
    mean = np.array([[np.sum(W2 * pad[y:y + 2 * R + 1, x:x + 2 * R + 1]) / W2.sum() for x in range(23)]
                     for y in range(19)])
    assert np.max(np.abs(big["g_guard"][0] - mean)) < 1e-6
    g = orc.brute(w.img, w.theta, w.sigma, rho, spatial="gauss")
    ref = np.empty((19, 23))
    for y in range(19):
        for x in range(23):
            v = pad[y:y + 2 * R + 1, x:x + 2 * R + 1]
            k = W2 * np.exp(-(v - w.theta[0, y, x]) ** 2 / (2.0 * float(w.sigma[0, y, x]) ** 2))
            ref[y, x] = np.sum(k * v) / np.sum(k)
    assert np.max(np.abs(g[0] - ref)) < 1e-9
