"""Pins of the oracle's Eq. 8 loss terms (NEXT-1) against things other than
itself (-m "not gpu"): closed forms of SSIM, the textbook Gaussian window
through impulse images, symmetry, finite differences of the image-loss
gradient, the SPEC.md worked example and numpy's eigenvalues for the
regularizers, and finite differences of the regularizer gradients as they
enter the sampler step.

PAPER.md:137-141 (Eq. 8): L = (1 - eps_D) L1 + eps_D L_D-SSIM
                              + eps_o sum |o_i| + eps_Sigma sum_ij sqrt(lambda_ij).
SSIM convention (R28): 11x11 Gaussian window,
sigma 1.5, K1 0.01, K2 0.03, dynamic range 1, valid window positions only.
"""
import math

import numpy as np
import pytest

from helpers import planes_from, raw_o_for

C1, C2 = 0.01 ** 2, 0.03 ** 2


def _gauss_1d():
    # textbook 11-tap Gaussian, sigma 1.5, normalised (Wang et al. 2004)
    g = np.array([math.exp(-(k - 5) ** 2 / (2 * 1.5 ** 2)) for k in range(11)])
    return g / g.sum()


def test_ssim_identical_images_is_one(orc):
    rng = np.random.default_rng(0)
    for shape in [(3, 11, 11), (3, 17, 29)]:
        x = rng.random(shape)
        assert orc.ssim(x, x) == pytest.approx(1.0, abs=1e-14)
        val, d = orc.image_loss(x, x, 1.0)
        assert val == pytest.approx(0.0, abs=1e-14)
        # at the optimum the D-SSIM gradient vanishes
        assert np.abs(d).max() < 1e-12


def test_ssim_constant_images_closed_form(orc):
    """constant a vs constant b -> (2ab + C1)/(a^2 + b^2 + C1)
    (the variance terms are (0 + C2)/(0 + C2))."""
    for a, b in [(0.2, 0.7), (0.5, 0.5), (0.0, 0.3), (0.9, 0.1)]:
        x = np.full((3, 14, 12), a)
        y = np.full((3, 14, 12), b)
        ref = (2 * a * b + C1) / (a * a + b * b + C1)
        assert orc.ssim(x, y) == pytest.approx(ref, rel=1e-12)


@pytest.mark.parametrize("at", [(5, 5), (5, 7), (2, 9), (0, 0)])
def test_ssim_impulse_pins_the_gaussian_window(orc, at):
    """One window (11x11 image): x = unit impulse at `at`, y = 0.  Then
    mx = w, E[x^2] = w with w = g_i g_j of the textbook window, my = sy = sxy = 0:
    SSIM = C1 C2 / ((w^2 + C1) (w - w^2 + C2))."""
    g = _gauss_1d()
    x = np.zeros((3, 11, 11))
    x[:, at[0], at[1]] = 1.0
    y = np.zeros_like(x)
    w = g[at[0]] * g[at[1]]
    ref = C1 * C2 / ((w * w + C1) * (w - w * w + C2))
    assert orc.ssim(x, y) == pytest.approx(ref, rel=1e-12)


def test_ssim_is_symmetric_and_bounded(orc):
    rng = np.random.default_rng(1)
    for _ in range(3):
        a, b = rng.random((3, 16, 19)), rng.random((3, 16, 19))
        s = orc.ssim(a, b)
        assert s == pytest.approx(orc.ssim(b, a), abs=1e-13)
        assert -1.0 <= s <= 1.0
        assert s < 1.0


def test_l1_only_when_eps_zero(orc):
    """eps_D = 0 leaves the BASELINE L1 objective: mean |C - T| and
    sign(C - T)/(3HW) (sign(0) = 0)."""
    rng = np.random.default_rng(2)
    x, y = rng.random((3, 9, 7)), rng.random((3, 9, 7))
    y[0, 0, 0] = x[0, 0, 0]
    val, d = orc.image_loss(x, y, 0.0)
    assert val == pytest.approx(np.abs(x - y).mean(), rel=1e-14)
    np.testing.assert_array_equal(d, np.sign(x - y) / x.size)


@pytest.mark.parametrize("eps_d", [0.2, 1.0])
def test_image_loss_gradient_finite_differences(orc, eps_d):
    """dL/dC against central differences of the oracle's own loss value at
    sampled pixels (values kept >= 1e-3 from the target so the L1 kink is not
    crossed), every channel, interior and border pixels."""
    rng = np.random.default_rng(3)
    H, W = 23, 19
    x = rng.random((3, H, W))
    y = rng.random((3, H, W))
    close = np.abs(x - y) < 1e-3
    x[close] += 2e-3
    _, d = orc.image_loss(x, y, eps_d)
    h = 1e-6
    picks = [(c, i, j) for c in range(3) for (i, j) in [(0, 0), (5, 7), (11, 9), (22, 18), (10, 0), (3, 17)]]
    for (c, i, j) in picks:
        xp, xm = x.copy(), x.copy()
        xp[c, i, j] += h
        xm[c, i, j] -= h
        fd = (orc.image_loss(xp, y, eps_d)[0] - orc.image_loss(xm, y, eps_d)[0]) / (2 * h)
        assert d[c, i, j] == pytest.approx(fd, rel=1e-5, abs=1e-10), (c, i, j)


def test_regularizers_worked_example(orc):
    """one component, o = -0.5, Sigma = diag(4, 1, 1) ->
    opacity_reg 0.5, sigma_reg 2 + 1 + 1 = 4."""
    pl = planes_from([dict(mu=(0, 0, 0), log_scale=(math.log(2.0), 0.0, 0.0), o=-0.5)])
    so, ss = orc.regularizers(pl, 0)
    assert so == pytest.approx(0.5, rel=1e-14)
    assert ss == pytest.approx(4.0, rel=1e-14)


def test_sigma_regularizer_is_sum_of_sqrt_eigenvalues(orc):
    """sum_j sqrt(lambda_j(Sigma)) with lambda from numpy.linalg.eigvalsh of the
    oracle's Sigma = R S S^T R^T."""
    rng = np.random.default_rng(4)
    comps = []
    for _ in range(7):
        q = rng.normal(size=4)
        comps.append(dict(mu=(0, 0, 0), log_scale=tuple(rng.normal(-1.0, 0.7, 3)), q=tuple(q),
                          o=float(rng.uniform(-0.9, 0.9))))
    pl = planes_from(comps)
    _, ss = orc.regularizers(pl, 0)
    ref = 0.0
    for i in range(pl.shape[1]):
        lam = np.linalg.eigvalsh(orc.cov3d(pl[3:6, i], pl[6:10, i]))
        ref += np.sqrt(np.clip(lam, 0, None)).sum()
    assert ss == pytest.approx(ref, rel=1e-10)
    so, _ = orc.regularizers(pl, 0)
    assert so == pytest.approx(sum(abs(c["o"]) for c in comps), rel=1e-12)


def test_regularizer_gradients_enter_the_sampler(orc):
    """The sampler's first Adam moment after one step from m = 0 is
    (1 - beta1) (grad_scale g + d reg / d theta); the regularizer part is
    checked against central differences of the regularizer values
    (eps_o sum |o| + eps_Sigma sum sqrt(lambda))."""
    from sss_synth import SGHMCParams

    rng = np.random.default_rng(5)
    comps = [dict(mu=(0, 0, 0), log_scale=tuple(rng.normal(-1.0, 0.5, 3)), o=float(o))
             for o in (-0.7, -0.1, 0.3, 0.8)]
    pl = planes_from(comps)
    P, n = pl.shape
    hp = SGHMCParams(noise=0.0, eps_o=0.03, eps_sigma=0.02, grad_scale=0.5)
    g = rng.normal(size=(P, n))
    _, m2, _, _ = orc.sghmc_step(pl, 0, g, np.zeros((P, n)), np.zeros((P, n)), np.zeros((3, n)), hp)

    def reg(p):
        so, ss = orc.regularizers(p, 0)
        return hp.eps_o * so + hp.eps_sigma * ss

    h = 1e-6
    for plane in (3, 4, 5, 11):
        for i in range(n):
            pp, pm = pl.copy(), pl.copy()
            pp[plane, i] += h
            pm[plane, i] -= h
            fd = (reg(pp) - reg(pm)) / (2 * h)
            want = (1 - hp.beta1) * (hp.grad_scale * g[plane, i] + fd)
            assert m2[plane, i] == pytest.approx(want, rel=1e-7, abs=1e-12), (plane, i)
    # planes without a regularizer are untouched by it
    for plane in (6, 7, 8, 9, 10, 12):
        np.testing.assert_allclose(m2[plane], (1 - hp.beta1) * hp.grad_scale * g[plane], rtol=1e-14)
