"""Pins of the oracle's NEXT-3 ablation variants (R32)
against closed forms, limits and finite differences:
  POSITIVE (1)  o = sigmoid(raw)                 settings 1-2 "positive t-dis"
  GAUSSIAN (2)  T = exp(-h/2), hmax = 2 ln(255|o|) "SGHMC with Gaussian distributions"
  LOWPASS  (4)  Sigma2D + 0.3 I                   setting 1's low-pass
and the sampler modes SGLD (F disabled) and Adam on the means
(setting 1's SGD optimiser).
"""
import math

import numpy as np
import pytest

from helpers import axis_camera, group_slices, planes_from, raw_o_for, rel_l2
from test_oracle_pins import _fd_scene

POS, GAUSS, LOWPASS = 1, 2, 4


def _cam():
    return axis_camera(width=64, height=64, f=100.0, c=(32.0, 32.0), t=(0, 0, 5))


def _h_grid(c00, c11):
    ys, xs = np.mgrid[0:64, 0:64]
    return ((xs + 0.5 - 32) ** 2) / c00 + ((ys + 0.5 - 32) ** 2) / c11


@pytest.mark.parametrize("variant", [GAUSS, GAUSS | LOWPASS, LOWPASS, POS | GAUSS])
def test_single_component_closed_forms(orc, variant):
    """mu = 0, S = diag(.5, .25, .5), f = 100, z = 5 -> Sigma2D = diag(100, 25)
    (+0.3 on the diagonal with LOWPASS); C = c o T(h), W = 1 - o T with the
    variant's kernel and opacity map (Eq. 7, Eq. 1 for the Gaussian)."""
    raw = 0.4 if variant & POS else raw_o_for(0.6)
    o = 1 / (1 + math.exp(-raw)) if variant & POS else 0.6
    pl = planes_from([dict(mu=(0, 0, 0), log_scale=(math.log(.5), math.log(.25), math.log(.5)),
                           nu=3.0, o=0.6, rgb=(0.8, 0.0, 0.0))])
    pl[11, 0] = raw
    fr = orc.render(pl, 0, _cam(), mode="brute", variant=variant)
    lp = 0.3 if variant & LOWPASS else 0.0
    h = _h_grid(100 + lp, 25 + lp)
    if variant & GAUSS:
        T = np.exp(-h / 2)
        hmax = 2 * math.log(255 * o)
    else:
        T = (1 + h / 3) ** -2.5
        hmax = 3 * ((255 * o) ** 0.4 - 1)
    inside = h <= hmax * (1 - 1e-9)
    outside = h > hmax * (1 + 1e-9)
    np.testing.assert_array_equal(fr.n_contrib[inside], 1)
    np.testing.assert_array_equal(fr.n_contrib[outside], 0)
    np.testing.assert_allclose(fr.rgb[0][inside], 0.8 * o * T[inside], rtol=1e-12)
    np.testing.assert_allclose(fr.final_T[inside], 1 - o * T[inside], rtol=1e-12)
    pr = orc.project(pl, 0, _cam(), variant=variant)
    assert pr.hmax[0] == pytest.approx(hmax, rel=1e-6)  # |o| T(hmax) = 1/255
    assert pr.o[0] == pytest.approx(o, rel=1e-15)


def test_positive_opacity_map(orc):
    for x in (-3.0, -0.2, 0.0, 0.7, 5.0):
        assert orc.opacity_of_v(x, POS) == pytest.approx(1 / (1 + math.exp(-x)), rel=1e-15)
        assert orc.opacity_of_v(x, 0) == pytest.approx(math.tanh(x), rel=1e-15)


def test_t_kernel_tends_to_the_gaussian_variant(orc):
    """nu -> inf recovers the Gaussian.  A scene at nu = 1e4
    renders within 2e-3 of the same scene with the Gaussian kernel where
    both include the same components (the t/Gaussian log-ratio is
    (h^2/4 - h)/nu + O(nu^-2), h <= ~11), and within the 1/255 cut-off
    level elsewhere (a pair at the edge of one kernel's truncation)."""
    rng = np.random.default_rng(3)
    comps = [dict(mu=tuple(rng.uniform(-0.4, 0.4, 3)), log_scale=tuple(rng.normal(-1.2, 0.2, 3)),
                  q=tuple(rng.normal(size=4)), nu=1e4, o=float(rng.uniform(0.2, 0.8)),
                  rgb=tuple(rng.uniform(0.2, 0.8, 3))) for _ in range(12)]
    pl = planes_from(comps)
    a = orc.render(pl, 0, _cam(), mode="brute")
    b = orc.render(pl, 0, _cam(), mode="brute", variant=GAUSS)
    same = a.n_contrib == b.n_contrib
    assert same.mean() > 0.9
    assert np.abs(a.rgb - b.rgb)[:, same].max() < 2e-3
    assert np.abs(a.rgb - b.rgb).max() < 2 / 255
    assert np.abs(a.rgb - b.rgb).max() > 0  # really two kernels


@pytest.mark.parametrize("variant", [POS, GAUSS, LOWPASS, POS | GAUSS | LOWPASS])
def test_variant_backward_matches_finite_differences(orc, variant):
    """Reverse mode of each variant (frozen gating) against central differences
    of <d_rgb, C>; the Gaussian kernel has no nu gradient."""
    sh_degree = 1
    pl, cam = _fd_scene(sh_degree, 7)
    if variant & POS:
        pl[11] = np.abs(pl[11])  # positive components: raw in the sigmoid's working range
    H, W = cam.height, cam.width
    d = np.random.default_rng(11).normal(size=(3, H, W))
    base = orc.render(pl, sh_degree, cam, mode="brute", record_lists=16, variant=variant)
    assert base.n_contrib.max() >= 2 and base.n_contrib.max() < 16
    lists = base.lists
    grad, _ = orc.backward(pl, sh_degree, cam, d, mode="frozen", lists_in=lists, variant=variant)

    def loss(p):
        fr = orc.render(p, sh_degree, cam, mode="frozen", lists_in=lists, variant=variant)
        return float(np.sum(fr.rgb * d))

    fd = np.zeros_like(pl)
    for a in range(pl.shape[0]):
        for i in range(pl.shape[1]):
            st = 1e-6 * max(1.0, abs(pl[a, i]))
            p1, p2 = pl.copy(), pl.copy()
            p1[a, i] += st
            p2[a, i] -= st
            fd[a, i] = (loss(p1) - loss(p2)) / (2 * st)
    for name, sl in group_slices(sh_degree).items():
        if name == "raw_nu" and variant & GAUSS:
            assert np.all(grad[sl] == 0) and np.abs(fd[sl]).max() < 1e-9
            continue
        assert np.linalg.norm(fd[sl]) > 0, name
        assert rel_l2(grad[sl], fd[sl]) < 1e-5, (name, rel_l2(grad[sl], fd[sl]))


def _hp(**kw):
    """Literal Eq. 10 (g = dL/dmu) unless g_adam is passed (R17)."""
    from sss_synth import SGHMCParams

    p = SGHMCParams()
    p.g_adam = False
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def test_sgld_mode_drops_the_friction_term(orc):
    """"if F is disabled, Eq. 10 is simplified to SGLD":
    mu' = mu - eps^2 g + gate N, r' = (1 - eps C) r - eps g + (eta/eps) xi."""
    rng = np.random.default_rng(4)
    n = 40
    pl = planes_from([dict(mu=(0.1, -0.2, 0.3), o=0.001)] * n)
    P = pl.shape[0]
    g = rng.normal(size=(P, n))
    r = rng.normal(size=(3, n))
    hp = _hp(noise=0.0, mu_mode=1)
    out, _, _, r2 = orc.sghmc_step(pl, 0, g, np.zeros((P, n)), np.zeros((P, n)), r, hp)
    eps, C = hp.lr, hp.friction
    np.testing.assert_allclose(out[:3], pl[:3] - eps * eps * g[:3] * hp.grad_scale, rtol=1e-14, atol=1e-18)
    np.testing.assert_allclose(r2, (1 - eps * C) * r - eps * g[:3] * hp.grad_scale, rtol=1e-13)
    hp0 = _hp(noise=0.0)  # the SGHMC default moves by the gated friction term
    out0, *_ = orc.sghmc_step(pl, 0, g, np.zeros((P, n)), np.zeros((P, n)), r, hp0)
    assert np.abs(out0[:3] - out[:3]).max() > 1e-8


def test_adam_mean_mode_first_step(orc):
    """Setting 1's optimiser: Adam on the means; the first bias-corrected
    step is mu - lr g/(|g| + eps_hat) (m^ = g, v^ = g^2)."""
    rng = np.random.default_rng(5)
    n = 30
    pl = planes_from([dict(mu=(0.1, -0.2, 0.3), o=0.5)] * n)
    P = pl.shape[0]
    g = rng.normal(size=(P, n))
    hp = _hp(noise=1e-3, mu_mode=2, grad_scale=1.0)
    out, m2, v2, r2 = orc.sghmc_step(pl, 0, g, np.zeros((P, n)), np.zeros((P, n)), np.zeros((3, n)), hp)
    np.testing.assert_allclose(out[:3], pl[:3] - hp.lr * g[:3] / (np.abs(g[:3]) + hp.adam_eps), rtol=1e-12)
    np.testing.assert_allclose(m2[:3], (1 - hp.beta1) * g[:3], rtol=1e-14)
    assert np.all(r2 == 0)  # no sampler momentum, no noise


def test_positive_variant_relocation(orc):
    """Recycling with sigmoid opacities: o_new from Eq. 12 stays in (0, 1)
    and is stored through the logit."""
    rng = np.random.default_rng(6)
    comps = [dict(mu=tuple(rng.normal(size=3)), log_scale=(-2.0, -2.0, -2.0), o=0.5) for _ in range(60)]
    pl = planes_from(comps)
    pl[11, :50] = rng.uniform(-1.0, 2.0, 50)  # live: sigmoid in (0.27, 0.88)
    pl[11, 50:] = -8.0                         # dead: sigmoid(-8) = 3.4e-4
    P, n = pl.shape
    out, *_, tgt, moved = orc.relocate(pl, 0, np.zeros((P, n)), np.zeros((P, n)), np.zeros((3, n)),
                                       cap_frac=0.5, seed=2, step=1, variant=POS)
    assert moved == 10
    for t in np.unique(tgt[tgt >= 0]):
        N = 1 + int(np.count_nonzero(tgt == t))
        o_old = 1 / (1 + math.exp(-pl[11, t]))
        o_new = 1 / (1 + math.exp(-out[11, t]))
        assert o_new == pytest.approx(1 - (1 - o_old) ** (1 / N), rel=1e-12)
        assert 0 < o_new < o_old
