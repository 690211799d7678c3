"""NEXT-3 on the GPU (through the C ABI) vs the fp64 oracle: the paper's
ablation variants (R32) — positive sigmoid opacity,
Gaussian kernel, +0.3 low-pass, and their combination — through projection,
binning, forward and backward; the SGLD and Adam-on-means sampler modes; and
recycling with sigmoid opacities.  Same bars as the SSS path: rects, depth
keys and tile lists bit-exact; images 1e-4; gradients rel-L2 1e-3.
"""
import numpy as np
import pytest

from helpers import group_slices, rel_l2
from sss_synth import make_custom_scene, make_optimizer_state

pytestmark = pytest.mark.gpu

POS, GAUSS, LOWPASS = 1, 2, 4
VARIANTS = [POS, GAUSS, LOWPASS, POS | GAUSS | LOWPASS]


def _scene(variant):
    sc = make_custom_scene(5000, 2, 150, 96, n_views=2, seed=71 + variant, layout="blobs", nu_hi=16.0)
    if variant & POS:
        sc.params[11] = np.abs(sc.params[11])  # raw >= 0: sigmoid opacity in [0.5, 1)
    return sc


def _gpu(sss, sc, variant, shift):
    import torch

    params = sss.Params(torch.from_numpy(np.ascontiguousarray(sc.params)).cuda(), sc.sh_degree, variant)
    pr = sss.sss_project(params, sc.cameras)
    bins = sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift)
    assert not sss.sss_check_overflow(bins)
    fr = sss.sss_render_fwd(pr, bins, sc.cameras)
    torch.cuda.synchronize()
    return params, pr, bins, fr


@pytest.mark.parametrize("variant", VARIANTS)
def test_variant_projection_and_bins(orc, sss, variant):
    sc = _scene(variant)
    _, pr, bins, _ = _gpu(sss, sc, variant, 0)
    for v, cam in enumerate(sc.cameras):
        o = orc.project(sc.params, sc.sh_degree, cam, variant=variant)
        rect = pr.rect[v].cpu().numpy().astype(np.int32)
        vis = o.n_tiles > 0
        assert np.array_equal(vis, rect[:, 0] <= rect[:, 2])
        assert np.array_equal(rect[vis], o.rect[vis])
        rec = pr.rec[v].cpu().numpy()
        for k, name in [(2, "A"), (5, "hmax")]:
            g, ref = rec[vis, k], getattr(o, name)[vis]
            assert (g.view(np.uint32) != ref.view(np.uint32)).mean() <= 1e-3, name
            np.testing.assert_allclose(g, ref, rtol=1e-6)
        np.testing.assert_allclose(rec[vis, 6], o.o[vis], rtol=1e-6, atol=1e-7)
        if variant & GAUSS:
            assert np.all(rec[vis, 7] == 0)  # inv_nu = 0 marks the Gaussian kernel
        counts, _, _ = orc.bin_sort(sc.params, sc.sh_degree, cam, want_keys=False, variant=variant)
        rg = bins.ranges[v].cpu().numpy()
        np.testing.assert_array_equal(rg[:, 1] - rg[:, 0], counts)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("shift", [0, 2])
def test_variant_render_and_backward(orc, sss, variant, shift):
    import torch

    from test_gpu_parity import _check_frame

    sc = _scene(variant)
    params, pr, bins, fr = _gpu(sss, sc, variant, shift)
    cam0 = sc.cameras[0]
    d = np.random.default_rng(3).normal(size=(sc.n_views, 3, cam0.height, cam0.width)).astype(np.float32)
    grad = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    g = grad.planes.cpu().numpy().astype(np.float64)
    ref = np.zeros_like(g)
    for v, cam in enumerate(sc.cameras):
        o = orc.render(sc.params, sc.sh_degree, cam, mode="tiled", variant=variant)
        _check_frame(f"variant{variant}", fr.rgb[v].cpu().numpy(), fr.final_T[v].cpu().numpy(),
                     fr.n_contrib[v].cpu().numpy(), o)
        ref += orc.backward(sc.params, sc.sh_degree, cam, d[v].astype(np.float64), mode="tiled",
                            variant=variant)[0]
    for grp, sl in group_slices(sc.sh_degree).items():
        if grp == "raw_nu" and variant & GAUSS:
            assert np.all(g[sl] == 0)
            continue
        assert rel_l2(g[sl], ref[sl]) <= 1e-3, (grp, rel_l2(g[sl], ref[sl]))


@pytest.mark.parametrize("mu_mode", [1, 2])
@pytest.mark.parametrize("variant", [0, POS])
def test_sampler_modes(orc, sss, mu_mode, variant):
    import torch

    from sss_synth import sghmc_params_for
    from test_gpu_parity import _hp32

    sc = make_custom_scene(30000, 1, 32, 32, seed=81)
    r, m, v = make_optimizer_state(sc, seed=3)
    rng = np.random.default_rng(4)
    grad = (rng.normal(size=sc.params.shape) * 1e-2).astype(np.float32)
    sc.params[11] = np.arctanh(rng.uniform(-0.03, 0.03, sc.n)).astype(np.float32)
    if variant & POS:
        sc.params[11] = rng.uniform(-7.0, -4.0, sc.n).astype(np.float32)  # sigmoid ~ 1e-3 .. 2e-2
    hp = _hp32(sghmc_params_for(sc, step=2, seed=17, noise=1e-4, grad_scale=0.5, mu_mode=mu_mode,
                                variant=variant, eps_o=0.01, eps_sigma=0.01))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    params = sss.Params(dev(sc.params), 1, variant)
    mm, vv, rr = sss.Params(dev(m), 1, variant), sss.Params(dev(v), 1, variant), dev(r)
    sss.sss_sghmc_step(params, sss.Params(dev(grad), 1, variant), mm, vv, rr, hp)
    torch.cuda.synchronize()
    p_ref, m_ref, v_ref, r_ref = orc.sghmc_step(sc.params, 1, grad, m, v, r, hp)
    got = params.planes.cpu().numpy().astype(np.float64)
    # fp32 state: the mean update sums up to three rounded fp32 terms, so the
    # per-element bound is two ulps of the result plus 1e-5 of the update
    ulp = np.spacing(np.abs(p_ref).astype(np.float32)).astype(np.float64)
    bound = 2 * ulp + 1e-5 * np.abs(p_ref - sc.params)
    assert np.all(np.abs(got - p_ref) <= bound + 1e-30), float((np.abs(got - p_ref) / (bound + 1e-30)).max())
    assert rel_l2(mm.planes.cpu().numpy(), m_ref) <= 1e-5
    if mu_mode == 1:
        assert rel_l2(rr.cpu().numpy() - r, r_ref - r) <= 1e-5


def test_positive_variant_relocation(orc, sss):
    import torch

    sc = make_custom_scene(20000, 0, 16, 16, seed=91)
    rng = np.random.default_rng(5)
    pl = sc.params.copy()
    pl[11] = rng.uniform(-1.0, 2.0, sc.n).astype(np.float32)
    dead = rng.random(sc.n) < 0.05
    pl[11, dead] = np.float32(-8.0)
    P, n = pl.shape
    z = lambda *s: np.zeros(s, np.float32)  # noqa: E731
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    params = sss.Params(dev(pl), 0, POS)
    mm, vv, rr = sss.Params(dev(z(P, n)), 0, POS), sss.Params(dev(z(P, n)), 0, POS), dev(z(3, n))
    tgt = torch.empty(n, dtype=torch.int32, device="cuda")
    moved = sss.sss_relocate(params, mm, vv, rr, target_of=tgt, seed=3, step=2)
    torch.cuda.synchronize()
    o_pl, *_, o_t, o_n = orc.relocate(pl, 0, z(P, n), z(P, n), z(3, n), seed=3, step=2, variant=POS)
    assert int(moved.item()) == o_n > 0
    np.testing.assert_array_equal(tgt.cpu().numpy(), o_t)
    np.testing.assert_allclose(params.planes.cpu().numpy(), o_pl, rtol=1e-6, atol=1e-6)
