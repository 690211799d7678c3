"""NEXT-1 on the GPU (through the C ABI) vs the fp64 oracle: the image part of
Eq. 8 (L1 + D-SSIM) with its gradient, the regularizer gradients folded into
the sampler step, and a full Eq. 8 training step.

Tolerances: loss values 1e-5 relative; image gradients relative L2 1e-4
(fp32 moments of 121-tap windows against fp64); parameter updates as in
test_gpu_parity.py::test_sghmc_parity.  Targets are kept >= 1e-3 from the
render so both sides take the same L1 sign (R20).
"""
import numpy as np
import pytest

from helpers import group_slices, rel_l2
from sss_synth import make_custom_scene, make_optimizer_state

pytestmark = pytest.mark.gpu


def _pair(V, H, W, seed):
    rng = np.random.default_rng(seed)
    x = rng.random((V, 3, H, W)).astype(np.float32)
    y = rng.random((V, 3, H, W)).astype(np.float32)
    close = np.abs(x - y) < 1e-3
    y[close] = np.where(x[close] > 0.5, x[close] - 2e-3, x[close] + 2e-3)
    return x, y


@pytest.mark.parametrize("shape", [(1, 11, 11), (3, 70, 53), (2, 97, 130), (1, 256, 200)])
@pytest.mark.parametrize("eps", [0.0, 0.2, 1.0])
def test_image_loss_parity(orc, sss, shape, eps):
    import torch

    V, H, W = shape
    x, y = _pair(V, H, W, seed=H * 7 + W)
    loss = torch.zeros(1, device="cuda")
    d = sss.sss_image_loss(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), eps, loss=loss)
    torch.cuda.synchronize()
    d = d.cpu().numpy()
    lref = 0.0
    for v in range(V):
        l, dref = orc.image_loss(x[v], y[v], eps)
        lref += l
        assert rel_l2(d[v], dref) <= 1e-4, (v, rel_l2(d[v], dref))
    assert loss.item() == pytest.approx(lref, rel=1e-5, abs=1e-7)


def test_image_loss_textured_images(orc, sss):
    """Smooth, correlated images (SSIM far from 0): a render-like x and a
    perturbed copy y, where the variance terms carry the gradient."""
    import torch

    rng = np.random.default_rng(9)
    H, W = 64, 48
    yy, xx = np.mgrid[0:H, 0:W]
    base = 0.5 + 0.3 * np.sin(xx / 5.0)[None] * np.cos(yy / 7.0)[None] * np.array([1.0, 0.7, -0.4])[:, None, None]
    x = base[None].astype(np.float32)
    y = (base + 0.05 * rng.normal(size=base.shape))[None].astype(np.float32)
    loss = torch.zeros(1, device="cuda")
    d = sss.sss_image_loss(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 0.2, loss=loss)
    torch.cuda.synchronize()
    l, dref = orc.image_loss(x[0], y[0], 0.2)
    assert rel_l2(d.cpu().numpy()[0], dref) <= 1e-4
    assert loss.item() == pytest.approx(l, rel=1e-5)


def test_image_loss_errors(sss):
    import torch

    from paper_2503_10148_b200 import _lib as L

    x = torch.zeros((1, 3, 10, 40), device="cuda")
    with pytest.raises(L.SSSError) as e:
        sss.sss_image_loss(x, x, 0.2)
    assert e.value.status == L.SSS_ERR_SHAPE
    with pytest.raises(L.SSSError) as e:
        sss.sss_image_loss(x, x, -0.1)
    assert e.value.status == L.SSS_ERR_ARG
    d = sss.sss_image_loss(x, x, 0.0)  # L1 only works below the window size
    torch.cuda.synchronize()
    assert float(d.abs().max()) == 0.0


def test_sghmc_regularizers_parity(orc, sss):
    import torch

    from sss_synth import sghmc_params_for
    from test_gpu_parity import _hp32

    sc = make_custom_scene(20000, 3, 32, 32, seed=41)
    r, m, v = make_optimizer_state(sc, seed=6)
    rng = np.random.default_rng(12)
    grad = (rng.normal(size=sc.params.shape) * 1e-2).astype(np.float32)
    hp = _hp32(sghmc_params_for(sc, step=3, seed=9, noise=1e-4, grad_scale=0.25, eps_o=0.02,
                                eps_sigma=0.05))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    params = sss.Params(dev(sc.params), 3)
    mm, vv, rr = sss.Params(dev(m), 3), sss.Params(dev(v), 3), dev(r)
    sss.sss_sghmc_step(params, sss.Params(dev(grad), 3), mm, vv, rr, hp)
    torch.cuda.synchronize()
    p_ref, m_ref, v_ref, _ = orc.sghmc_step(sc.params, 3, grad, m, v, r, hp)
    got = params.planes.cpu().numpy().astype(np.float64)
    from gpu_helpers import update_ulp

    ulp = update_ulp(p_ref, sc.params)
    bound = ulp + 1e-5 * np.abs(p_ref - sc.params)
    assert np.all(np.abs(got - p_ref) <= bound + 1e-30)
    assert rel_l2(mm.planes.cpu().numpy(), m_ref) <= 1e-5
    assert rel_l2(vv.planes.cpu().numpy(), v_ref) <= 1e-5
    # the regularizers changed the moments of log_scale and raw_opacity
    _, m0, _, _ = orc.sghmc_step(sc.params, 3, grad, m, v, r, _hp32(sghmc_params_for(
        sc, step=3, seed=9, noise=1e-4, grad_scale=0.25)))
    assert rel_l2(m_ref[3:6], m0[3:6]) > 1e-3 and rel_l2(m_ref[11:12], m0[11:12]) > 1e-3


def test_trainstep_full_eq8(orc, sss):
    """TrainStep with the full Eq. 8 objective (eps_D = 0.2, eps_o, eps_Sigma)
    equals the oracle's iteration: per view image loss -> backward on its
    image gradient, summed, grad_scale 1/V, regularizers in the step."""
    import torch

    from paper_2503_10148_b200.step import TrainStep
    from sss_synth import make_targets, sghmc_params_for
    from test_gpu_parity import _hp32

    sc = make_custom_scene(3000, 1, 80, 64, n_views=3, seed=29, layout="blobs", nu_hi=16.0)
    tg = make_targets(sc)
    hp = _hp32(sghmc_params_for(sc, step=1, seed=5, noise=0.0, eps_o=0.01, eps_sigma=0.01))
    ts = TrainStep(torch.from_numpy(sc.params).cuda(), 1, sc.cameras, hp, bin_shift=1,
                   views_per_batch=2, eps_dssim=0.2)
    loss = ts.step(torch.from_numpy(tg).cuda())
    torch.cuda.synchronize()
    assert not ts.overflowed()
    g = ts.grad.planes.cpu().numpy()
    ref, lref = 0, 0.0
    for v, cam in enumerate(sc.cameras):
        fr = orc.render(sc.params, 1, cam, mode="tiled")
        l, dl = orc.image_loss(fr.rgb, tg[v], 0.2)
        lref += l
        ref = ref + orc.backward(sc.params, 1, cam, dl, mode="tiled")[0]
    assert abs(loss.item() - lref) <= 1e-4 * lref
    for grp, sl in group_slices(1).items():
        assert rel_l2(g[sl], ref[sl]) <= 2e-3, grp  # L1 sign ties (R20) add a little
    P, n = sc.params.shape
    p_ref, _, _, _ = orc.sghmc_step(sc.params, 1, ref, np.zeros((P, n)), np.zeros((P, n)),
                                    np.zeros((3, n)), hp)
    got = ts.params.planes.cpu().numpy().astype(np.float64)
    assert rel_l2(got[3:] - sc.params[3:], p_ref[3:] - sc.params[3:]) <= 5e-3
