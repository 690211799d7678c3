"""NEXT-4: the torus scooping toy (Fig. 2) on the GPU.

1. Parity: three iterations of the toy's training loop (TrainStep: project,
   bin, composite, fused L1, backward, SGHMC with the Adam direction) equal
   the oracle's loop (render -> L1 gradient -> backward -> sampler step) for
   the signed 1+/1- fit and the positive-only (sigmoid) 2+ fit.
2. The paper's claim, on seeded runs: one positive and one negative
   component capture the torus topology (a dark hole, a lit ring) and reach a
   lower L1 than two positive components in every seed; two positive
   components fill the hole (underfit); five positive components also beat
   two.
"""
import numpy as np
import pytest

from helpers import rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_pos,n_neg", [(1, 1), (2, 0)])
def test_toy_loop_matches_oracle(orc, sss, n_pos, n_neg):
    import torch

    from paper_2503_10148_b200 import _lib as L
    from paper_2503_10148_b200 import toy
    from paper_2503_10148_b200.step import TrainStep
    from sss_synth.scenes import torus_cameras, torus_init, torus_targets

    cams = torus_cameras(4, 64)
    tg = torus_targets(cams)
    pl = torus_init(n_pos, n_neg, seed=3)
    variant = 0
    if n_neg == 0:
        variant = L.SSS_VARIANT_POSITIVE
        o = np.tanh(pl[11].astype(np.float64))
        pl[11] = np.log(o / (1 - o)).astype(np.float32)
    hp = toy.toy_hparams(0.1, 0.1, seed=3)
    hp.variant = variant
    ts = TrainStep(torch.from_numpy(pl.copy()).cuda(), 0, cams, hp, bin_shift=0, views_per_batch=4,
                   variant=variant)
    tgd = torch.from_numpy(tg).cuda()
    steps = 3
    for _ in range(steps):
        ts.step(tgd)
    torch.cuda.synchronize()
    got = ts.params.planes.cpu().numpy().astype(np.float64)
    # the oracle's loop
    P, n = pl.shape
    p = pl.astype(np.float64)
    m, v, r = np.zeros((P, n)), np.zeros((P, n)), np.zeros((3, n))
    for t in range(1, steps + 1):
        g = np.zeros((P, n))
        for k, cam in enumerate(cams):
            fr = orc.render(p, 0, cam, mode="tiled", variant=variant)
            _, dl = orc.l1_loss_and_grad(fr.rgb, tg[k])
            g += orc.backward(p, 0, cam, dl, mode="tiled", variant=variant)[0]
        hp.step, hp.grad_scale = t, 1.0 / len(cams)
        p, m, v, r = orc.sghmc_step(p, 0, g, m, v, r, hp)
    assert rel_l2(got - pl, p - pl) <= 2e-3, rel_l2(got - pl, p - pl)


def test_negative_component_captures_the_torus_topology(sss):
    from paper_2503_10148_b200 import toy

    seeds = range(6)
    pm, two, five = [], [], []
    for s in seeds:
        pm.append(toy.fit_torus(1, 1, seed=s, iters=1000, lr_mu=0.1, lr=0.1))
        two.append(toy.fit_torus(2, 0, seed=s, iters=1000, lr_mu=0.1, lr=0.1))
        five.append(toy.fit_torus(5, 0, seed=s, iters=1000, lr_mu=0.1, lr=0.1))
    for a, b in zip(pm, two):
        assert a.final_loss < b.final_loss, (a.final_loss, b.final_loss)
    for a, b in zip(five, two):
        assert a.final_loss < b.final_loss
    ratio = lambda rs: np.mean([r.hole / r.ring for r in rs])  # noqa: E731
    assert ratio(pm) < 0.05 < 0.2 < ratio(two), (ratio(pm), ratio(two))  # a dark hole vs a filled one
    assert np.mean([r.ring for r in pm]) > 1.3 * np.mean([r.ring for r in two])  # the ring is lit
    print({"pm": np.mean([r.final_loss for r in pm]), "2+": np.mean([r.final_loss for r in two]),
           "5+": np.mean([r.final_loss for r in five]), "ms_per_iter": pm[0].ms_per_iter})
