"""NEXT-4 — the torus scooping toy of Fig. 2 on the GPU.

"We use a torus with only ambient lighting and frontal views ... We
initialize the component means near the center.  Only using positive
densities either underfits if two components are used, or requires at least
5 components to capture the topology correctly.  In contrast, we only need
two components (one positive and one negative)."

`fit_torus` runs the product's training loop (TrainStep: project, bin,
composite, fused-L1 backward, SGHMC/Adam — every step in the CUDA kernels)
on the silhouettes of sss_synth.torus_targets, with signed tanh opacities
(SSS) or, for the positive-only fits, the sigmoid opacity of the
POSITIVE variant (R32).  The targets and initialisation are
inputs (sss_synth); this module only drives the loop.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import _lib as L
from .step import TrainStep


@dataclass
class ToyResult:
    n_pos: int
    n_neg: int
    seed: int
    losses: List[float] = field(default_factory=list)
    final_loss: float = float("nan")
    params: np.ndarray = None
    ms_per_iter: float = float("nan")
    hole: float = float("nan")  # mean rendered intensity in the torus hole (target 0)
    ring: float = float("nan")  # mean rendered intensity on the ring (target = the torus colour)


def toy_hparams(lr_mu: float = 0.1, lr: float = 0.1, seed: int = 0):
    """Sampler settings of the toy: Eq. 10 with the Adam direction as g
    (R17's g_adam), the friction/noise gate of the paper (k = 100, t = 0.005)
    and Adam on every other group."""
    from sss_synth import SGHMCParams

    return SGHMCParams(lr=lr_mu, friction=0.1, noise=0.0, g_adam=True, lr_scale=lr, lr_rot=lr,
                       lr_nu=lr, lr_opacity=lr, lr_sh=lr, seed=seed)


def fit_torus(n_pos: int, n_neg: int, seed: int = 0, iters: int = 1000, size: int = 64,
              n_views: int = 4, lr_mu: float = 0.1, lr: float = 0.1, device="cuda") -> ToyResult:
    from sss_synth.scenes import torus_cameras, torus_init, torus_targets

    cams = torus_cameras(n_views, size)
    tg = torch.from_numpy(torus_targets(cams)).to(device)
    planes = torus_init(n_pos, n_neg, seed)
    variant = 0
    if n_neg == 0:  # positive-only fit: sigmoid opacity, same initial |o|
        variant = L.SSS_VARIANT_POSITIVE
        o = np.tanh(planes[11].astype(np.float64))
        planes[11] = np.log(o / (1.0 - o)).astype(np.float32)
    hp = toy_hparams(lr_mu, lr, seed)
    hp.variant = variant
    ts = TrainStep(torch.from_numpy(planes).to(device), 0, cams, hp, bin_shift=0,
                   views_per_batch=n_views, variant=variant)
    res = ToyResult(n_pos, n_neg, seed)
    losses = torch.zeros(iters, device=device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(iters):
        loss = ts.step(tg)
        losses[it] = loss[0] / n_views
    e1.record()
    torch.cuda.synchronize()
    if ts.overflowed():
        raise RuntimeError("toy bin capacity overflow")
    res.ms_per_iter = e0.elapsed_time(e1) / iters
    res.losses = losses.cpu().tolist()
    res.final_loss = float(np.mean(res.losses[-20:]))
    res.params = ts.params.planes.cpu().numpy()
    # topology check on the last rendered frames: the hole must be dark
    from sss_synth.scenes import TORUS_R, TORUS_r

    img = ts.frame.rgb[:n_views].mean(dim=1).cpu().numpy()  # [V][H][W] intensity
    tgt = tg.mean(dim=1).cpu().numpy()
    c = size / 2.0
    ys, xs = np.mgrid[0:size, 0:size]
    rad = np.hypot(xs + 0.5 - c, ys + 0.5 - c)
    f = cams[0].fx / 3.0  # pixels per world unit at the torus plane
    hole = rad < 0.6 * (TORUS_R - TORUS_r) * f
    res.hole = float(img[:, hole].mean())
    res.ring = float(img[tgt > 0].mean())
    return res


def summarize(results: List[ToyResult]) -> dict:
    out = {}
    for r in results:
        key = f"{r.n_pos}+{r.n_neg}-"
        out.setdefault(key, []).append((r.final_loss, r.hole, r.ring))
    return {k: {"loss_mean": float(np.mean([x[0] for x in v])), "loss_min": float(np.min([x[0] for x in v])),
                "loss_max": float(np.max([x[0] for x in v])), "hole": float(np.mean([x[1] for x in v])),
                "ring": float(np.mean([x[2] for x in v])), "n": len(v)}
            for k, v in out.items()}
