"""GPU-side helpers for the parity tests: run the CUDA path through the C ABI
(paper_2503_10148_b200.api) on a seeded scene and return numpy arrays."""
import numpy as np
import torch

import paper_2503_10148_b200 as P


def to_dev(scene):
    planes = torch.from_numpy(np.ascontiguousarray(scene.params, np.float32)).cuda()
    return P.Params(planes, scene.sh_degree)


def gpu_forward(scene, cams=None, bin_shift=0, bg=(0.0, 0.0, 0.0), keys=False, params=None):
    cams = scene.cameras if cams is None else cams
    params = to_dev(scene) if params is None else params
    pr = P.sss_project(params, cams)
    bins = P.sss_bin_sort(pr, cams, bin_shift=bin_shift, keys=keys)
    assert not P.sss_check_overflow(bins)
    fr = P.sss_render_fwd(pr, bins, cams, bg=bg)
    torch.cuda.synchronize()
    return params, pr, bins, fr


def bin_lists(bins, v, n_bins):
    """Per-bin id lists of view v (numpy)."""
    ids = bins.ids[v].cpu().numpy()
    rg = bins.ranges[v].cpu().numpy()
    return [ids[rg[b, 0]:rg[b, 1]] for b in range(n_bins)]


def ulp_diff(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(a - b)


def update_ulp(p_ref, p_old):
    """One fp32 ulp of the coarser of the old and new parameter binades: the
    kernels form mu' from mu in two fp32 roundings (each <= 1/2 ulp of its
    larger operand), so an update that crosses a power of two can be off by
    half an ulp of the old binade plus half of the new one."""
    big = np.maximum(np.abs(p_ref), np.abs(p_old)).astype(np.float32)
    return np.spacing(big).astype(np.float64)
