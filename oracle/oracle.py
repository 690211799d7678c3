"""ctypes wrapper of the fp64 SSS oracle — TEST INFRASTRUCTURE ONLY.

See oracle/sss_oracle.cpp for the definitions and their PAPER.md citations.
All parameters are passed as float64 copies of the (float32) scene arrays, so
the oracle sees exactly the values the CUDA path sees, promoted exactly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sss_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -fopenmp -ffp-contract=off)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
           "-fPIC", "-shared", _SRC, "-o", tmp]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB)
    return _LIB


class _Cam(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("z_near", C.c_double)]


class _Params(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_degree", C.c_int32), ("variant", C.c_int32),
                ("planes", C.POINTER(C.c_double))]


class _ProjOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in
                ("mx", "my", "A", "B2", "C", "hmax", "depth", "rect", "n_tiles", "cull", "p",
                 "mean2d", "cov2d", "conic", "nu", "o", "color")]


class _HP(C.Structure):
    _fields_ = [("lr", C.c_double), ("friction", C.c_double), ("noise", C.c_double),
                ("gate_k", C.c_double), ("gate_t", C.c_double), ("burn_in", C.c_int32),
                ("g_adam", C.c_int32), ("lr_scale", C.c_double), ("lr_rot", C.c_double),
                ("lr_nu", C.c_double), ("lr_opacity", C.c_double), ("lr_sh", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("adam_eps", C.c_double),
                ("grad_scale", C.c_double), ("step", C.c_int64), ("seed", C.c_uint64),
                ("eps_o", C.c_double), ("eps_sigma", C.c_double), ("mu_mode", C.c_int32),
                ("variant", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, p, i32, i64 = C.c_double, C.c_void_p, C.c_int32, C.c_int64
        for name, res, args in [
            ("orc_num_planes", C.c_int, [C.c_int]),
            ("orc_nu_of", d, [d]), ("orc_opacity_of", d, [d]),
            ("orc_t2d", d, [d, d]), ("orc_t3d", d, [d, d]), ("orc_dT_dh", d, [d, d]),
            ("orc_dT_dnu", d, [d, d, C.c_int]),
            ("orc_sh_basis", None, [C.c_int, p, p]), ("orc_cov3d", None, [p, p, p]),
            ("orc_project", C.c_int, [p, p, p]),
            ("orc_bin", i64, [p, p, p, p, p]),
            ("orc_tile_lists", i64, [p, p, i32, p, p, p, i64]),
            ("orc_render", C.c_int, [p, p, p, i32, p, p, p, p, p, p, i32, i32, p]),
            ("orc_backward", C.c_int, [p, p, p, p, i32, i32, p, p, p, i32, i32, p]),
            ("orc_philox4x32_10", None, [p, p, p]),
            ("orc_normals3", None, [C.c_uint64, i64, i64, p]),
            ("orc_sghmc_step", C.c_int, [i64, i32, p, p, p, p, p, p]),
            ("orc_image_loss", d, [p, p, i32, i32, d, p]),
            ("orc_regularizers", None, [i64, i32, p, p, i32]),
            ("orc_opacity_of_v", d, [d, i32]),
            ("orc_beta", d, [d, d]), ("orc_reloc_opacity", d, [d, i32]),
            ("orc_reloc_K", d, [i32, d, d]), ("orc_reloc_scale", d, [d, d, d, i32]),
            ("orc_relocate", i64, [i64, i32, p, p, p, p, d, d, i32, C.c_uint64, i64, p, i32]),
        ]:
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _cam(cam) -> _Cam:
    c = _Cam()
    R = np.asarray(cam.R, np.float64).reshape(9)
    t = np.asarray(cam.t, np.float64).reshape(3)
    for k in range(9):
        c.R[k] = float(R[k])
    for k in range(3):
        c.t[k] = float(t[k])
    # the CUDA path takes fp32 intrinsics: use exactly those values
    c.fx, c.fy = float(np.float32(cam.fx)), float(np.float32(cam.fy))
    c.cx, c.cy = float(np.float32(cam.cx)), float(np.float32(cam.cy))
    c.width, c.height = int(cam.width), int(cam.height)
    c.z_near = float(np.float32(cam.z_near))
    return c


class _P:
    """Keeps the fp64 plane copy alive while ctypes holds a pointer to it."""

    def __init__(self, planes, sh_degree, variant=0):
        self.arr = np.ascontiguousarray(np.asarray(planes, np.float64))
        self.s = _Params(self.arr.shape[1], int(sh_degree), int(variant),
                         self.arr.ctypes.data_as(C.POINTER(C.c_double)))

    @property
    def ref(self):
        return C.byref(self.s)


# --------------------------------------------------------------- primitives
def nu_of(raw):
    return lib().orc_nu_of(float(raw))


def opacity_of_v(raw, variant):
    return lib().orc_opacity_of_v(float(raw), int(variant))


def opacity_of(raw):
    return lib().orc_opacity_of(float(raw))


def t2d(h, nu):
    return lib().orc_t2d(float(h), float(nu))


def t3d(h, nu):
    return lib().orc_t3d(float(h), float(nu))


def dT_dh(h, nu):
    return lib().orc_dT_dh(float(h), float(nu))


def dT_dnu(h, nu, paper=False):
    return lib().orc_dT_dnu(float(h), float(nu), int(paper))


def sh_basis(deg, d):
    d = np.ascontiguousarray(np.asarray(d, np.float64))
    out = np.zeros(16, np.float64)
    lib().orc_sh_basis(int(deg), _ptr(d), _ptr(out))
    return out[: (deg + 1) ** 2]


def cov3d(log_scale, q):
    s = np.ascontiguousarray(np.asarray(log_scale, np.float64))
    qq = np.ascontiguousarray(np.asarray(q, np.float64))
    out = np.zeros(9, np.float64)
    lib().orc_cov3d(_ptr(s), _ptr(qq), _ptr(out))
    return out.reshape(3, 3)


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(np.asarray(ctr, np.uint32))
    k = np.ascontiguousarray(np.asarray(key, np.uint32))
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def normals3(seed, i, step):
    out = np.zeros(3, np.float64)
    lib().orc_normals3(int(seed), int(i), int(step), _ptr(out))
    return out


# --------------------------------------------------------------- hot path
@dataclass
class Projection:
    mx: np.ndarray
    my: np.ndarray
    A: np.ndarray
    B2: np.ndarray
    C: np.ndarray
    hmax: np.ndarray
    depth: np.ndarray
    rect: np.ndarray
    n_tiles: np.ndarray
    cull: np.ndarray
    p: np.ndarray
    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    nu: np.ndarray
    o: np.ndarray
    color: np.ndarray


def project(planes, sh_degree, cam, variant=0) -> Projection:
    P = _P(planes, sh_degree, variant)
    n = P.arr.shape[1]
    f32 = lambda: np.zeros(n, np.float32)  # noqa: E731
    pr = Projection(mx=f32(), my=f32(), A=f32(), B2=f32(), C=f32(), hmax=f32(), depth=f32(),
                    rect=np.zeros((n, 4), np.int32), n_tiles=np.zeros(n, np.int32),
                    cull=np.zeros(n, np.int32), p=np.zeros((n, 3)), mean2d=np.zeros((n, 2)),
                    cov2d=np.zeros((n, 3)), conic=np.zeros((n, 3)), nu=np.zeros(n),
                    o=np.zeros(n), color=np.zeros((n, 3)))
    po = _ProjOut(*[pr.__dict__[k].ctypes.data for k in
                    ("mx", "my", "A", "B2", "C", "hmax", "depth", "rect", "n_tiles", "cull", "p",
                     "mean2d", "cov2d", "conic", "nu", "o", "color")])
    c = _cam(cam)
    lib().orc_project(P.ref, C.byref(c), C.byref(po))
    return pr


def tiles_of(cam):
    return (cam.width + 15) // 16, (cam.height + 15) // 16


def bin_sort(planes, sh_degree, cam, want_keys=True, variant=0):
    """Returns (tile_counts[tiles], ids[M], keys[M] or None)."""
    P = _P(planes, sh_degree, variant)
    c = _cam(cam)
    tw, th = tiles_of(cam)
    counts = np.zeros(tw * th, np.int32)
    M = lib().orc_bin(P.ref, C.byref(c), _ptr(counts), None, None)
    ids = np.zeros(M, np.int32)
    keys = np.zeros(M, np.uint64) if want_keys else None
    lib().orc_bin(P.ref, C.byref(c), _ptr(counts), _ptr(ids), _ptr(keys) if want_keys else None)
    return counts, ids, keys


def tile_lists(planes, sh_degree, cam, tiles, variant=0):
    P = _P(planes, sh_degree, variant)
    c = _cam(cam)
    sel = np.ascontiguousarray(np.asarray(tiles, np.int32))
    counts = np.zeros(len(sel), np.int32)
    M = lib().orc_tile_lists(P.ref, C.byref(c), len(sel), _ptr(sel), _ptr(counts), None, 0)
    ids = np.zeros(max(M, 1), np.int32)
    lib().orc_tile_lists(P.ref, C.byref(c), len(sel), _ptr(sel), _ptr(counts), _ptr(ids), M)
    out, o = [], 0
    for k in counts:
        out.append(ids[o:o + k].copy())
        o += k
    return out


MODES = {"brute": 0, "tiled": 1, "frozen": 2}


@dataclass
class Frame:
    rgb: np.ndarray  # [3][H][W] (or [3][n_sel])
    final_T: np.ndarray
    n_contrib: np.ndarray
    tie: np.ndarray
    lists: np.ndarray = None


def render(planes, sh_degree, cam, bg=(0.0, 0.0, 0.0), mode="tiled", lists_in=None,
           record_lists=0, pixels=None, variant=0) -> Frame:
    """Forward composite (Eq. 7).  `pixels`: optional flat pixel indices."""
    P = _P(planes, sh_degree, variant)
    c = _cam(cam)
    H, W = cam.height, cam.width
    bgv = np.ascontiguousarray(np.asarray(bg, np.float64))
    if pixels is not None:
        sel = np.ascontiguousarray(np.asarray(pixels, np.int32))
        shape = (len(sel),)
    else:
        sel = None
        shape = (H, W)
    rgb = np.zeros((3,) + shape)
    T = np.zeros(shape)
    nc = np.zeros(shape, np.int32)
    tie = np.zeros(shape)
    cap = 0
    lin = None
    if mode == "frozen":
        lin = np.ascontiguousarray(lists_in, dtype=np.int32)
        cap = lin.shape[-1]
    lout = None
    if record_lists:
        cap = int(record_lists) if lin is None else cap
        lout = np.zeros(shape + (cap,), np.int32)
    lib().orc_render(P.ref, C.byref(c), _ptr(bgv), MODES[mode], _ptr(rgb), _ptr(T), _ptr(nc),
                     _ptr(tie), _ptr(lin) if lin is not None else None,
                     _ptr(lout) if lout is not None else None, cap,
                     len(sel) if sel is not None else 0, _ptr(sel) if sel is not None else None)
    return Frame(rgb=rgb, final_T=T, n_contrib=nc, tie=tie, lists=lout)


def backward(planes, sh_degree, cam, d_rgb, bg=(0.0, 0.0, 0.0), mode="tiled", lists_in=None,
             nu_grad_paper=False, want_g2d=False, pixels=None, variant=0):
    """Reverse mode of render(): (grad planes [P][n] fp64, g2d [n][10] or None).
    `pixels`: optional flat pixel indices; then d_rgb is [3][len(pixels)]."""
    P = _P(planes, sh_degree, variant)
    c = _cam(cam)
    n = P.arr.shape[1]
    bgv = np.ascontiguousarray(np.asarray(bg, np.float64))
    d = np.ascontiguousarray(np.asarray(d_rgb, np.float64))
    grads = np.zeros(P.arr.shape)
    g2d = np.zeros((n, 10)) if want_g2d else None
    cap = 0
    lin = None
    if mode == "frozen":
        lin = np.ascontiguousarray(lists_in, dtype=np.int32)
        cap = lin.shape[-1]
    sel = None if pixels is None else np.ascontiguousarray(np.asarray(pixels, np.int32))
    lib().orc_backward(P.ref, C.byref(c), _ptr(bgv), _ptr(d), MODES[mode], int(nu_grad_paper),
                       _ptr(grads), _ptr(g2d) if g2d is not None else None,
                       _ptr(lin) if lin is not None else None, cap,
                       len(sel) if sel is not None else 0, _ptr(sel) if sel is not None else None)
    return grads, g2d


def l1_loss_and_grad(rgb, target):
    """Eq. 8's L1 term for one view: mean |C - target|, dL/dC = sign/(3P)."""
    diff = np.asarray(rgb, np.float64) - np.asarray(target, np.float64)
    return float(np.mean(np.abs(diff))), np.sign(diff) / diff.size


def image_loss(rgb, target, eps_dssim):
    """Image part of Eq. 8 for one view: (1 - eps) L1 + eps (1 - SSIM) and
    dL/dC (see orc_image_loss).  rgb, target: [3][H][W]."""
    x = np.ascontiguousarray(np.asarray(rgb, np.float64))
    y = np.ascontiguousarray(np.asarray(target, np.float64))
    assert x.shape == y.shape and x.ndim == 3 and x.shape[0] == 3
    d = np.zeros_like(x)
    val = lib().orc_image_loss(_ptr(x), _ptr(y), x.shape[1], x.shape[2], float(eps_dssim), _ptr(d))
    return float(val), d


def ssim(a, b):
    """Mean SSIM of two [3][H][W] images (1 - the D-SSIM term)."""
    return 1.0 - image_loss(a, b, 1.0)[0]


def regularizers(planes, sh_degree, variant=0):
    """(sum_i |o_i|, sum_i sum_j sqrt(lambda_ij)) of Eq. 8."""
    pl = np.ascontiguousarray(np.asarray(planes, np.float64))
    out = np.zeros(2)
    lib().orc_regularizers(pl.shape[1], int(sh_degree), _ptr(pl), _ptr(out), int(variant))
    return float(out[0]), float(out[1])


def beta(x, y):
    return lib().orc_beta(float(x), float(y))


def reloc_opacity(o_old, N):
    return lib().orc_reloc_opacity(float(o_old), int(N))


def reloc_K(N, o_new, nu_new):
    return lib().orc_reloc_K(int(N), float(o_new), float(nu_new))


def reloc_scale(o_old, nu_old, nu_new, N):
    return lib().orc_reloc_scale(float(o_old), float(nu_old), float(nu_new), int(N))


def relocate(planes, sh_degree, m, v, r, threshold=0.005, cap_frac=0.05, n_max=32, seed=0, step=1,
             variant=0):
    """One recycling pass (orc_relocate) on fp64 copies; returns
    (planes, m, v, r, target_of, moved)."""
    pl = np.ascontiguousarray(np.asarray(planes, np.float64)).copy()
    mm = np.ascontiguousarray(np.asarray(m, np.float64)).copy()
    vv = np.ascontiguousarray(np.asarray(v, np.float64)).copy()
    rr = np.ascontiguousarray(np.asarray(r, np.float64)).copy()
    tg = np.zeros(pl.shape[1], np.int32)
    moved = lib().orc_relocate(pl.shape[1], int(sh_degree), _ptr(pl), _ptr(mm), _ptr(vv), _ptr(rr),
                               float(threshold), float(cap_frac), int(n_max), int(seed), int(step),
                               _ptr(tg), int(variant))
    return pl, mm, vv, rr, tg, int(moved)


def sghmc_step(planes, sh_degree, grad, m, v, r, hp):
    """One a7 step on fp64 copies; returns (planes, m, v, r) updated."""
    pl = np.ascontiguousarray(np.asarray(planes, np.float64)).copy()
    g = np.ascontiguousarray(np.asarray(grad, np.float64))
    mm = np.ascontiguousarray(np.asarray(m, np.float64)).copy()
    vv = np.ascontiguousarray(np.asarray(v, np.float64)).copy()
    rr = np.ascontiguousarray(np.asarray(r, np.float64)).copy()
    h = _HP(hp.lr, hp.friction, hp.noise, hp.gate_k, hp.gate_t, int(hp.burn_in), int(hp.g_adam),
            hp.lr_scale, hp.lr_rot, hp.lr_nu, hp.lr_opacity, hp.lr_sh, hp.beta1, hp.beta2,
            hp.adam_eps, hp.grad_scale, int(hp.step), int(hp.seed),
            getattr(hp, "eps_o", 0.0), getattr(hp, "eps_sigma", 0.0), int(getattr(hp, "mu_mode", 0)),
            int(getattr(hp, "variant", 0)))
    lib().orc_sghmc_step(pl.shape[1], int(sh_degree), _ptr(pl), _ptr(g), _ptr(mm), _ptr(vv),
                         _ptr(rr), C.byref(h))
    return pl, mm, vv, rr
