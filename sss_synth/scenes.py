"""Seeded synthetic SSS scenes shaped like BASELINE.json's five configs.

Recipe (restated in DESIGN.md "Input recipe"):

* Host numpy ``Generator(PCG64(20250313 + config))`` draws in float64, cast
  once to float32, stored as SoA planes ``[P][n]`` with
  ``P = 12 + 3K`` (``K = (D+1)^2``):
  ``mean[0:3] | log_scale[3:6] | rot[6:10] (w,x,y,z) | raw_nu[10] |
  raw_opacity[11] | sh[12 + 3k + c]``.
* configs 1-2: means U[-1,1]^3; configs 3-5: 64 anisotropic Gaussian blobs
  of means (centres U[-1,1]^3, random rotation, sigma U[0.05,0.3]^3).
* log-scales N(-3, 0.5); quaternions z/|z| with z ~ N(0, I4).
* nu U[1.001, 8] (configs 1-2) or U[1.001, 16] (3-5), stored raw as the
  value whose image under nu = 1 + softplus(raw) is nu.
* |o| ~ U(0, 0.999); sign negative w.p. 0.2 (configs 1-2) or 0.3 (3-5);
  stored raw so that tanh(raw) = o.
* SH: DC spans the colour range ((rgb - 1/2) * 2 sqrt(pi), rgb U[0,1]^3);
  higher bands N(0, 0.1).
* Pinhole cameras, fov 60 deg horizontal, c = (W/2, H/2), z_near = 0.2,
  OpenCV axes (x right, y down, z forward), looking at the origin, world up
  +z.  Configs 1-3: one camera at 4 * normalize(0.3, -1, 0.45); config 4:
  8 cameras on a ring (4 cos t, 4 sin t, 0.5); config 5: 64 cameras on the
  upper hemisphere (Fibonacci lattice, radius 4).
* Targets U[0,1] per pixel and channel, seeded per view; background 0.

Nothing here evaluates the method (no projection, kernel, compositing,
gradient or sampler arithmetic).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

BASE_SEED = 20250313

CONFIG_NAMES = {
    1: "cfg1_tiny_1k_64x64",
    2: "cfg2_100k_sh3_256x256",
    3: "cfg3_500k_blobs_1297x840",
    4: "cfg4_2M_blobs_8views_980x545",
    5: "cfg5_3M_blobs_64views_1297x840_train",
}

# (n, sh_degree, width, height, n_views, layout, nu_hi, p_negative)
_CONFIGS = {
    1: (1_000, 0, 64, 64, 1, "uniform", 8.0, 0.2),
    2: (100_000, 3, 256, 256, 1, "uniform", 8.0, 0.2),
    3: (500_000, 3, 1297, 840, 1, "blobs", 16.0, 0.3),
    4: (2_000_000, 3, 980, 545, 8, "blobs", 16.0, 0.3),
    5: (3_000_000, 3, 1297, 840, 64, "blobs", 16.0, 0.3),
}


def sh_coeff_count(sh_degree: int) -> int:
    return (sh_degree + 1) ** 2


def param_plane_count(sh_degree: int) -> int:
    return 12 + 3 * sh_coeff_count(sh_degree)


@dataclass
class Camera:
    """Pinhole camera: p_cam = R @ x + t (world -> camera), OpenCV axes."""

    R: np.ndarray  # (3,3) float32, row-major
    t: np.ndarray  # (3,) float32
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    z_near: float = 0.2

    def center(self) -> np.ndarray:
        return -(self.R.astype(np.float64).T @ self.t.astype(np.float64))


@dataclass
class SGHMCParams:
    """Hyper-parameters of one sampler step (BASELINE configs 3 and 5)."""

    lr: float = 1e-3  # epsilon of Eq. 10 (mu step)
    friction: float = 0.1  # C
    noise: float = 1e-4  # eta: std of the pre-gate mu noise (R15)
    gate_k: float = 100.0
    gate_t: float = 0.005
    burn_in: bool = False
    g_adam: bool = True  # R17: "we employ the Adam gradient in SGHMC"
    lr_scale: float = 1e-3
    lr_rot: float = 1e-3
    lr_nu: float = 1e-3
    lr_opacity: float = 1e-3
    lr_sh: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-15
    grad_scale: float = 1.0
    step: int = 1
    seed: int = 1234
    eps_o: float = 0.0  # Eq. 8 opacity regularizer weight (0: the BASELINE L1 objective)
    eps_sigma: float = 0.0  # Eq. 8 sqrt-eigenvalue regularizer weight
    mu_mode: int = 0  # NEXT-3: 0 SGHMC, 1 SGLD (F disabled), 2 Adam on the means
    variant: int = 0  # parameter-set variant (oracle: opacity map of gate / regularizer)
    plane_begin: int = 0  # planes updated by one call (0, 0 = all; ZeRO-1 shards)
    plane_end: int = 0


@dataclass
class Scene:
    config: int
    params: np.ndarray  # (P, n) float32 SoA planes
    sh_degree: int
    cameras: List[Camera]
    bg: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))
    seed: int = 0
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.params.shape[1])

    @property
    def n_views(self) -> int:
        return len(self.cameras)

    # named plane views (no copies)
    @property
    def mean(self):
        return self.params[0:3]

    @property
    def log_scale(self):
        return self.params[3:6]

    @property
    def rot(self):
        return self.params[6:10]

    @property
    def raw_nu(self):
        return self.params[10:11]

    @property
    def raw_opacity(self):
        return self.params[11:12]

    @property
    def sh(self):
        return self.params[12:]


def look_at(pos, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
    """World->camera rotation/translation, OpenCV axes, looking at target."""
    pos = np.asarray(pos, np.float64)
    fwd = np.asarray(target, np.float64) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    t = -R @ pos
    return R, t


def _pinhole(pos, width, height, fov_deg=60.0, z_near=0.2) -> Camera:
    R, t = look_at(pos)
    f = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return Camera(R=R.astype(np.float32), t=t.astype(np.float32), fx=float(np.float32(f)),
                  fy=float(np.float32(f)), cx=width / 2.0, cy=height / 2.0,
                  width=int(width), height=int(height), z_near=z_near)


def make_cameras(layout: str, n_views: int, width: int, height: int) -> List[Camera]:
    if layout == "single":
        d = np.array([0.3, -1.0, 0.45])
        return [_pinhole(4.0 * d / np.linalg.norm(d), width, height)]
    if layout == "ring":
        cams = []
        for k in range(n_views):
            th = 2.0 * math.pi * k / n_views
            cams.append(_pinhole((4.0 * math.cos(th), 4.0 * math.sin(th), 0.5), width, height))
        return cams
    if layout == "hemisphere":
        cams = []
        for k in range(n_views):
            z = (k + 0.5) / n_views
            phi = k * 2.39996
            s = math.sqrt(max(0.0, 1.0 - z * z))
            cams.append(_pinhole((4.0 * s * math.cos(phi), 4.0 * s * math.sin(phi), 4.0 * z),
                                 width, height))
        return cams
    raise ValueError(layout)


def _random_rotations(rng, m):
    # Haar-random orthogonal matrices via QR of Gaussian matrices (blob
    # orientations of the input distribution; not the method's R(q)).
    a = rng.standard_normal((m, 3, 3))
    q, r = np.linalg.qr(a)
    d = np.sign(np.diagonal(r, axis1=1, axis2=2))
    d[d == 0] = 1.0
    q = q * d[:, None, :]
    det = np.linalg.det(q)
    q[:, :, 0] *= np.sign(det)[:, None]
    return q


def _raw_from_nu(nu):
    # inverse of nu = 1 + log1p(exp(raw)) on the generator side
    return np.log(np.expm1(nu - 1.0))


def make_params(rng, n: int, sh_degree: int, layout: str, nu_hi: float, p_negative: float,
                n_blobs: int = 64, extent: float = 1.0) -> np.ndarray:
    K = sh_coeff_count(sh_degree)
    P = param_plane_count(sh_degree)
    out = np.empty((P, n), np.float64)
    if layout == "uniform":
        out[0:3] = rng.uniform(-extent, extent, (3, n))
    elif layout == "blobs":
        centers = rng.uniform(-extent, extent, (n_blobs, 3))
        rots = _random_rotations(rng, n_blobs)
        sig = rng.uniform(0.05, 0.3, (n_blobs, 3))
        member = rng.integers(0, n_blobs, n)
        z = rng.standard_normal((n, 3)) * sig[member]
        mu = centers[member] + np.einsum("nij,nj->ni", rots[member], z)
        out[0:3] = mu.T
    else:
        raise ValueError(layout)
    out[3:6] = rng.normal(-3.0, 0.5, (3, n))
    q = rng.standard_normal((4, n))
    out[6:10] = q / np.linalg.norm(q, axis=0, keepdims=True)
    nu = rng.uniform(1.001, nu_hi, n)
    out[10] = _raw_from_nu(nu)
    mag = rng.uniform(0.0, 0.999, n)
    sign = np.where(rng.uniform(0.0, 1.0, n) < p_negative, -1.0, 1.0)
    out[11] = np.arctanh(sign * mag)
    rgb = rng.uniform(0.0, 1.0, (3, n))
    out[12:15] = (rgb - 0.5) * 2.0 * math.sqrt(math.pi)
    if K > 1:
        out[15:12 + 3 * K] = rng.normal(0.0, 0.1, (3 * (K - 1), n))
    return out.astype(np.float32)


def make_scene(config: int, n: Optional[int] = None, n_views: Optional[int] = None,
               width: Optional[int] = None, height: Optional[int] = None,
               seed: Optional[int] = None) -> Scene:
    """One of BASELINE.json's five configs (optionally shrunk for tests)."""
    n0, deg, w0, h0, v0, layout, nu_hi, pneg = _CONFIGS[config]
    n = n0 if n is None else int(n)
    w = w0 if width is None else int(width)
    h = h0 if height is None else int(height)
    v = v0 if n_views is None else int(n_views)
    s = BASE_SEED + config if seed is None else int(seed)
    rng = np.random.Generator(np.random.PCG64(s))
    params = make_params(rng, n, deg, layout, nu_hi, pneg)
    cam_layout = {1: "single", 2: "single", 3: "single", 4: "ring", 5: "hemisphere"}[config]
    if cam_layout == "single" and v > 1:
        cam_layout = "ring"
    cams = make_cameras(cam_layout, v, w, h)
    return Scene(config=config, params=params, sh_degree=deg, cameras=cams, seed=s,
                 name=CONFIG_NAMES[config])


def make_custom_scene(n: int, sh_degree: int, width: int, height: int, n_views: int = 1,
                      seed: int = 7, layout: str = "uniform", nu_hi: float = 8.0,
                      p_negative: float = 0.3, log_scale_mean: Optional[float] = None,
                      cam_layout: str = "single", extent: float = 1.0) -> Scene:
    rng = np.random.Generator(np.random.PCG64(seed))
    params = make_params(rng, n, sh_degree, layout, nu_hi, p_negative, extent=extent)
    if log_scale_mean is not None:
        params[3:6] += np.float32(log_scale_mean + 3.0)
    if cam_layout == "single" and n_views > 1:
        cam_layout = "ring"
    return Scene(config=0, params=params, sh_degree=sh_degree,
                 cameras=make_cameras(cam_layout, n_views, width, height), seed=seed,
                 name=f"custom_n{n}_d{sh_degree}_{width}x{height}_v{n_views}")


def make_stress_scene(n: int = 600, sh_degree: int = 1, width: int = 157, height: int = 119,
                      seed: int = 5, n_views: int = 1) -> Scene:
    """Edge-case components for the binning / inclusion parity cases: a mix of
    huge (log-scale U[-1.2, -0.4]), strongly elongated (one axis up to e^3.8
    ~ 45x the others), off-image (means outside the view frustum, so only a
    fat tail reaches the frame), near-plane (camera depth 0.25-0.8) and
    ordinary components, with nu from {1.001, U[1, 16], 200, 5000}, |o| in
    U(0.002, 0.999) (below the 1/255 visibility level and up to the alpha
    clamp) and 30 % negative.  Ragged frame (157 x 119: partial tiles).
    Inputs only; nothing of the method is evaluated here."""
    rng = np.random.Generator(np.random.PCG64(seed))
    params = make_params(rng, n, sh_degree, "uniform", 8.0, 0.3).astype(np.float64)
    cams = make_cameras("single" if n_views == 1 else "ring", n_views, width, height)
    cam = cams[0]
    R = cam.R.astype(np.float64)
    cpos = -(R.T @ cam.t.astype(np.float64))
    kind = rng.integers(0, 5, n)
    for i in range(n):
        k = kind[i]
        if k == 0:    # huge
            params[3:6, i] = rng.uniform(-1.2, -0.4, 3)
        elif k == 1:  # elongated: one long axis, two short
            ax = rng.integers(0, 3)
            ls = rng.uniform(-4.6, -3.8, 3)
            ls[ax] = rng.uniform(-1.4, -0.8)
            params[3:6, i] = ls
        elif k == 2:  # off-image: a point in camera space beyond the frame edges
            z = rng.uniform(2.5, 5.5)
            xs = rng.choice([-1.0, 1.0]) * rng.uniform(0.55, 0.95) * z * cam.width / (2 * cam.fx)
            ys = rng.uniform(-0.9, 0.9) * z * cam.height / (2 * cam.fy)
            if rng.uniform() < 0.5:
                xs, ys = rng.uniform(-0.9, 0.9) * z * cam.width / (2 * cam.fx), \
                    rng.choice([-1.0, 1.0]) * rng.uniform(0.55, 0.95) * z * cam.height / (2 * cam.fy)
            f = rng.uniform(1.1, 2.2)  # past the edge (some AABBs miss the frame)
            pc = np.array([xs * f, ys * f, z])
            params[0:3, i] = R.T @ pc + cpos
            params[3:6, i] = rng.uniform(-2.5, -1.2, 3)
        elif k == 3:  # near plane (a few behind it)
            pc = np.array([rng.uniform(-0.1, 0.1), rng.uniform(-0.08, 0.08), rng.uniform(0.15, 0.8)])
            params[0:3, i] = R.T @ pc + cpos
            params[3:6, i] = rng.uniform(-4.5, -3.0, 3)
        c = rng.integers(0, 4)
        nu = [1.001, rng.uniform(1.0, 16.0), 200.0, 5000.0][c]
        params[10, i] = _raw_from_nu(nu) if nu - 1.0 <= 30.0 else nu - 1.0
        mag = rng.uniform(0.002, 0.999)
        params[11, i] = np.arctanh(mag if rng.uniform() >= 0.3 else -mag)
    return Scene(config=0, params=params.astype(np.float32), sh_degree=sh_degree, cameras=cams,
                 seed=seed, name=f"stress_n{n}_d{sh_degree}_{width}x{height}")


def make_stop_rule_scene(bg=(0.0, 0.0, 0.0)) -> Scene:
    """Five co-located components on the optical axis of a 64 x 64 camera
    whose principal point is a pixel centre (h = 0 there, so alpha = o):
    opacities 0.98, 0.97, 0.9, -0.9, 0.5 front to back (depths 4.6 .. 5.0),
    each with one pure colour channel pattern so a composited component shows
    in the image.  Used for the R11 stop-rule pin."""
    from math import atanh
    n, deg = 5, 0
    P = param_plane_count(deg)
    params = np.zeros((P, n), np.float64)
    ops = [0.98, 0.97, 0.9, -0.9, 0.5]
    cols = [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0), (1.0, 1.0, 0.0), (1.0, 1.0, 1.0)]
    for i in range(n):
        params[0:3, i] = (0.0, 0.0, -0.4 + 0.1 * i)  # camera at z = -5: depth 4.6 + 0.1 i
        params[3:6, i] = -1.0
        params[6, i] = 1.0
        params[10, i] = _raw_from_nu(4.0)
        params[11, i] = atanh(ops[i])
        params[12:15, i] = (np.asarray(cols[i]) - 0.5) * 2.0 * math.sqrt(math.pi)
    cam = Camera(R=np.eye(3, dtype=np.float32), t=np.array([0.0, 0.0, 5.0], np.float32), fx=100.0,
                 fy=100.0, cx=32.5, cy=32.5, width=64, height=64)
    return Scene(config=0, params=params.astype(np.float32), sh_degree=deg, cameras=[cam],
                 bg=np.asarray(bg, np.float32), seed=0, name="stop_rule")


def make_targets(scene: Scene, views=None, seed_offset: int = 0) -> np.ndarray:
    """U[0,1] target images [len(views)][3][H][W] float32, seeded per view."""
    views = range(scene.n_views) if views is None else views
    views = list(views)
    cam = scene.cameras[0]
    out = np.empty((len(views), 3, cam.height, cam.width), np.float32)
    for i, v in enumerate(views):
        rng = np.random.Generator(np.random.PCG64(scene.seed * 1000 + 17 + v + seed_offset))
        out[i] = rng.random((3, cam.height, cam.width), dtype=np.float32)
    return out


def make_targets_u8(scene: Scene, views=None, seed_offset: int = 0) -> np.ndarray:
    """8-bit target images [len(views)][3][H][W] uint8 (uniform 0..255),
    seeded per view: the form of the paper's datasets (8-bit PNG/JPEG); the
    losses read them as u / 255 (sss.h SSS_BWD_TARGET_U8)."""
    views = range(scene.n_views) if views is None else views
    views = list(views)
    cam = scene.cameras[0]
    out = np.empty((len(views), 3, cam.height, cam.width), np.uint8)
    for i, v in enumerate(views):
        rng = np.random.Generator(np.random.PCG64(scene.seed * 1000 + 17 + v + seed_offset))
        out[i] = rng.integers(0, 256, (3, cam.height, cam.width), dtype=np.uint8)
    return out


def make_optimizer_state(scene: Scene, seed: int = 99, zero: bool = False):
    """(momentum r [3][n], adam m [P][n], adam v [P][n]) float32.

    Parity runs use a non-zero state so the friction term and the Adam
    moments are exercised; timing runs start from zeros.
    """
    P, n = scene.params.shape
    if zero:
        return (np.zeros((3, n), np.float32), np.zeros((P, n), np.float32),
                np.zeros((P, n), np.float32))
    rng = np.random.Generator(np.random.PCG64(seed))
    r = rng.normal(0.0, 1e-2, (3, n)).astype(np.float32)
    m = rng.normal(0.0, 1e-3, (P, n)).astype(np.float32)
    v = (rng.normal(0.0, 1e-3, (P, n)) ** 2).astype(np.float32)
    return r, m, v


def sghmc_params_for(scene: Scene, **kw) -> SGHMCParams:
    p = SGHMCParams(grad_scale=1.0 / max(1, scene.n_views))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


# ------------------------------------------------------------------ NEXT-4
# Torus scooping toy (Fig. 2): a torus with ambient
# lighting seen in frontal views; the targets are its silhouettes (constant
# colour on black).  Input generation only (ray marching of the implicit
# torus); the fit itself runs through the product's TrainStep.
TORUS_R, TORUS_r, TORUS_COLOR = 0.6, 0.25, (0.9, 0.8, 0.3)


def torus_cameras(n_views: int = 4, size: int = 64, dist: float = 3.0, tilt: float = 0.12) -> List[Camera]:
    """Frontal cameras on the torus axis (+z), slightly tilted around it."""
    cams = []
    for k in range(n_views):
        a = 2 * math.pi * k / max(1, n_views)
        pos = np.array([tilt * math.cos(a), tilt * math.sin(a), 1.0])
        pos = dist * pos / np.linalg.norm(pos)
        R, t = look_at(pos, up=(0.0, 1.0, 0.0))
        f = (size / 2.0) / math.tan(math.radians(60.0) / 2.0)
        cams.append(Camera(R=R.astype(np.float32), t=t.astype(np.float32), fx=float(np.float32(f)),
                           fy=float(np.float32(f)), cx=size / 2.0, cy=size / 2.0, width=size,
                           height=size, z_near=0.2))
    return cams


def torus_targets(cams: List[Camera], R: float = TORUS_R, r: float = TORUS_r,
                  color=TORUS_COLOR, samples: int = 512) -> np.ndarray:
    """Silhouette images [V][3][H][W] float32: a pixel (centre ray) is the
    torus colour iff its ray enters (sqrt(x^2 + y^2) - R)^2 + z^2 <= r^2."""
    out = []
    for cam in cams:
        H, W = cam.height, cam.width
        ys, xs = np.mgrid[0:H, 0:W]
        d_cam = np.stack([(xs + 0.5 - cam.cx) / cam.fx, (ys + 0.5 - cam.cy) / cam.fy, np.ones_like(xs, float)], -1)
        Rm = np.asarray(cam.R, np.float64).reshape(3, 3)
        t = np.asarray(cam.t, np.float64)
        o = -Rm.T @ t
        d = d_cam @ Rm  # world directions (R^T d_cam)
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        dist = np.linalg.norm(o)
        ts = np.linspace(dist - (R + r) * 1.5, dist + (R + r) * 1.5, samples)
        hit = np.zeros((H, W), bool)
        for tt in ts:
            p = o + tt * d
            q = (np.sqrt(p[..., 0] ** 2 + p[..., 1] ** 2) - R) ** 2 + p[..., 2] ** 2
            hit |= q <= r * r
        img = np.zeros((3, H, W), np.float32)
        for c in range(3):
            img[c][hit] = color[c]
        out.append(img)
    return np.stack(out)


def torus_init(n_pos: int, n_neg: int, seed: int, sh_degree: int = 0) -> np.ndarray:
    """Component planes initialised near the torus centre (Fig. 2: "We
    initialize the component means near the center"): means N(0, 0.05^2),
    flattened isotropic-in-plane scales, nu 3, colour 0.5, |o| 0.5 with the
    requested signs (negative ones slightly smaller)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = n_pos + n_neg
    P = param_plane_count(sh_degree)
    pl = np.zeros((P, n), np.float32)
    pl[0:3] = rng.normal(0.0, 0.05, (3, n))
    pl[3] = pl[4] = math.log(0.3)
    pl[5] = math.log(0.1)
    pl[3:6] += rng.normal(0.0, 0.05, (3, n))
    pl[6] = 1.0
    pl[10] = _raw_from_nu(np.full(n, 3.0))
    o = np.concatenate([np.full(n_pos, 0.5), np.full(n_neg, -0.4)])
    pl[11] = np.arctanh(o)
    pl[12:15] = 0.0  # colour 0.5 (SH DC 0)
    return pl
