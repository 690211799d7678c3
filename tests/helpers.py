"""Test helpers: hand-built components and cameras (no method arithmetic)."""
import math

import numpy as np

from sss_synth import Camera

# Real-SH degree-0 basis constant 1/(2 sqrt(pi)) (textbook value; the oracle's
# basis is pinned against scipy in test_oracle_pins.py::test_sh_matches_scipy).
Y00 = 0.5 / math.sqrt(math.pi)


def raw_nu_for(nu):
    if nu <= 1.0:
        return -50.0  # softplus(-50) ~ 2e-22: nu == 1 in fp64
    if nu - 1.0 > 30.0:
        return nu - 1.0  # softplus(x) = x there (R1)
    return math.log(math.expm1(nu - 1.0))


def raw_o_for(o):
    return math.atanh(o)


def planes_from(comps, sh_degree=0, dtype=np.float64):
    """comps: list of dicts(mu, log_scale, q, nu, o, rgb[, sh_rest]) -> [P][n]."""
    K = (sh_degree + 1) ** 2
    P = 12 + 3 * K
    out = np.zeros((P, len(comps)), np.float64)
    for i, c in enumerate(comps):
        out[0:3, i] = c["mu"]
        out[3:6, i] = c.get("log_scale", (0.0, 0.0, 0.0))
        out[6:10, i] = c.get("q", (1.0, 0.0, 0.0, 0.0))
        out[10, i] = raw_nu_for(c.get("nu", 3.0))
        out[11, i] = raw_o_for(c.get("o", 0.5))
        rgb = np.asarray(c.get("rgb", (0.5, 0.5, 0.5)), np.float64)
        out[12:15, i] = (rgb - 0.5) / Y00
        if K > 1 and "sh_rest" in c:
            out[15:12 + 3 * K, i] = c["sh_rest"]
    return out.astype(dtype)


def axis_camera(width=64, height=64, f=100.0, c=None, t=(0.0, 0.0, 5.0), z_near=0.2):
    cx, cy = (width / 2.0, height / 2.0) if c is None else c
    return Camera(R=np.eye(3, dtype=np.float32), t=np.asarray(t, np.float32), fx=f, fy=f,
                  cx=cx, cy=cy, width=width, height=height, z_near=z_near)


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def group_slices(sh_degree):
    K = (sh_degree + 1) ** 2
    return {"mean": slice(0, 3), "log_scale": slice(3, 6), "rot": slice(6, 10),
            "raw_nu": slice(10, 11), "raw_opacity": slice(11, 12), "sh": slice(12, 12 + 3 * K)}
