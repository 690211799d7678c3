"""Pins of the fp64 oracle against things other than itself (-m "not gpu").

Each test names the PAPER.md passage and the kind of pin (closed form,
special case, invariant, independent library, brute force, finite
differences, worked example).  See DESIGN.md §3 for the pin table.
"""
import math

import numpy as np
import pytest
from scipy import integrate, special
from scipy.spatial.transform import Rotation

from conftest import load_golden
from helpers import Y00, axis_camera, group_slices, planes_from, raw_o_for, rel_l2
from sss_synth import make_custom_scene, make_scene
from sss_synth.scenes import look_at, Camera


# ----------------------------------------------------------------- maps
def test_parameter_maps_worked_examples(orc):
    """SPEC.md:67-69 / PAPER.md:1077 (nu in [1, 10000]); tanh."""
    g = load_golden("spec_examples.json")
    for row in g["nu_of"]:
        assert orc.nu_of(row["raw"]) == pytest.approx(row["nu"], rel=1e-14)
    assert abs(orc.nu_of(-40.0) - 1.0) < 1e-12
    for x in (0.1, 0.7, 3.0, 19.0):
        assert orc.opacity_of(-x) == -orc.opacity_of(x)
        assert orc.opacity_of(x) == pytest.approx(math.tanh(x), rel=1e-15)
    assert orc.opacity_of(20.0) > 1 - 1e-15


def test_covariance_against_scipy_rotation(orc):
    """Sigma = R S S^T R^T: R from scipy's quaternion code,
    eigenvalues exp(2 s) (SPEC.md:81-83 worked examples)."""
    g = load_golden("spec_examples.json")
    for row in g["covariance_of"]:
        np.testing.assert_allclose(orc.cov3d(row["log_scale"], row["q"]), row["sigma"],
                                   atol=1e-14)
    rng = np.random.default_rng(3)
    for _ in range(50):
        s = rng.normal(-1.0, 0.7, 3)
        q = rng.normal(size=4) * rng.uniform(0.3, 3.0)  # un-normalised on purpose
        Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scalar-last
        ref = Rs @ np.diag(np.exp(2 * s)) @ Rs.T
        got = orc.cov3d(s, q)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(got)), np.sort(np.exp(2 * s)),
                                   rtol=1e-10)


# ----------------------------------------------------------- projection
def test_projection_worked_example(orc):
    """mu=0, W=I, t=(0,0,5), f=1, c=0, Sigma=I -> mean2d 0,
    cov2d 0.04 I, depth 5 (Eq. 4)."""
    cam = axis_camera(width=16, height=16, f=1.0, c=(0.0, 0.0))
    pl = planes_from([dict(mu=(0, 0, 0), log_scale=(0, 0, 0), o=0.9)])
    pr = orc.project(pl, 0, cam)
    np.testing.assert_allclose(pr.mean2d[0], [0.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(pr.cov2d[0], [0.04, 0.0, 0.04], rtol=1e-14, atol=1e-17)
    assert pr.depth[0] == np.float32(5.0)


def _pinhole_h(cam, x):
    """Independent route: homogeneous K [R|t] x, then dehomogenise."""
    K = np.array([[cam.fx, 0, cam.cx], [0, cam.fy, cam.cy], [0, 0, 1.0]], np.float64)
    Rt = np.hstack([np.asarray(cam.R, np.float64), np.asarray(cam.t, np.float64)[:, None]])
    xh = K @ Rt @ np.append(np.asarray(x, np.float64), 1.0)
    return xh[:2] / xh[2], xh[2]


def _ray_map(cam, x):
    uv, z = _pinhole_h(cam, x)
    return np.array([uv[0], uv[1], z])


def _fd_jacobian(f, x, h=1e-6):
    x = np.asarray(x, np.float64)
    f0 = f(x)
    J = np.zeros((len(f0), len(x)))
    for k in range(len(x)):
        e = np.zeros_like(x)
        e[k] = h
        J[:, k] = (f(x + e) - f(x - e)) / (2 * h)
    return J


def _cam_from(pos, w=64, h=64, f=60.0):
    R, t = look_at(pos)
    return Camera(R=R.astype(np.float32), t=t.astype(np.float32), fx=f, fy=f, cx=w / 2, cy=h / 2,
                  width=w, height=h)


def test_projection_matches_pinhole_and_fd_jacobian(orc):
    """mean2d = pinhole(mu) (homogeneous route) and Sigma2D = J_fd W Sigma W^T J_fd^T
    with J_fd the finite-difference Jacobian of the pinhole map (Eq. 4, EWA)."""
    rng = np.random.default_rng(11)
    cam = _cam_from((1.2, -3.5, 1.7))
    comps = []
    for _ in range(20):
        comps.append(dict(mu=rng.uniform(-0.5, 0.5, 3), log_scale=rng.normal(-1.5, 0.4, 3),
                          q=rng.normal(size=4), nu=rng.uniform(1, 10), o=0.7))
    pl = planes_from(comps)
    pr = orc.project(pl, 0, cam)
    R = np.asarray(cam.R, np.float64)
    for i, c in enumerate(comps):
        uv, z = _pinhole_h(cam, c["mu"])
        np.testing.assert_allclose(pr.mean2d[i], uv, rtol=1e-12, atol=1e-10)
        assert pr.p[i][2] == pytest.approx(z, rel=1e-14)
        q = np.asarray(c["q"], np.float64)
        Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
        Sig = Rs @ np.diag(np.exp(2 * np.asarray(c["log_scale"]))) @ Rs.T
        Jw = _fd_jacobian(lambda x: _pinhole_h(cam, x)[0], c["mu"])  # d(u,v)/dx = J W
        ref = Jw @ Sig @ Jw.T
        np.testing.assert_allclose(pr.cov2d[i], [ref[0, 0], ref[0, 1], ref[1, 1]], rtol=2e-7,
                                   atol=1e-9 * abs(ref).max())
        # conic is the inverse of Sigma2D
        Q = np.array([[pr.conic[i][0], pr.conic[i][1]], [pr.conic[i][1], pr.conic[i][2]]])
        S2 = np.array([[pr.cov2d[i][0], pr.cov2d[i][1]], [pr.cov2d[i][1], pr.cov2d[i][2]]])
        np.testing.assert_allclose(Q @ S2, np.eye(2), atol=1e-10)


@pytest.mark.parametrize("nu", [1.0, 2.5, 7.0, 50.0])
def test_2d_kernel_is_the_ray_marginal_of_the_3d_t(orc, nu):
    """PAPER.md:1172-1215 (marginalisation) + 1126-1167 (affine closure):
    under the EWA affine map x -> (u, v, z) the 3D t (Eq. 3) integrated along
    z equals sqrt(nu s) B(1/2, (nu+2)/2) * T2D(u), with s the Schur complement
    of the ray axis.  T2D is read from the oracle's rendered pixel values
    (single component, bg 0: C = c o T2D); the 3D side uses quadrature and a
    finite-difference Jacobian only."""
    cam = _cam_from((1.0, -3.6, 1.5))
    comp = dict(mu=(0.05, -0.1, 0.08), log_scale=(-1.2, -1.6, -1.0), q=(0.9, 0.2, -0.3, 0.1),
                nu=nu, o=0.5, rgb=(1.0, 1.0, 1.0))
    pl = planes_from([comp])
    fr = orc.render(pl, 0, cam, mode="brute")
    pr = orc.project(pl, 0, cam)
    c, o = pr.color[0][0], pr.o[0]
    q = np.asarray(comp["q"], np.float64)
    Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    Sig = Rs @ np.diag(np.exp(2 * np.asarray(comp["log_scale"]))) @ Rs.T
    J3 = _fd_jacobian(lambda x: _ray_map(cam, x), comp["mu"])
    Sr = J3 @ Sig @ J3.T
    m = _ray_map(cam, comp["mu"])
    Sinv = np.linalg.inv(Sr)
    s_schur = Sr[2, 2] - Sr[2, :2] @ np.linalg.solve(Sr[:2, :2], Sr[:2, 2])
    expect = math.sqrt(nu * s_schur) * special.beta(0.5, (nu + 2) / 2)
    ys, xs = np.nonzero((fr.n_contrib == 1) & (fr.rgb[0] > 0.03 * c * o))
    sel = np.random.default_rng(0).choice(len(ys), size=min(20, len(ys)), replace=False)
    ratios = []
    for k in sel:
        u = np.array([xs[k] + 0.5, ys[k] + 0.5])

        def t3(z):
            d = np.array([u[0], u[1], z]) - m
            return (1.0 + d @ Sinv @ d / nu) ** (-(nu + 3) / 2)  # Eq. 3

        zc = m[2] + Sr[2, :2] @ np.linalg.solve(Sr[:2, :2], u - m[:2])
        w = math.sqrt(s_schur)
        val = 0.0
        for a, b in [(-np.inf, zc - 50 * w), (zc - 50 * w, zc + 50 * w), (zc + 50 * w, np.inf)]:
            val += integrate.quad(t3, a, b, epsabs=0, epsrel=1e-12, limit=400)[0]
        T2 = fr.rgb[0][ys[k], xs[k]] / (c * o)
        ratios.append(val / T2)
    ratios = np.array(ratios)
    assert len(ratios) >= 10
    assert np.ptp(ratios) / ratios.mean() < 1e-6
    np.testing.assert_allclose(ratios, expect, rtol=1e-6)


def test_nu_limits(orc):
    """nu -> 1 Cauchy-type, nu -> inf Gaussian.  nu=1: T2D =
    (1+h)^-3/2, T3D = (1+h)^-2 exactly; nu -> inf: nu (ln T2D + h/2) ->
    h^2/4 - h with an O(h^3/nu) remainder (series of ln(1+x))."""
    g = load_golden("spec_examples.json")
    assert orc.t3d(g["density3d"][0]["h"], g["density3d"][0]["nu"]) == g["density3d"][0]["value"]
    assert orc.t2d(g["density2d"][0]["h"], g["density2d"][0]["nu"]) == g["density2d"][0]["value"]
    for h in np.linspace(0, 30, 31):
        assert orc.t2d(h, 1.0) == pytest.approx((1 + h) ** -1.5, rel=1e-14)
        assert orc.t3d(h, 1.0) == pytest.approx((1 + h) ** -2.0, rel=1e-14)
    for h in (0.5, 1.0, 4.0, 9.0, 25.0):
        errs = []
        for nu in (1e2, 1e3, 1e4):
            lhs = nu * (math.log(orc.t2d(h, nu)) + h / 2)
            err = abs(lhs - (h * h / 4 - h))
            assert err <= 1.1 * (h ** 3 / 6 + h * h / 2) / nu
            errs.append(err)
        assert errs[1] < errs[0] and errs[2] < errs[1]
    # Gaussian closeness at the paper's cap nu = 1e4 (rate-aware)
    for h in (1.0, 9.0):
        assert orc.t2d(h, 1e4) == pytest.approx(math.exp(-h / 2), rel=2 * h * h / 1e4)


def test_cutoff_is_the_alpha_1_over_255_level(orc):
    """R9: hmax = nu((255|o|)^(2/(nu+2)) - 1) is exactly where |o| T2D = 1/255
    (self-consistency of two different closed forms)."""
    rng = np.random.default_rng(5)
    comps = [dict(mu=(0, 0, 0), log_scale=(-1, -1, -1), nu=rng.uniform(1, 200),
                  o=rng.choice([-1, 1]) * rng.uniform(0.01, 0.99)) for _ in range(200)]
    pr = orc.project(planes_from(comps), 0, axis_camera())
    for i in range(len(comps)):
        if pr.cull[i] == 2:
            assert 255 * abs(pr.o[i]) <= 1
            continue
        val = abs(pr.o[i]) * orc.t2d(float(pr.hmax[i]), pr.nu[i])
        assert val == pytest.approx(1 / 255, rel=2e-6)  # hmax is stored as fp32


# ------------------------------------------------------------ compositing
def _golden_camera():
    return axis_camera(width=64, height=64, f=100.0, c=(32.0, 32.0), t=(0, 0, 5))


def test_single_component_analytic_pixels(orc):
    """Single positive and negative component: C(u) = c o T2D(h(u)) and
    W = 1 - o T2D with h from the hand-derived Sigma2D = diag(100, 25)
    (mu=0, S=diag(.5,.25,.5), f=100, z=5) -- Eq. 4 and Eq. 7."""
    cam = _golden_camera()
    for o in (0.6, -0.6):
        comp = dict(mu=(0, 0, 0), log_scale=(math.log(.5), math.log(.25), math.log(.5)),
                    nu=3.0, o=o, rgb=(0.8, 0.0, 0.0))
        fr = orc.render(planes_from([comp]), 0, cam, mode="brute")
        ys, xs = np.mgrid[0:64, 0:64]
        h = ((xs + 0.5 - 32) ** 2) / 100.0 + ((ys + 0.5 - 32) ** 2) / 25.0
        T = (1 + h / 3) ** -2.5
        hmax = 3 * (153 ** 0.4 - 1)
        inside = h <= hmax * (1 - 1e-9)
        outside = h > hmax * (1 + 1e-9)
        np.testing.assert_array_equal(fr.n_contrib[inside], 1)
        np.testing.assert_array_equal(fr.n_contrib[outside], 0)
        np.testing.assert_allclose(fr.rgb[0][inside], 0.8 * o * T[inside], rtol=1e-12)
        np.testing.assert_allclose(fr.final_T[inside], 1 - o * T[inside], rtol=1e-12)
        assert np.all(fr.rgb[:, outside] == 0) and np.all(fr.final_T[outside] == 1)
        assert np.all(fr.rgb[1:] == 0)
    # the printed golden row of SURVEY §8(c) for pixel (31.5, 31.5)
    fr = orc.render(planes_from([dict(mu=(0, 0, 0), nu=3.0, o=0.6, rgb=(0.8, 0, 0),
                                      log_scale=(math.log(.5), math.log(.25), math.log(.5)))]),
                    0, cam, mode="brute")
    assert fr.rgb[0][31, 31] == pytest.approx(0.47503623177, abs=1e-10)


def test_scooping_pair_and_telescoping(orc):
    """Fig. 2 scooping: a co-located negative component
    behind a positive one dims the pixel; with bg equal to every colour the
    pixel equals bg exactly for any signed opacities (telescoping of Eq. 7)."""
    cam = _golden_camera()
    B = dict(mu=(0, 0, -0.1), log_scale=(math.log(.5),) * 3, nu=2.0, o=0.9, rgb=(1, 1, 1))
    Cc = dict(mu=(0, 0, 0), log_scale=(math.log(.3),) * 3, nu=2.0, o=-0.5, rgb=(1, 1, 1))
    fr = orc.render(planes_from([B, Cc]), 0, cam, mode="brute")
    hB = 0.5 / (0.25 * (100 / 4.9) ** 2)
    hC = 0.5 / (0.09 * 400.0)
    aB = 0.9 * (1 + hB / 2) ** -2
    aC = -0.5 * (1 + hC / 2) ** -2
    assert fr.n_contrib[31, 31] == 2
    assert fr.rgb[0][31, 31] == pytest.approx(aB + aC * (1 - aB), rel=1e-12)
    assert fr.final_T[31, 31] == pytest.approx((1 - aB) * (1 - aC), rel=1e-12)
    assert fr.rgb[0][31, 31] < aB  # scooping dims the centre
    assert fr.rgb[0][31, 31] == pytest.approx(0.84425744608, abs=1e-10)
    fr1 = orc.render(planes_from([B, Cc]), 0, cam, bg=(1, 1, 1), mode="brute")
    assert fr1.rgb[0][31, 31] == pytest.approx(1.0, abs=1e-14)
    # telescoping on a random signed scene with early termination active
    sc = make_custom_scene(400, 0, 48, 40, seed=21, p_negative=0.35, log_scale_mean=-2.0)
    bg = np.array([0.3, 0.6, 0.9])
    pl = sc.params.astype(np.float64)
    pl[12:15] = ((bg - 0.5) / Y00)[:, None]
    fr = orc.render(pl, 0, sc.cameras[0], bg=bg, mode="tiled")
    assert fr.n_contrib.max() > 3
    np.testing.assert_allclose(fr.rgb, np.broadcast_to(bg[:, None, None], fr.rgb.shape), atol=1e-12)


def test_compositing_worked_examples(orc):
    """SPEC.md:211-213, 282-283 (Eq. 7 and its derivative) with T = 1 exactly
    (components on the optical axis, pixel centre at the projected mean)."""
    g = load_golden("spec_examples.json")
    cam = axis_camera(width=64, height=64, f=100.0, c=(32.5, 32.5))
    for row in g["composite_pixel"]:
        comps = [dict(mu=(0, 0, 0.1 * k), log_scale=(-1, -1, -1), nu=4.0, o=o, rgb=(c, c, c))
                 for k, (c, o) in enumerate(row["entries"])]
        fr = orc.render(planes_from(comps), 0, cam, mode="brute")
        assert fr.rgb[0][32, 32] == pytest.approx(row["rgb"], abs=1e-12)
        assert fr.final_T[32, 32] == pytest.approx(row["W"], abs=1e-12)
    # backward: dL/dc, dL/do for L = C_R at pixel (32, 32)
    for row in g["composite_backward"]:
        comps = [dict(mu=(0, 0, 0.1 * k), log_scale=(-1, -1, -1), nu=4.0, o=o, rgb=(c, c, c))
                 for k, (c, o) in enumerate(row["entries"])]
        d = np.zeros((3, 64, 64))
        d[0, 32, 32] = 1.0
        # pixel-local: restrict the image gradient to the centre pixel
        _, g2d = orc.backward(planes_from(comps), 0, cam, d, mode="brute", want_g2d=True)
        if "d_color" in row:
            assert g2d[0, 5] == pytest.approx(row["d_color"], abs=1e-12)
            assert g2d[0, 8] == pytest.approx(row["d_opacity"], abs=1e-12)
        else:
            assert g2d[0, 8] == pytest.approx(row["front_d_opacity"], abs=1e-12)


# ---------------------------------------------------------- tiling/binning
def _scenes_small():
    return [make_scene(1), make_custom_scene(1500, 1, 100, 72, seed=4, p_negative=0.3),
            make_custom_scene(800, 3, 64, 48, n_views=2, seed=8, layout="blobs")]


def test_tiled_equals_brute_force(orc):
    """Tile lists are an acceleration of Eq. 7, not a change of it (SPEC.md:232,
    659): bit-identical fp64 images, transmittance and counts.  The brute force
    tests every component not culled (including those whose tile AABB misses
    the frame) with the fp32 h <= hmax rule alone -- no tile rect -- so any
    pair a non-conservative rect dropped would show here.  The stress scenes
    carry huge, 45:1 elongated, off-image, near-plane, nu = 1 and nu = 5000
    components on a ragged 157 x 119 frame."""
    from sss_synth import make_stress_scene
    stress = [make_stress_scene(seed=s, sh_degree=s % 4) for s in (5, 6, 7)]
    for sc in stress:
        pr = orc.project(sc.params, sc.sh_degree, sc.cameras[0])
        assert np.sum(pr.cull == 4) > 10 and np.sum(pr.cull == 1) > 3  # AABB off-frame / behind
    for sc in _scenes_small() + stress:
        for cam in sc.cameras:
            a = orc.render(sc.params, sc.sh_degree, cam, bg=(0.1, 0.2, 0.3), mode="brute")
            b = orc.render(sc.params, sc.sh_degree, cam, bg=(0.1, 0.2, 0.3), mode="tiled")
            assert np.array_equal(a.rgb, b.rgb)
            assert np.array_equal(a.final_T, b.final_T)
            assert np.array_equal(a.n_contrib, b.n_contrib)
            assert a.n_contrib.max() > 0


@pytest.mark.slow
def test_tiled_equals_brute_force_config2_full(orc):
    """Config 2 at its stated size (100,000 components, 256 x 256, SH 3):
    rect-free brute force == tiled, bit for bit (~11 s on 8 cores)."""
    sc = make_scene(2)
    assert sc.n == 100_000
    a = orc.render(sc.params, 3, sc.cameras[0], mode="brute")
    b = orc.render(sc.params, 3, sc.cameras[0], mode="tiled")
    assert np.array_equal(a.rgb, b.rgb) and np.array_equal(a.n_contrib, b.n_contrib)
    assert np.array_equal(a.final_T, b.final_T)
    assert a.n_contrib.mean() > 50


def test_extreme_elongation_rect_stays_conservative(orc):
    """Axis ratios up to e^11 (elongated splats seen from the side): the +1 px
    AABB margin still covers every pixel the fp32 h test accepts."""
    from sss_synth import make_stress_scene
    sc = make_stress_scene(seed=3)
    for ratio_log in (5, 9, 11):
        p = sc.params.astype(np.float64)
        p[3:6] = -4.0
        p[3] = -4.0 + 0.5 * ratio_log
        p[4] = -4.0 - 0.5 * ratio_log
        p = p.astype(np.float32)
        a = orc.render(p, sc.sh_degree, sc.cameras[0], mode="brute")
        b = orc.render(p, sc.sh_degree, sc.cameras[0], mode="tiled")
        assert a.n_contrib.max() > 0
        assert np.array_equal(a.rgb, b.rgb) and np.array_equal(a.n_contrib, b.n_contrib)


def test_stop_rule_pin(orc):
    """R11 on a hand-derived pixel: five co-located
    components with alpha = o (h = 0 at the principal point, T = 1):
    0.98, 0.97, 0.9, -0.9, 0.5 front to back.  W = 1 -> 0.02 -> 6e-4 -> 6e-5:
    the third component drives W below 1e-4, IS composited, and the pixel
    stops; the negative fourth (which would re-grow W to 1.14e-4 > 1e-4 and
    let the fifth in) is ignored.  Stopping before the crossing component
    (n = 2, W = 6e-4) or not stopping (n = 5) both fail."""
    from sss_synth import make_stop_rule_scene
    sc = make_stop_rule_scene()
    cam = sc.cameras[0]
    o = np.tanh(sc.params[11].astype(np.float64))  # the fp32-stored opacities
    a1, a2, a3 = o[0], o[1], o[2]
    for bg in ((0.0, 0.0, 0.0), (0.25, 0.5, 0.75)):
        for mode in ("brute", "tiled"):
            fr = orc.render(sc.params, 0, cam, bg=bg, mode=mode)
            assert fr.n_contrib[32, 32] == 3
            W = (1 - a1) * (1 - a2) * (1 - a3)
            assert fr.final_T[32, 32] == pytest.approx(W, rel=1e-12)
            assert 5e-5 < W < 1e-4 < W * (1 - o[3])
            # colours (1,0,0), (0,1,0), (0,0,1): one channel per composited component
            col = np.clip(sc.params[12:15, :3].astype(np.float64) * Y00 + 0.5, 0, None)  # fp32-stored DC
            al = np.array([a1, a2 * (1 - a1), a3 * (1 - a1) * (1 - a2)])
            exp = col @ al + np.asarray(bg) * W
            assert np.allclose(col, np.eye(3), atol=1e-7)
            np.testing.assert_allclose(fr.rgb[:, 32, 32], exp, rtol=1e-12, atol=1e-15)
    # backward: the post-stop components get exactly zero gradient from this pixel
    d = np.zeros((3, 64, 64))
    d[:, 32, 32] = (1.0, -0.5, 0.25)
    _, g2d = orc.backward(sc.params, 0, cam, d, mode="brute", want_g2d=True)
    assert np.all(g2d[3:] == 0.0) and np.all(g2d[:3, 8] != 0.0)
    # closed-form dC/do of the third (last composited) component: dL/da3 * T,
    # T = 1: W3 sum_k g_k (c3_k - S3_k) with S3 = bg = 0
    W3 = (1 - a1) * (1 - a2)
    c3 = np.clip(sc.params[12:15, 2].astype(np.float64) * Y00 + 0.5, 0, None)
    assert g2d[2, 8] == pytest.approx(W3 * float(np.dot((1.0, -0.5, 0.25), c3)), rel=1e-12)


def test_alpha_clamp_pin(orc):
    """R10: alpha = clamp(o T, -0.99, 0.99) with zero gradient through an
    active clamp.  One component with o = 0.999 seen at h = 0: alpha = 0.99
    (not 0.999), W = 0.01, C = 0.99 c; with the image gradient on that pixel
    only, dL/do and every geometry / nu gradient are exactly 0 while dL/dc =
    alpha W_before g = 0.99 g.  With o = 0.98 (no clamp) dL/do = T c g."""
    from sss_synth import make_stop_rule_scene
    sc = make_stop_rule_scene()
    cam = sc.cameras[0]
    for o, clamped in ((0.999, True), (-0.999, True), (0.98, False)):
        p = sc.params[:, :1].astype(np.float64).copy()
        p[11, 0] = math.atanh(o)
        p[12:15, 0] = (np.array([0.8, 0.8, 0.8]) - 0.5) / Y00
        fr = orc.render(p, 0, cam, mode="brute")
        a = float(np.clip(np.tanh(p[11, 0]), -0.99, 0.99))
        assert fr.rgb[0, 32, 32] == pytest.approx(0.8 * a, rel=1e-12)
        assert fr.final_T[32, 32] == pytest.approx(1 - a, rel=1e-12)
        d = np.zeros((3, 64, 64))
        d[0, 32, 32] = 1.0
        _, g2d = orc.backward(p, 0, cam, d, mode="brute", want_g2d=True)
        assert g2d[0, 5] == pytest.approx(a, rel=1e-12)  # dL/dc_R = alpha W g
        if clamped:
            assert abs(a) == 0.99
            assert np.all(g2d[0, [0, 1, 2, 3, 4, 8, 9]] == 0.0)
        else:
            assert g2d[0, 8] == pytest.approx(0.8, rel=1e-6)  # T = 1 (h = 0), c = 0.8


def test_binning_is_the_sorted_rect_instances(orc):
    """Brute force over tiny inputs: the key list equals the lexicographic sort
    of (tile, depth bits, index) over every (visible component, tile in rect)."""
    for sc in _scenes_small():
        cam = sc.cameras[0]
        pr = orc.project(sc.params, sc.sh_degree, cam)
        counts, ids, keys = orc.bin_sort(sc.params, sc.sh_degree, cam)
        tw, th = orc.tiles_of(cam)
        vis = np.nonzero((pr.cull == 0) & (pr.n_tiles > 0))[0]
        inst = []
        for i in vis:
            x0, y0, x1, y1 = pr.rect[i]
            assert pr.n_tiles[i] == (x1 - x0 + 1) * (y1 - y0 + 1)
            for ty in range(y0, y1 + 1):
                for tx in range(x0, x1 + 1):
                    inst.append((ty * tw + tx, int(pr.depth[i].view(np.uint32)), int(i)))
        inst.sort()
        assert len(inst) == len(ids) == int(counts.sum())
        ref_keys = np.array([(t << 32) | d for t, d, _ in inst], np.uint64)
        assert np.array_equal(keys, ref_keys)
        assert np.array_equal(ids, np.array([i for _, _, i in inst], np.int32))
        assert np.array_equal(counts, np.bincount([t for t, _, _ in inst], minlength=tw * th))


def test_tile_rect_is_conservative(orc):
    """Every pixel whose exact (fp64) h is below hmax lies in a tile of the
    component's rect, so the tile gate never drops a pair the cutoff keeps."""
    sc = make_scene(1)
    cam = sc.cameras[0]
    pr = orc.project(sc.params, 0, cam)
    ys, xs = np.mgrid[0:cam.height, 0:cam.width]
    px, py = xs.ravel() + 0.5, ys.ravel() + 0.5
    tx, ty = xs.ravel() // 16, ys.ravel() // 16
    checked = 0
    for i in np.nonzero(pr.cull == 0)[0]:
        dx, dy = px - pr.mean2d[i, 0], py - pr.mean2d[i, 1]
        A, B, Cc = pr.conic[i]
        h = A * dx * dx + 2 * B * dx * dy + Cc * dy * dy
        inc = h <= pr.hmax[i] * (1 - 1e-6)
        x0, y0, x1, y1 = pr.rect[i]
        inrect = (tx >= x0) & (tx <= x1) & (ty >= y0) & (ty <= y1)
        assert not np.any(inc & ~inrect)
        checked += int(inc.sum())
    assert checked > 1000


# ---------------------------------------------------------------- backward
def _fd_scene(sh_degree, seed, n=6, w=24, h=20, o_range=(0.15, 0.85), ls_mean=-0.9):
    rng = np.random.default_rng(seed)
    comps = []
    K = (sh_degree + 1) ** 2
    for _ in range(n):
        comps.append(dict(mu=rng.uniform(-0.35, 0.35, 3), log_scale=rng.normal(ls_mean, 0.25, 3),
                          q=rng.normal(size=4) * rng.uniform(0.5, 2.0), nu=rng.uniform(1.2, 12),
                          o=rng.choice([-1, 1], p=[0.3, 0.7]) * rng.uniform(*o_range),
                          rgb=rng.uniform(0.25, 0.75, 3),
                          sh_rest=rng.normal(0, 0.05, 3 * (K - 1))))
    cam = _cam_from((0.8, -3.7, 1.1), w=w, h=h, f=18.0)
    return planes_from(comps, sh_degree), cam


@pytest.mark.parametrize("sh_degree,seed,o_range", [(0, 1, (0.15, 0.85)), (3, 2, (0.15, 0.85)),
                                                     (1, 3, (0.15, 0.85)), (2, 4, (0.15, 0.85)),
                                                     (0, 5, (0.993, 0.999)), (3, 6, (0.993, 0.999))])
def test_backward_matches_finite_differences(orc, sh_degree, seed, o_range):
    """SM backward with the full dT/dnu (R13): central
    differences of L = <d_rgb, C> in fp64 with frozen gating.
    The high-opacity cases (|o| up to 0.999) put pixels on the active
    +-0.99 alpha clamp (R10), whose zero gradient the differences confirm."""
    pl, cam = _fd_scene(sh_degree, seed, o_range=o_range, ls_mean=-0.9 if o_range[1] < 0.99 else 0.6)
    H, W = cam.height, cam.width
    d = np.random.default_rng(seed + 100).normal(size=(3, H, W))
    base = orc.render(pl, sh_degree, cam, mode="brute", record_lists=16)
    assert base.n_contrib.max() >= 2 and base.n_contrib.max() < 16
    lists = base.lists
    grad, _ = orc.backward(pl, sh_degree, cam, d, mode="frozen", lists_in=lists)
    grad_g, _ = orc.backward(pl, sh_degree, cam, d, mode="brute")
    np.testing.assert_allclose(grad, grad_g, rtol=0, atol=1e-13)

    def loss(p):
        fr = orc.render(p, sh_degree, cam, mode="frozen", lists_in=lists)
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
        assert np.linalg.norm(fd[sl]) > 0, name
        assert rel_l2(grad[sl], fd[sl]) < 1e-5, (name, rel_l2(grad[sl], fd[sl]))
    if o_range[1] > 0.99:  # the clamp is active somewhere in the frozen lists
        o = np.tanh(pl[11])
        clamped = 0
        for i in range(pl.shape[1]):
            if abs(o[i]) > 0.99:
                T = orc.render(pl[:, i:i + 1], sh_degree, cam, mode="brute")
                clamped += int(np.sum(np.abs(1 - T.final_T) >= 0.99 - 1e-12))
        assert clamped > 0


def test_printed_dT_dnu_fails_finite_differences(orc):
    """R13: the full dT/dnu matches finite differences; PAPER.md:1301-1314's
    printed form (log term dropped) does not, and flips sign in the tail."""
    for h, nu in [(0.5, 2.0), (3.0, 5.0), (10.0, 2.0), (1.0, 40.0)]:
        st = 1e-6 * nu
        fd = (orc.t2d(h, nu + st) - orc.t2d(h, nu - st)) / (2 * st)
        assert orc.dT_dnu(h, nu) == pytest.approx(fd, rel=1e-7)
        assert abs(orc.dT_dnu(h, nu, paper=True) - fd) > 0.1 * abs(fd)
        fdh = (orc.t2d(h + 1e-6, nu) - orc.t2d(h - 1e-6, nu)) / 2e-6
        assert orc.dT_dh(h, nu) == pytest.approx(fdh, rel=1e-7)
    assert orc.dT_dnu(0.0, 3.0) == 0.0
    assert orc.dT_dnu(10.0, 2.0) < 0 < orc.dT_dnu(10.0, 2.0, paper=True)
    g = load_golden("spec_examples.json")
    for row in g["dT2D_dh"]:
        assert orc.dT_dh(row["h"], row["nu"]) == row["value"]


def test_backward_is_linear_in_the_image_gradient(orc):
    """bwd(a g1 + g2) = a bwd(g1) + bwd(g2)."""
    sc = make_custom_scene(300, 2, 40, 32, seed=12)
    cam = sc.cameras[0]
    rng = np.random.default_rng(0)
    g1, g2 = rng.normal(size=(2, 3, 32, 40))
    a1, _ = orc.backward(sc.params, 2, cam, g1)
    a2, _ = orc.backward(sc.params, 2, cam, g2)
    a3, _ = orc.backward(sc.params, 2, cam, 2.5 * g1 + g2)
    np.testing.assert_allclose(a3, 2.5 * a1 + a2, atol=1e-12 * np.abs(a3).max())


def test_invisible_components_get_zero_gradient(orc):
    """Culled components (behind the camera, |o| <= 1/255) have exactly zero
    gradients (SURVEY §8(b) semantics)."""
    cam = _golden_camera()
    comps = [dict(mu=(0, 0, 0), log_scale=(-1, -1, -1), o=0.5),
             dict(mu=(0, 0, -6), log_scale=(-1, -1, -1), o=0.5),     # behind the camera
             dict(mu=(0, 0, 0.2), log_scale=(-1, -1, -1), o=0.003)]  # 255|o| < 1
    pl = planes_from(comps)
    pr = orc.project(pl, 0, cam)
    assert list(pr.cull) == [0, 1, 2]
    grad, _ = orc.backward(pl, 0, cam, np.ones((3, 64, 64)), mode="brute")
    assert np.abs(grad[:, 0]).sum() > 0
    assert np.all(grad[:, 1:] == 0)


# ---------------------------------------------------------------------- SH
def _real_sh_scipy(l, m, d):
    th = math.acos(max(-1.0, min(1.0, d[2])))
    ph = math.atan2(d[1], d[0])
    if m == 0:
        return special.sph_harm_y(l, 0, th, ph).real
    Y = special.sph_harm_y(l, abs(m), th, ph)
    return math.sqrt(2) * (Y.imag if m < 0 else Y.real)


def test_sh_matches_scipy(orc):
    """R7: the oracle's real SH basis (index l^2+l+m) equals sqrt(2) Im/Re of
    scipy's complex Y_l^|m| (Condon-Shortley phase included) -- the
    3DGS-lineage convention the paper builds on."""
    rng = np.random.default_rng(2)
    for _ in range(40):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        Y = orc.sh_basis(3, d)
        for l in range(4):
            for m in range(-l, l + 1):
                assert Y[l * l + l + m] == pytest.approx(_real_sh_scipy(l, m, d), abs=1e-13)


def test_sh_orthonormal(orc):
    """Orthonormality over the sphere (Gauss-Legendre x uniform azimuth)."""
    xg, wg = np.polynomial.legendre.leggauss(16)
    phis = np.linspace(0, 2 * np.pi, 32, endpoint=False)
    G = np.zeros((16, 16))
    for ct, w in zip(xg, wg):
        st = math.sqrt(1 - ct * ct)
        for ph in phis:
            Y = orc.sh_basis(3, [st * math.cos(ph), st * math.sin(ph), ct])
            G += w * (2 * np.pi / len(phis)) * np.outer(Y, Y)
    np.testing.assert_allclose(G, np.eye(16), atol=1e-12)


# ------------------------------------------------------------------- SGHMC
def _hp(**kw):
    """Literal Eq. 10 (g = dL/dmu) unless g_adam is passed: these pins check
    the equation's algebra; the Adam-direction default (R17) has its own pin."""
    from sss_synth import SGHMCParams

    p = SGHMCParams()
    p.g_adam = False
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def _state(n, sh_degree=0, o=0.5, log_scale=(-1, -1, -1), q=(1, 0, 0, 0)):
    pl = planes_from([dict(mu=(0.1, -0.2, 0.3), log_scale=log_scale, q=q, o=o)] * n, sh_degree)
    P = pl.shape[0]
    return pl, np.zeros((P, n)), np.zeros((P, n)), np.zeros((3, n))


def test_philox_known_answers(orc):
    g = load_golden("philox_kat.json")
    for row in g["vectors"]:
        out = orc.philox4x32_10([int(x, 16) for x in row["ctr"]], [int(x, 16) for x in row["key"]])
        assert [int(x) for x in out] == [int(x, 16) for x in row["out"]]


def test_normals_statistics(orc):
    z = np.array([orc.normals3(77, i, 3) for i in range(30000)]).ravel()
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.03
    from scipy import stats

    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_gate_values(orc):
    """Eq. 10 switch sigma(-k(|o| - t)) (R16),
    exposed through the friction-only update (g = 0, eta = 0)."""
    g = load_golden("spec_examples.json")
    for row in g["gate"]:
        o = row["abs_o"]
        pl, m, v, r = _state(2, o=0.3)
        pl[11, :] = [raw_o_for(o), raw_o_for(-o) if o > 0 else 0.0]
        r[:] = 1.0
        hp = _hp(noise=0.0, gate_k=row["k"], gate_t=row["t"])
        pl2, *_ = orc.sghmc_step(pl, 0, np.zeros_like(pl), m, v, r, hp)
        gate = (pl2[0] - pl[0]) / (hp.lr * (1 - hp.lr * hp.friction))
        np.testing.assert_allclose(gate, row["value"], rtol=1e-9)


def test_sghmc_degenerate_updates(orc):
    """SPEC.md:404-406 / PAPER.md:1504-1521: gate 0 & no noise -> mu - eps^2 g;
    g = 0, gate 1, no noise -> mu + eps (1 - eps C) r; r' = (1 - eps C) r - eps g."""
    rng = np.random.default_rng(1)
    pl, m, v, r = _state(50, o=0.99)
    g = rng.normal(size=pl.shape)
    r[:] = rng.normal(size=r.shape)
    hp = _hp(noise=0.0, grad_scale=0.5)
    pl2, m2, v2, r2 = orc.sghmc_step(pl, 0, g, m, v, r, hp)
    eps, Cf = hp.lr, hp.friction
    np.testing.assert_allclose(pl2[0:3], pl[0:3] - eps * eps * 0.5 * g[0:3], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(r2, (1 - eps * Cf) * r - eps * 0.5 * g[0:3], rtol=1e-12)
    pl, m, v, r = _state(50, o=0.3)
    r[:] = rng.normal(size=r.shape)
    hp = _hp(noise=0.0, gate_t=1e9)  # gate == 1
    pl2, *_ = orc.sghmc_step(pl, 0, np.zeros_like(pl), m, v, r, hp)
    np.testing.assert_allclose(pl2[0:3], pl[0:3] + eps * (1 - eps * Cf) * r, rtol=1e-12)
    # burn-in drops F
    hp = _hp(noise=0.0, gate_t=1e9, burn_in=True)
    pl3, *_ = orc.sghmc_step(pl, 0, np.zeros_like(pl), m, v, r, hp)
    np.testing.assert_array_equal(pl3[0:3], pl[0:3])


def test_sghmc_adam_direction_closed_form(orc):
    """R17 ("we employ the Adam gradient in SGHMC"): g in Eq. 10
    is Adam's direction m^/(sqrt(v^) + eps); on the first step from zero
    moments that is g/|g| (up to eps) = sign(g), so with gate 0 and no noise
    mu' = mu - eps^2 sign(g) and r' = (1 - eps C) r - eps sign(g)."""
    rng = np.random.default_rng(7)
    pl, m, v, r = _state(60, o=0.99)
    g = rng.normal(size=pl.shape)
    r[:] = rng.normal(size=r.shape)
    hp = _hp(noise=0.0, g_adam=True, grad_scale=0.5)
    pl2, m2, v2, r2 = orc.sghmc_step(pl, 0, g, m, v, r, hp)
    eps, Cf = hp.lr, hp.friction
    np.testing.assert_allclose(pl2[0:3], pl[0:3] - eps * eps * np.sign(g[0:3]), rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(r2, (1 - eps * Cf) * r - eps * np.sign(g[0:3]), rtol=1e-9)
    np.testing.assert_allclose(m2[0:3], 0.1 * 0.5 * g[0:3], rtol=1e-12)  # the mean moments move
    from sss_synth import SGHMCParams
    assert SGHMCParams().g_adam  # the default reading (R17)


def test_adam_closed_forms(orc):
    """Adam on all non-mu groups: zero gradient leaves the
    parameter unchanged; the first step with zero moments is lr * g/(|g|+eps)."""
    rng = np.random.default_rng(4)
    pl, m, v, r = _state(40, sh_degree=1)
    pl2, m2, v2, _ = orc.sghmc_step(pl, 1, np.zeros_like(pl), m, v, r, _hp(noise=0.0))
    np.testing.assert_array_equal(pl2[3:], pl[3:])
    g = rng.normal(size=pl.shape)
    hp = _hp(noise=0.0, lr_scale=2e-3, lr_rot=3e-3, lr_nu=4e-3, lr_opacity=5e-3, lr_sh=6e-3)
    pl2, m2, v2, _ = orc.sghmc_step(pl, 1, g, m, v, r, hp)
    lrs = np.array([2e-3] * 3 + [3e-3] * 4 + [4e-3, 5e-3] + [6e-3] * 12)
    np.testing.assert_allclose(pl2[3:], pl[3:] - lrs[:, None] * np.sign(g[3:]), rtol=1e-9)
    np.testing.assert_allclose(m2[3:], 0.1 * g[3:], rtol=1e-12)
    assert np.all(m2[0:3] == 0)  # mean moments untouched unless g_adam


def test_burn_in_noise_covariance(orc):
    """PAPER.md:163 / 1523: during burn-in N is multiplied by Sigma (R18), so
    the mu-noise covariance is eta^2 Sigma^2 (Sigma from scipy's rotation)."""
    n = 20000
    s = np.array([-0.2, -0.9, -0.5])
    q = np.array([0.8, 0.3, -0.4, 0.2])
    pl, m, v, r = _state(n, o=0.3, log_scale=s, q=q)
    hp = _hp(noise=1.0, gate_t=1e9, burn_in=True)
    pl2, *_ = orc.sghmc_step(pl, 0, np.zeros_like(pl), m, v, r, hp)
    X = (pl2[0:3] - pl[0:3]).T
    Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    Sig = Rs @ np.diag(np.exp(2 * s)) @ Rs.T
    emp = X.T @ X / n
    assert np.linalg.norm(emp - Sig @ Sig) / np.linalg.norm(Sig @ Sig) < 0.05
    hp = _hp(noise=1e-2, gate_t=1e9)
    pl2, _, _, r2 = orc.sghmc_step(pl, 0, np.zeros_like(pl), m, v, r, hp)
    X = (pl2[0:3] - pl[0:3]).T
    np.testing.assert_allclose(X.T @ X / n, 1e-4 * np.eye(3), atol=4e-6)
    np.testing.assert_allclose(r2.std(axis=1), 1e-2 / hp.lr, rtol=0.03)
