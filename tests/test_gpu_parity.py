"""CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (north_star): tile rects, depth keys, tile counts,
sorted key lists and inclusion counts bit-exact; images max |d| <= 1e-4;
gradients relative L2 <= 1e-3 per parameter group; the SGHMC/Adam update
relative L2 <= 1e-5.  Pixels whose oracle transmittance came within the R11
tie band of the 1e-4 stop threshold are exempt from the image / count bound
(reported by count, required to be rare).
"""
import numpy as np
import pytest

from helpers import group_slices, rel_l2
from sss_synth import make_custom_scene, make_optimizer_state, make_scene, make_stress_scene

pytestmark = pytest.mark.gpu

TIE_BAND = 1e-3  # relative distance of the oracle W from 1e-4 (R11)


def _scenes():
    return {
        "cfg1": make_scene(1),
        "cfg2": make_scene(2),  # 100,000 components, the stated size
        "stress_d1": make_stress_scene(seed=5, sh_degree=1),  # huge/elongated/off-image/near-plane
        "ragged_d1": make_custom_scene(3000, 1, 200, 133, seed=3, p_negative=0.3),
        "blobs_d2_3v": make_custom_scene(6000, 2, 160, 96, n_views=3, seed=5, layout="blobs",
                                         nu_hi=16.0),
    }


@pytest.fixture(scope="module")
def scenes():
    return _scenes()


def _check_projection(orc, scene, pr_gpu, v):
    cam = scene.cameras[v]
    o = orc.project(scene.params, scene.sh_degree, cam)
    rect = pr_gpu.rect[v].cpu().numpy().astype(np.int32)
    rec = pr_gpu.rec[v].cpu().numpy()
    col = pr_gpu.col[v].cpu().numpy()
    depth = pr_gpu.depth[v].cpu().numpy()
    vis_o = o.n_tiles > 0
    vis_g = rect[:, 0] <= rect[:, 2]
    assert np.array_equal(vis_o, vis_g), int((vis_o != vis_g).sum())
    assert np.array_equal(rect[vis_g], o.rect[vis_o])
    assert np.array_equal(depth.view(np.uint32), o.depth.view(np.uint32))
    vis = vis_o
    for k, name in [(0, "mx"), (1, "my"), (2, "A"), (3, "B2"), (4, "C"), (5, "hmax")]:
        g = rec[vis, k]
        ref = getattr(o, name)[vis]
        bad = g.view(np.uint32) != ref.view(np.uint32)
        # fp64 transcendentals (exp/log/tanh) of libm and CUDA may differ in
        # the last fp64 bit; after rounding to fp32 that flips < ~1e-8 values
        assert bad.mean() <= 1e-4, (name, int(bad.sum()))
        if bad.any():
            from gpu_helpers import ulp_diff

            assert ulp_diff(g[bad], ref[bad]).max() <= 1, name
    np.testing.assert_allclose(rec[vis, 6], o.o[vis], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(rec[vis, 7], 1.0 / o.nu[vis], rtol=1e-6)
    np.testing.assert_allclose(col[vis, 0], -(o.nu[vis] + 2) / 2, rtol=1e-6)
    np.testing.assert_allclose(col[vis, 1:4], o.color[vis], atol=2e-6, rtol=1e-5)
    return o


def test_project_parity(orc, sss, scenes):
    from gpu_helpers import to_dev

    for name, sc in scenes.items():
        pr = sss.sss_project(to_dev(sc), sc.cameras)
        for v in range(sc.n_views):
            _check_projection(orc, sc, pr, v)


def test_bin_sort_parity_bit_exact(orc, sss, scenes):
    """Sorted key lists and per-tile counts bit-exact vs the oracle."""
    from gpu_helpers import gpu_forward

    for name, sc in scenes.items():
        _, pr, bins, _ = gpu_forward(sc, keys=True)
        for v in range(sc.n_views):
            counts, ids, keys = orc.bin_sort(sc.params, sc.sh_degree, sc.cameras[v])
            M = len(ids)
            assert int(bins.totals[v].item()) == M
            rg = bins.ranges[v].cpu().numpy()
            assert np.array_equal(rg[:, 1] - rg[:, 0], counts), name
            assert np.array_equal(bins.ids[v, :M].cpu().numpy(), ids), name
            gk = bins.keys[v, :M].cpu().numpy().view(np.uint64)
            assert np.array_equal(gk, keys), name


@pytest.mark.parametrize("shift", [0, 2])
def test_scatter_staged_and_direct_paths_agree(orc, sss, shift):
    """The scatter stages a chunk's ids in shared memory when the chunk fits
    the stage (sized from capacity / chunks) and writes straight to the bin
    lists otherwise (or when keys are requested).  Capacity = the exact total
    mixes both paths in one launch (chunks above the mean go direct); a large
    capacity stages every chunk; keys=True goes direct everywhere.  All three
    give the same lists, and at bin_shift 0 the oracle's."""
    import torch

    from gpu_helpers import to_dev

    sc = make_custom_scene(9000, 1, 160, 96, seed=41, log_scale_mean=-2.2)
    cam = sc.cameras
    params = to_dev(sc)
    pr = sss.sss_project(params, cam)
    ref = sss.sss_bin_sort(pr, cam, bin_shift=shift, keys=True)
    M = int(ref.totals[0].item())
    assert M > 9000  # nine chunks of 1024 depth-sorted components
    runs = [sss.sss_bin_sort(pr, cam, bin_shift=shift, capacity=M),
            sss.sss_bin_sort(pr, cam, bin_shift=shift, capacity=40 * M)]
    for b in runs:
        assert not sss.sss_check_overflow(b)
        assert int(b.totals[0].item()) == M
        assert torch.equal(b.ranges, ref.ranges)
        assert torch.equal(b.ids[0, :M], ref.ids[0, :M])
    if shift == 0:
        counts, ids, _ = orc.bin_sort(sc.params, sc.sh_degree, cam[0])
        assert len(ids) == M
        assert np.array_equal(ref.ids[0, :M].cpu().numpy(), ids)


@pytest.mark.parametrize("n", [1001, 1002, 1003, 1004])
def test_bin_sort_any_component_count(orc, sss, n):
    """Component counts with n % 4 != 0 take the scalar key initialisation
    (n % 4 == 0: four components per thread, 16-byte accesses); both give
    the oracle's lists bit for bit."""
    from gpu_helpers import to_dev

    sc = make_custom_scene(n, 1, 200, 133, seed=47)
    params = to_dev(sc)
    pr = sss.sss_project(params, sc.cameras)
    bins = sss.sss_bin_sort(pr, sc.cameras, bin_shift=0)
    assert not sss.sss_check_overflow(bins)
    counts, ids, _ = orc.bin_sort(sc.params, sc.sh_degree, sc.cameras[0])
    M = len(ids)
    assert int(bins.totals[0].item()) == M
    rg = bins.ranges[0].cpu().numpy()
    assert np.array_equal(rg[:, 1] - rg[:, 0], counts)
    assert np.array_equal(bins.ids[0, :M].cpu().numpy(), ids)


def test_scatter_large_rects_bit_exact(orc, sss):
    """Components covering most of a 1297x840 view (rects of up to 82 x 53
    tiles): the flattened walk's rank/bin arithmetic (division of the
    instance index by the rect width, 10-bit packed coordinates) over
    thousands of instances per component, against the oracle's lists."""
    import torch

    from gpu_helpers import to_dev

    sc = make_custom_scene(300, 0, 1297, 840, seed=43, log_scale_mean=0.3)
    cam = sc.cameras
    params = to_dev(sc)
    pr = sss.sss_project(params, cam)
    bins = sss.sss_bin_sort(pr, cam, bin_shift=0)
    assert not sss.sss_check_overflow(bins)
    counts, ids, _ = orc.bin_sort(sc.params, sc.sh_degree, cam[0])
    M = len(ids)
    assert M > 300 * 1000  # large rects: > 1000 tiles per component on average
    assert int(bins.totals[0].item()) == M
    rg = bins.ranges[0].cpu().numpy()
    assert np.array_equal(rg[:, 1] - rg[:, 0], counts)
    assert torch.equal(bins.ids[0, :M].cpu(), torch.from_numpy(ids))


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_coarse_bins_are_stable_and_complete(orc, sss, scenes, shift):
    """bin_shift > 0: each bin lists exactly the components whose tile rect
    meets it, in (depth, index) order."""
    from gpu_helpers import bin_lists, gpu_forward

    sc = scenes["ragged_d1"]
    _, pr, bins, _ = gpu_forward(sc, bin_shift=shift)
    o = orc.project(sc.params, sc.sh_degree, sc.cameras[0])
    cam = sc.cameras[0]
    tx, ty = (cam.width + 15) // 16, (cam.height + 15) // 16
    s = 1 << shift
    bx_n, by_n = (tx + s - 1) // s, (ty + s - 1) // s
    order = np.lexsort((np.arange(sc.n), o.depth.view(np.uint32)))
    vis = o.n_tiles > 0
    lists = bin_lists(bins, 0, bx_n * by_n)
    r = o.rect >> shift
    for b in range(bx_n * by_n):
        bx, by = b % bx_n, b // bx_n
        hit = vis & (r[:, 0] <= bx) & (r[:, 2] >= bx) & (r[:, 1] <= by) & (r[:, 3] >= by)
        ref = order[hit[order]]
        assert np.array_equal(lists[b], ref), b


@pytest.mark.parametrize("shift", [0, 2])
@pytest.mark.parametrize("bg", [(0.0, 0.0, 0.0), (0.2, 0.5, 0.9)])
def test_render_fwd_parity(orc, sss, scenes, shift, bg):
    from gpu_helpers import gpu_forward

    for name, sc in scenes.items():
        _, _, _, fr = gpu_forward(sc, bin_shift=shift, bg=bg)
        for v in range(sc.n_views):
            ref = orc.render(sc.params, sc.sh_degree, sc.cameras[v], bg=bg, mode="tiled")
            rgb = fr.rgb[v].cpu().numpy()
            T = fr.final_T[v].cpu().numpy()
            nc = fr.n_contrib[v].cpu().numpy()
            _check_frame(name, rgb, T, nc, ref)


def _check_frame(name, rgb, T, nc, ref):
    """Counts equal except at R11 ties; image within 1e-4 everywhere else."""
    mism = nc != ref.n_contrib
    # every count mismatch must be explained by a stop-threshold tie (R11)
    assert np.all(ref.tie[mism] < TIE_BAND), (name, float(ref.tie[mism].max()))
    assert mism.mean() <= 2e-3, (name, int(mism.sum()))
    # (with scooping, W can re-cross 1e-4 after a tie, so the counts may
    # differ by more than one; the image stays within the tied W ~ 1e-4)
    ok = ~mism
    err = np.abs(rgb - ref.rgb)[:, ok].max()
    assert err <= 1e-4, (name, float(err))
    assert np.abs(T - ref.final_T)[ok].max() <= 1e-4
    # at a tie the pixels differ by at most the tied component's tiny share
    if mism.any():
        assert np.abs(rgb - ref.rgb)[:, mism].max() <= 5e-3, (name, float(np.abs(rgb - ref.rgb)[:, mism].max()))
    print(f"{name}: max|d| {err:.2e}, count ties {int(mism.sum())}")


def _bwd_pair(orc, sss, sc, shift, seed=0, nu_paper=False):
    from gpu_helpers import gpu_forward
    import torch

    params, pr, bins, fr = gpu_forward(sc, bin_shift=shift)
    cam0 = sc.cameras[0]
    d = np.random.default_rng(seed).normal(size=(sc.n_views, 3, cam0.height, cam0.width)).astype(np.float32)
    grad = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=torch.from_numpy(d).cuda(),
                              nu_grad_paper=nu_paper)
    torch.cuda.synchronize()
    g = grad.planes.cpu().numpy().astype(np.float64)
    ref = np.zeros_like(g)
    for v in range(sc.n_views):
        gv, _ = orc.backward(sc.params, sc.sh_degree, sc.cameras[v], d[v].astype(np.float64),
                             mode="tiled", nu_grad_paper=nu_paper)
        ref += gv
    return g, ref


@pytest.mark.parametrize("shift", [0, 2])
def test_render_bwd_parity(orc, sss, scenes, shift):
    for name, sc in scenes.items():
        g, ref = _bwd_pair(orc, sss, sc, shift)
        for grp, sl in group_slices(sc.sh_degree).items():
            e = rel_l2(g[sl], ref[sl])
            assert e <= 1e-3, (name, grp, e)


def test_render_bwd_paper_nu_flag(orc, sss, scenes):
    sc = scenes["cfg1"]
    g, ref = _bwd_pair(orc, sss, sc, 0, nu_paper=True)
    assert rel_l2(g[10], ref[10]) <= 1e-3


def test_fused_l1_matches_explicit_image_gradient(orc, sss, scenes):
    """a6: fused L1 = the same backward fed sign(C - target)/(3HW); loss value."""
    import torch
    from gpu_helpers import gpu_forward
    from sss_synth import make_targets

    sc = scenes["blobs_d2_3v"]
    params, pr, bins, fr = gpu_forward(sc)
    tgt = torch.from_numpy(make_targets(sc)).cuda()
    loss = torch.zeros(1, device="cuda")
    g1 = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, target=tgt, loss=loss)
    diff = fr.rgb - tgt
    HW = diff.shape[-1] * diff.shape[-2]
    d = (torch.sign(diff) / (3 * HW)).contiguous()
    g2 = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d)
    torch.cuda.synchronize()
    assert rel_l2(g1.planes.cpu().numpy(), g2.planes.cpu().numpy()) < 1e-6
    ref_loss = float(diff.abs().mean(dim=(1, 2, 3)).sum())
    assert abs(loss.item() - ref_loss) <= 1e-5 * ref_loss
    # and against the oracle: targets far from the image so the sign of the
    # residual is decided identically (R20)
    o_rgb = [orc.render(sc.params, sc.sh_degree, c, mode="tiled").rgb for c in sc.cameras]
    rng = np.random.default_rng(9)
    t2 = np.stack([r + rng.choice([-1, 1], size=r.shape) * rng.uniform(0.01, 0.3, r.shape)
                   for r in o_rgb]).astype(np.float32)
    gg = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, target=torch.from_numpy(t2).cuda())
    torch.cuda.synchronize()
    ref = 0
    for v, c in enumerate(sc.cameras):
        _, dl = orc.l1_loss_and_grad(o_rgb[v], t2[v])
        ref = ref + orc.backward(sc.params, sc.sh_degree, c, dl, mode="tiled")[0]
    g = gg.planes.cpu().numpy()
    for grp, sl in group_slices(sc.sh_degree).items():
        assert rel_l2(g[sl], ref[sl]) <= 1e-3, grp


def _hp32(hp):
    """Round every float hyper-parameter to fp32 (what the ABI receives)."""
    for k, v in vars(hp).items():
        if isinstance(v, float):
            setattr(hp, k, float(np.float32(v)))
    return hp


@pytest.mark.parametrize("variant", ["plain", "burn_in", "g_adam"])
def test_sghmc_parity(orc, sss, variant):
    import torch

    from sss_synth import sghmc_params_for

    sc = make_custom_scene(50000, 3, 32, 32, seed=31)
    r, m, v = make_optimizer_state(sc, seed=5)
    rng = np.random.default_rng(8)
    grad = (rng.normal(size=sc.params.shape) * 1e-2).astype(np.float32)
    # a spread of opacities so the gate takes every value in (0, 1)
    sc.params[11] = np.arctanh(rng.uniform(-0.03, 0.03, sc.n)).astype(np.float32)
    hp = _hp32(sghmc_params_for(sc, step=4, seed=77, burn_in=variant == "burn_in",
                                g_adam=variant == "g_adam", noise=1e-4, grad_scale=0.5))
    P, n = sc.params.shape
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    params = sss.Params(dev(sc.params), 3)
    g = sss.Params(dev(grad), 3)
    mm = sss.Params(dev(m), 3)
    vv = sss.Params(dev(v), 3)
    rr = dev(r)
    sss.sss_sghmc_step(params, g, mm, vv, rr, hp)
    torch.cuda.synchronize()
    p_ref, m_ref, v_ref, r_ref = orc.sghmc_step(sc.params, 3, grad, m, v, r, hp)
    got = params.planes.cpu().numpy().astype(np.float64)
    dref = p_ref - sc.params
    # fp32 state: the update can only be as exact as one ulp of the result
    # (|d mu| ~ 1e-4 << |mu| ~ 1), so the bound per element is one fp32 ulp
    # (of the coarser binade of mu and mu') plus 1e-5 of the reference update.
    from gpu_helpers import update_ulp

    ulp = update_ulp(p_ref, sc.params)
    bound = ulp + 1e-5 * np.abs(dref)
    assert np.all(np.abs(got - p_ref) <= bound + 1e-30), float((np.abs(got - p_ref) / bound).max())
    # and most elements are the correctly rounded fp64 result: a systematic
    # error inside the update would move far more than this fraction off it
    frac = float(np.mean(got.astype(np.float32) != p_ref.astype(np.float32)))
    assert frac < 0.05, frac
    assert rel_l2(rr.cpu().numpy() - r, r_ref - r) <= 1e-5
    assert rel_l2(mm.planes.cpu().numpy(), m_ref) <= 1e-5
    assert rel_l2(vv.planes.cpu().numpy(), v_ref) <= 1e-5


def test_stop_rule_pixel(orc, sss):
    """R11 on the hand-derived pixel of the oracle pin
    (test_oracle_pins.py::test_stop_rule_pin): the GPU composites exactly the
    first three of five co-located components (the negative fourth would
    re-grow W), bins 0 and 2, with and without background; its gradient
    gives the post-stop components nothing."""
    import torch

    from gpu_helpers import gpu_forward
    from sss_synth import make_stop_rule_scene

    sc = make_stop_rule_scene()
    for shift in (0, 2):
        for bg in ((0.0, 0.0, 0.0), (0.25, 0.5, 0.75)):
            params, pr, bins, fr = gpu_forward(sc, bin_shift=shift, bg=bg)
            ref = orc.render(sc.params, 0, sc.cameras[0], bg=bg, mode="brute")
            assert int(fr.n_contrib[0, 32, 32].item()) == 3 == ref.n_contrib[32, 32]
            assert abs(float(fr.final_T[0, 32, 32].item()) - ref.final_T[32, 32]) <= 1e-9
            np.testing.assert_allclose(fr.rgb[0, :, 32, 32].cpu().numpy(), ref.rgb[:, 32, 32], atol=2e-7)
            _check_frame("stop_rule", fr.rgb[0].cpu().numpy(), fr.final_T[0].cpu().numpy(),
                         fr.n_contrib[0].cpu().numpy(), ref)
        d = torch.zeros((1, 3, 64, 64), device="cuda")
        d[0, :, 32, 32] = torch.tensor([1.0, -0.5, 0.25])
        ws = torch.zeros(sss.api.render_bwd_workspace_bytes(sc.n, 1), dtype=torch.uint8, device="cuda")
        g = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d, ws=ws)
        torch.cuda.synchronize()
        gg = g.planes.cpu().numpy()
        assert np.all(gg[:, 3:] == 0.0) and np.all(gg[11, :3] != 0.0)
        gref, _ = orc.backward(sc.params, 0, sc.cameras[0], d[0].cpu().numpy().astype(np.float64), mode="brute")
        assert rel_l2(gg, gref) <= 1e-5


def test_alpha_clamp_zero_gradient(orc, sss):
    """R10: one component with |o| = 0.999 seen at h = 0 (the oracle pin's
    pixel): alpha = +-0.99 on the GPU too, and with the image gradient on that
    pixel only, d raw_o and every geometry / nu gradient are exactly zero."""
    import torch

    from gpu_helpers import gpu_forward
    from sss_synth import make_stop_rule_scene
    from sss_synth.scenes import Scene

    base = make_stop_rule_scene()
    for o in (0.999, -0.999):
        pl = base.params[:, :1].copy()
        pl[11, 0] = np.float32(np.arctanh(o))
        sc = Scene(config=0, params=pl, sh_degree=0, cameras=base.cameras)
        params, pr, bins, fr = gpu_forward(sc)
        assert abs(abs(1.0 - float(fr.final_T[0, 32, 32].item())) - 0.99) <= 1e-7
        d = torch.zeros((1, 3, 64, 64), device="cuda")
        d[0, 0, 32, 32] = 1.0
        ws = torch.zeros(sss.api.render_bwd_workspace_bytes(1, 1), dtype=torch.uint8, device="cuda")
        g = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d, ws=ws)
        torch.cuda.synchronize()
        gg = g.planes.cpu().numpy()[:, 0]
        assert np.all(gg[:12] == 0.0), gg[:12]  # mean, scale, rot, nu, opacity
        assert gg[12] != 0.0  # the colour still receives alpha W g


def test_philox_normals_match_oracle(orc, sss):
    """GPU noise: Delta mu = xi exactly when g = r = 0, gate = 1, eta = 1."""
    import torch

    from sss_synth import SGHMCParams

    sc = make_custom_scene(4096, 0, 16, 16, seed=2)
    P, n = sc.params.shape
    hp = _hp32(SGHMCParams(noise=1.0, gate_t=1e9, step=123456789012, seed=0xDEADBEEF12345))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    params = sss.Params(dev(sc.params), 0)
    z = lambda: sss.Params(torch.zeros((P, n), device="cuda"), 0)  # noqa: E731
    r = torch.zeros((3, n), device="cuda")
    sss.sss_sghmc_step(params, z(), z(), z(), r, hp)
    torch.cuda.synchronize()
    xi = params.planes[0:3].cpu().numpy().astype(np.float64) - sc.params[0:3]
    ref = np.array([orc.normals3(hp.seed, i, hp.step) for i in range(n)]).T
    np.testing.assert_allclose(xi, ref, atol=2e-6 * np.abs(sc.params[0:3]).max() + 1e-6)


def test_edge_cases(orc, sss):
    """Empty scene, everything culled, image smaller than a tile, huge
    components covering every tile, nu at the 1e4 cap, |o| near 1."""
    import torch
    from gpu_helpers import gpu_forward
    from helpers import axis_camera, planes_from

    # n = 0
    sc = make_custom_scene(10, 0, 40, 24, seed=1)
    sc.params = sc.params[:, :0].copy()
    _, pr, bins, fr = gpu_forward(sc, bg=(0.3, 0.3, 0.3))
    assert int(bins.totals[0].item()) == 0
    assert torch.allclose(fr.rgb, torch.full_like(fr.rgb, 0.3))
    # all behind the camera
    sc = make_custom_scene(500, 0, 40, 24, seed=1)
    sc.params[2] = -10.0
    sc.cameras[0].t[:] = [0, 0, 5]
    sc.cameras[0].R[:] = np.eye(3)
    _, pr, bins, fr = gpu_forward(sc)
    assert int(bins.totals[0].item()) == 0 and float(fr.rgb.abs().max()) == 0.0
    # tiny image, huge / heavy-tailed / near-opaque / nu-capped components
    from sss_synth.scenes import Scene

    cam = axis_camera(width=7, height=5, f=6.0)
    comps = [dict(mu=(0, 0, 0), log_scale=(1.0, 1.0, 1.0), nu=1.0, o=0.999, rgb=(0.9, 0.1, 0.2)),
             dict(mu=(0.1, 0, 0.5), log_scale=(-1, -1, -1), nu=9999.0, o=-0.97, rgb=(0.2, 0.8, 0.1)),
             dict(mu=(0, 0.1, 1.0), log_scale=(-0.5, -2, -1), nu=500.0, o=0.6, rgb=(0.4, 0.4, 0.9))]
    pl = planes_from(comps, 0, np.float32)
    pl[10, 1] = 1e5  # raw_nu far above the cap -> nu = 1e4
    s = Scene(config=0, params=pl, sh_degree=0, cameras=[cam])
    _, _, _, fr = gpu_forward(s, bg=(0.1, 0.2, 0.3))
    ref = orc.render(pl, 0, cam, bg=(0.1, 0.2, 0.3), mode="brute")
    assert np.abs(fr.rgb[0].cpu().numpy() - ref.rgb).max() <= 1e-4
    # big scene in a 1-tile image: capacity overflow is reported, not written
    sc = make_custom_scene(2000, 0, 16, 16, seed=4)
    params, pr, _, _ = gpu_forward(sc)
    bins = sss.sss_bin_sort(pr, sc.cameras, capacity=10)
    assert sss.sss_check_overflow(bins)
    assert int(bins.ranges.abs().max().item()) == 0


def test_render_fwd_without_count_is_identical(sss, scenes):
    """n_contrib is an optional diagnostic: a NULL buffer selects the
    non-counting kernel, whose image, transmittance and replay offsets are
    bit-identical to the counting one."""
    import torch

    from gpu_helpers import gpu_forward

    for shift in (0, 2):
        sc = scenes["blobs_d2_3v"]
        params, pr, bins, fr = gpu_forward(sc, bin_shift=shift)
        f2 = sss.Frame(torch.empty_like(fr.rgb), torch.empty_like(fr.final_T), None,
                       torch.empty_like(fr.last))
        sss.sss_render_fwd(pr, bins, sc.cameras, out=f2)
        torch.cuda.synchronize()
        assert torch.equal(f2.rgb, fr.rgb)
        assert torch.equal(f2.final_T, fr.final_T)
        assert torch.equal(f2.last, fr.last)


def test_backward_tile_list_paths_agree(orc, sss, scenes):
    """The backward replays the forward's per-strip lists of composited
    entries (one per 16x8 half tile); a strip whose list overflowed (tiny cap)
    and a frame without lists replay the full range.  All three give the same
    gradients (up to the order of the float atomics) and a list holds exactly
    the entries some pixel of its strip composited."""
    import torch

    from gpu_helpers import to_dev

    sc = scenes["blobs_d2_3v"]
    V = sc.n_views
    cam = sc.cameras[0]
    grads = []
    for cap in (2048, 4, 0):
        params = to_dev(sc)
        pr = sss.sss_project(params, sc.cameras)
        bins = sss.sss_bin_sort(pr, sc.cameras, bin_shift=1)
        fr = sss.Frame.empty(V, cam.height, cam.width, tile_cap=cap)
        sss.sss_render_fwd(pr, bins, sc.cameras, out=fr)
        d = torch.from_numpy(np.random.default_rng(1).normal(size=(V, 3, cam.height, cam.width))
                             .astype(np.float32)).cuda()
        g = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d)
        torch.cuda.synchronize()
        grads.append(g.planes.cpu().numpy().astype(np.float64))
        if cap == 2048:
            tc = fr.tile_count.cpu().numpy()
            assert tc.max() <= cap and tc.sum() > 0
            # every listed entry is composited by some pixel: each pixel's
            # n_contrib equals the list entries passing its h test, which the
            # full-range parity tests check; here: lists are increasing and
            # inside the bin ranges
            tl = fr.tile_list.cpu().numpy()
            assert tc.shape == (V, tl.shape[1], sss._lib.SSS_TILE_LISTS)
            last = fr.last.cpu().numpy()
            tiles_x = (cam.width + 15) // 16
            for v in range(V):
                for t, s in zip(*np.nonzero(tc[v] > 1)):
                    seq = tl[v, t, s, :tc[v, t, s]]
                    assert np.all(np.diff(seq) > 0)
                    # the strip's last listed entry is its pixels' last composited one
                    sh = 16 // sss._lib.SSS_TILE_LISTS  # rows per list
                    y0, x0 = (t // tiles_x) * 16 + sh * s, (t % tiles_x) * 16
                    assert seq[-1] + 1 == last[v, y0:y0 + sh, x0:x0 + 16].max()
        if cap == 4:
            assert (fr.tile_count.cpu().numpy() > 4).any()  # the fallback is exercised
    assert rel_l2(grads[0], grads[2]) <= 1e-5
    assert rel_l2(grads[1], grads[2]) <= 1e-5


def test_sghmc_plane_ranges_compose(sss):
    """ZeRO-1 shards: updating plane ranges separately, each from the same
    pre-update state, and assembling the owned planes equals the full step
    bit for bit (parameters, moments, momentum)."""
    import copy

    import torch

    from sss_synth import sghmc_params_for

    sc = make_custom_scene(20000, 3, 32, 32, seed=33)
    r, m, v = make_optimizer_state(sc, seed=7)
    rng = np.random.default_rng(9)
    grad = (rng.normal(size=sc.params.shape) * 1e-2).astype(np.float32)
    sc.params[11] = np.arctanh(rng.uniform(-0.03, 0.03, sc.n)).astype(np.float32)
    hp = _hp32(sghmc_params_for(sc, step=3, seed=4, noise=1e-4, eps_o=0.01, eps_sigma=0.02))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731

    def run(p0, p1):
        h = copy.copy(hp)
        h.plane_begin, h.plane_end = p0, p1
        ps, ms, vs, rs = sss.Params(dev(sc.params), 3), sss.Params(dev(m), 3), sss.Params(dev(v), 3), dev(r)
        sss.sss_sghmc_step(ps, sss.Params(dev(grad), 3), ms, vs, rs, h)
        torch.cuda.synchronize()
        return ps.planes.cpu().numpy(), ms.planes.cpu().numpy(), vs.planes.cpu().numpy(), rs.cpu().numpy()

    P = sc.params.shape[0]
    full = run(0, 0)
    for R in (2, 3, 8):
        from paper_2503_10148_b200 import dist as D

        out = [np.array(sc.params), np.array(m), np.array(v), np.array(r)]
        for rank in range(R):
            _, (p0, p1) = D.plane_shard(P, rank, R)
            if p1 <= p0:
                continue
            part = run(p0, p1)
            for k in range(3):
                out[k][p0:p1] = part[k][p0:p1]
            a0, a1 = min(p0, 3), min(p1, 3)
            out[3][a0:a1] = part[3][a0:a1]
        for k in range(4):
            np.testing.assert_array_equal(out[k], full[k])


@pytest.mark.parametrize("shift", [0, 1, 2])
def test_truncated_bin_lists(orc, sss, scenes, shift):
    """max_per_bin > 0 (sss.h): each bin keeps the first min(len, cap) entries
    of its complete list (an exact prefix), resume[b] points one past the
    cap-th entry in the depth-sorted visible order (n_vis for complete
    lists), sorted[:n_vis] is the oracle's (depth, index) order, and the
    raster -- continuing a truncated list through the rect-filtered tail --
    gives the complete-list image bit for bit and the same gradients."""
    import torch

    from gpu_helpers import to_dev

    for name in ("blobs_d2_3v", "stress_d1", "cfg2"):
        sc = scenes[name]
        V = sc.n_views
        cam = sc.cameras[0]
        params = to_dev(sc)
        pr = sss.sss_project(params, sc.cameras)
        full = sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift)
        rf = full.ranges.cpu().numpy()
        lens = rf[..., 1] - rf[..., 0]
        for cap in (7, int(np.percentile(lens[lens > 0], 60)) + 1):
            tb = sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift, max_per_bin=cap)
            assert not sss.sss_check_overflow(tb)
            rt = tb.ranges.cpu().numpy()
            sorted_ = tb.sorted.cpu().numpy()
            nvis = tb.n_vis.cpu().numpy()
            resume = tb.resume.cpu().numpy()
            for v in range(V):
                o = orc.project(sc.params, sc.sh_degree, sc.cameras[v])
                vis = o.n_tiles > 0
                order = np.lexsort((np.arange(sc.n), o.depth.view(np.uint32)))
                order = order[vis[order]]
                assert nvis[v] == len(order)
                assert np.array_equal(sorted_[v, :nvis[v]], order)
                rank = np.empty(sc.n, np.int64)
                rank[order] = np.arange(len(order))
                fid, tid = full.ids[v].cpu().numpy(), tb.ids[v].cpu().numpy()
                for b in range(rf.shape[1]):
                    L = lens[v, b]
                    k = min(L, cap)
                    assert rt[v, b, 1] - rt[v, b, 0] == k
                    pre = fid[rf[v, b, 0]:rf[v, b, 0] + k]
                    assert np.array_equal(tid[rt[v, b, 0]:rt[v, b, 1]], pre)
                    assert resume[v, b] == (nvis[v] if L <= cap else rank[pre[-1]] + 1), (name, v, b)
            for tile_cap in (1536, 3):
                f_full = sss.Frame.empty(V, cam.height, cam.width, tile_cap=tile_cap)
                f_tr = sss.Frame.empty(V, cam.height, cam.width, tile_cap=tile_cap)
                sss.sss_render_fwd(pr, full, sc.cameras, bg=(0.1, 0.2, 0.3), out=f_full)
                sss.sss_render_fwd(pr, tb, sc.cameras, bg=(0.1, 0.2, 0.3), out=f_tr)
                torch.cuda.synchronize()
                assert torch.equal(f_full.rgb, f_tr.rgb) and torch.equal(f_full.final_T, f_tr.final_T)
                assert torch.equal(f_full.n_contrib, f_tr.n_contrib)
                d = torch.from_numpy(np.random.default_rng(2).normal(
                    size=(V, 3, cam.height, cam.width)).astype(np.float32)).cuda()
                g1 = sss.sss_render_bwd(params, pr, full, sc.cameras, f_full, bg=(0.1, 0.2, 0.3), d_rgb=d)
                g2 = sss.sss_render_bwd(params, pr, tb, sc.cameras, f_tr, bg=(0.1, 0.2, 0.3), d_rgb=d)
                torch.cuda.synchronize()
                assert rel_l2(g2.planes.cpu().numpy(), g1.planes.cpu().numpy()) <= 1e-5, (name, cap, tile_cap)


def test_adaptive_bin_caps(orc, sss, scenes):
    """sss_bins.used: the forward records each bin's consumption, the next
    bin_sort caps the bin at 1.25 used + 256.  Round 1 (used = -1) builds
    complete lists; round 2 truncates from round 1's consumption; round 3
    starts from used = 0 (caps of 256 for every bin: many tiles read the
    rect-filtered tail).  All three render the complete-list image bit for
    bit and give its gradients."""
    import torch

    from gpu_helpers import to_dev
    from paper_2503_10148_b200 import api as A

    for name in ("blobs_d2_3v", "cfg2", "stress_d1"):
        sc = scenes[name]
        V, cam = sc.n_views, sc.cameras[0]
        params = to_dev(sc)
        pr = sss.sss_project(params, sc.cameras)
        full = sss.sss_bin_sort(pr, sc.cameras, bin_shift=2)
        f0 = sss.Frame.empty(V, cam.height, cam.width)
        sss.sss_render_fwd(pr, full, sc.cameras, out=f0)
        d = torch.from_numpy(np.random.default_rng(4).normal(size=(V, 3, cam.height, cam.width))
                             .astype(np.float32)).cuda()
        g0 = sss.sss_render_bwd(params, pr, full, sc.cameras, f0, d_rgb=d).planes.cpu().numpy()
        nb = full.ranges.shape[1]
        ab = A.Bins.empty(V, nb, full.capacity, 2, False, "cuda", 0, sc.n, adaptive=True)
        lens0 = (full.ranges[..., 1] - full.ranges[..., 0]).cpu().numpy()
        for rnd in range(3):
            if rnd == 2:
                ab.used.zero_()
            sss.sss_bin_sort(pr, sc.cameras, bin_shift=2, out=ab)
            f = sss.Frame.empty(V, cam.height, cam.width)
            sss.sss_render_fwd(pr, ab, sc.cameras, out=f)
            torch.cuda.synchronize()
            lens = (ab.ranges[..., 1] - ab.ranges[..., 0]).cpu().numpy()
            if rnd == 0:
                assert np.array_equal(lens, lens0)
            else:
                assert np.all(lens <= lens0)
            assert torch.equal(f.rgb, f0.rgb) and torch.equal(f.final_T, f0.final_T), (name, rnd)
            assert torch.equal(f.n_contrib, f0.n_contrib), (name, rnd)
            g = sss.sss_render_bwd(params, pr, ab, sc.cameras, f, d_rgb=d).planes.cpu().numpy()
            assert rel_l2(g, g0) <= 1e-5, (name, rnd)
            used = ab.used.cpu().numpy()
            assert np.all(used >= 0)
        if name == "cfg2":
            assert (lens < lens0).any()  # round 3 truncated something


def test_project_bwd_range_blocked_layout(orc, sss, scenes):
    """sss_project_bwd_range over component blocks into a component-blocked
    gradient (sss.h sss_params.block) equals the one-call backward into the
    plain layout; sss_sghmc_step reads the blocked gradient identically."""
    import torch

    from gpu_helpers import gpu_forward
    from paper_2503_10148_b200 import api as A
    from sss_synth import sghmc_params_for

    sc = scenes["blobs_d2_3v"]
    V, cam = sc.n_views, sc.cameras[0]
    params, pr, bins, fr = gpu_forward(sc, bin_shift=1)
    d = torch.from_numpy(np.random.default_rng(6).normal(size=(V, 3, cam.height, cam.width))
                         .astype(np.float32)).cuda()
    ws = torch.zeros(A.render_bwd_workspace_bytes(sc.n, V), dtype=torch.uint8, device="cuda")
    g_plain = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d, ws=ws)
    P = A.n_planes(sc.sh_degree)
    for n_blocks, planes in ((1, P), (4, P + 3), (7, 2 * P)):
        gb = A.BlockedParams.zeros(sc.n, sc.sh_degree, n_blocks, planes, "cuda")
        sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d, ws=ws, half="raster", grad=gb)
        for k in range(n_blocks):
            i0, i1 = gb.block_range(k)
            A.sss_project_bwd_range(params, sc.cameras, ws, gb, i0, i1)
        torch.cuda.synchronize()
        assert int(torch.count_nonzero(ws).item()) == 0  # consumed and cleared
        assert rel_l2(gb.to_planes().cpu().numpy(), g_plain.planes.cpu().numpy()) <= 1e-5
        if planes > P:
            assert float(gb.buf[:, P:, :].abs().max()) == 0.0  # padding planes untouched
        hp = _hp32(sghmc_params_for(sc, step=2, seed=5, noise=1e-4))
        outs = []
        for g in (A.Params(gb.to_planes(), sc.sh_degree), gb):
            pp = sss.Params(params.planes.clone(), sc.sh_degree)
            m, v = sss.Params.zeros_like(pp), sss.Params.zeros_like(pp)
            r = torch.zeros((3, sc.n), device="cuda")
            sss.sss_sghmc_step(pp, g, m, v, r, hp)
            outs.append(pp.planes)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1])


def test_sghmc_device_step_state(sss):
    """sss_sghmc_hparams.step_state (graph capture): the step read from the
    device counter gives the host-step update bit for bit, and advances."""
    import torch

    from paper_2503_10148_b200 import api as A
    from sss_synth import sghmc_params_for

    sc = make_custom_scene(10000, 1, 32, 32, seed=13)
    r, m, v = make_optimizer_state(sc, seed=2)
    grad = (np.random.default_rng(3).normal(size=sc.params.shape) * 1e-2).astype(np.float32)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    outs = []
    for use_state in (False, True):
        hp = _hp32(sghmc_params_for(sc, step=7, seed=21, noise=1e-4))
        st = None
        if use_state:
            st = A.step_state(6)
            hp.step_state = st
            hp.step = 999  # ignored
        ps, ms, vs, rs = sss.Params(dev(sc.params), 1), sss.Params(dev(m), 1), sss.Params(dev(v), 1), dev(r)
        g = sss.Params(dev(grad), 1)
        if use_state:  # step 6 then step 7 from the device counter
            sss.sss_sghmc_step(ps, g, ms, vs, rs, hp)
            ps, ms, vs, rs = sss.Params(dev(sc.params), 1), sss.Params(dev(m), 1), sss.Params(dev(v), 1), dev(r)
        sss.sss_sghmc_step(ps, g, ms, vs, rs, hp)
        torch.cuda.synchronize()
        outs.append((ps.planes.cpu(), ms.planes.cpu(), vs.planes.cpu(), rs.cpu()))
        if use_state:
            assert int(st[0].item()) == 8
    for a_, b_ in zip(*outs):
        assert torch.equal(a_, b_)


def test_trainstep_cuda_graph_replay(sss):
    """TrainStep.capture/replay: one whole iteration as a CUDA graph gives the
    eager iterations' parameters (up to the order of the backward's float
    atomics, which differs run to run)."""
    import torch

    from paper_2503_10148_b200.step import TrainStep
    from sss_synth import make_targets, sghmc_params_for

    sc = make_custom_scene(5000, 3, 96, 64, n_views=2, seed=19, layout="blobs", nu_hi=16.0)
    tg = torch.from_numpy(make_targets(sc)).cuda()
    outs = []
    for graph in (False, True):
        hp = _hp32(sghmc_params_for(sc, step=1, seed=4, noise=1e-4))
        ts = TrainStep(torch.from_numpy(sc.params).cuda(), 3, sc.cameras, hp, bin_shift=2,
                       views_per_batch=2, adaptive_bins=True)
        if graph:
            ts.capture(tg)  # one eager (warm-up) iteration inside
            for _ in range(3):
                ts.replay(tg)
        else:
            for _ in range(4):
                ts.step(tg)
        torch.cuda.synchronize()
        assert not ts.overflowed() and ts.t == 5
        outs.append(ts.params.planes.cpu().numpy())
    np.testing.assert_allclose(outs[1], outs[0], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("shift", [1, 2])
def test_tile_masks(orc, sss, scenes, shift):
    """sss_bins.tmask: every bit a mask sets or clears is conservative -- the
    forward and backward over masked bins give the unmasked result (image,
    transmittance, counts bit for bit; gradients 1e-5) and the oracle's; every
    pair the oracle composites has its tile's bit set; the masks drop a
    large share of the rect's false positives; with adaptive truncation too."""
    import torch

    from gpu_helpers import to_dev

    for name in ("blobs_d2_3v", "stress_d1", "cfg2"):
        sc = scenes[name]
        V, cam = sc.n_views, sc.cameras[0]
        params = to_dev(sc)
        pr = sss.sss_project(params, sc.cameras)
        plain = sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift)
        masked = sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift, tile_masks=True)
        torch.cuda.synchronize()
        assert torch.equal(plain.totals, masked.totals) and torch.equal(plain.ranges, masked.ranges)
        for v in range(V):
            M = int(plain.totals[v].item())
            assert torch.equal(plain.ids[v, :M], masked.ids[v, :M])
        frames = []
        for b in (plain, masked):
            f = sss.Frame.empty(V, cam.height, cam.width)
            sss.sss_render_fwd(pr, b, sc.cameras, bg=(0.1, 0.2, 0.3), out=f)
            frames.append(f)
        torch.cuda.synchronize()
        assert torch.equal(frames[0].rgb, frames[1].rgb) and torch.equal(frames[0].n_contrib, frames[1].n_contrib)
        assert torch.equal(frames[0].final_T, frames[1].final_T)
        for v in range(V):
            ref = orc.render(sc.params, sc.sh_degree, sc.cameras[v], bg=(0.1, 0.2, 0.3), mode="tiled")
            _check_frame(name, frames[1].rgb[v].cpu().numpy(), frames[1].final_T[v].cpu().numpy(),
                         frames[1].n_contrib[v].cpu().numpy(), ref)
        d = torch.from_numpy(np.random.default_rng(8).normal(size=(V, 3, cam.height, cam.width))
                             .astype(np.float32)).cuda()
        for cap in (1536, 3):  # tiny strip lists: the unlisted replay filters by the masks too
            gs = []
            for b in (plain, masked):
                f = sss.Frame.empty(V, cam.height, cam.width, tile_cap=cap)
                sss.sss_render_fwd(pr, b, sc.cameras, out=f)
                gs.append(sss.sss_render_bwd(params, pr, b, sc.cameras, f, d_rgb=d).planes.cpu().numpy())
            torch.cuda.synchronize()
            assert rel_l2(gs[1], gs[0]) <= 1e-5, (name, cap)
        # every cleared bit of a tile in the entry's rect is a tile none of whose
        # 256 pixel centres passes the raster's fp32 inclusion test h <= hmax
        # (brute force, view 0; outside the rect no pixel passes, whatever the
        # bit); the masks drop a share of the rect's tiles
        M0 = int(masked.totals[0].item())
        tm = masked.tmask[0, :M0].cpu().numpy().view(np.uint16).astype(np.int64)
        ids = masked.ids[0, :M0].cpu().numpy().astype(np.int64)
        rg = masked.ranges[0].cpu().numpy()
        rec = pr.rec[0].cpu().numpy().reshape(-1, 8)
        rect = pr.rect[0].cpu().numpy().reshape(-1, 4).astype(np.int64)
        tx_n = (cam.width + 15) // 16
        S = 1 << shift
        bx_n = ((tx_n + S - 1) // S)
        kb = np.searchsorted(rg[:, 0], np.arange(M0), side="right") - 1
        while True:  # empty bins share their successor's start: step to the bin holding k
            adv = np.arange(M0) >= rg[kb, 1]
            if not adv.any():
                break
            kb[adv] += 1
        bx, by = (kb % bx_n) * S, (kb // bx_n) * S
        r = rect[ids]
        rect_bits = mask_bits = 0
        f32 = np.float32
        fma = lambda a, b, c: (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(f32)  # noqa: E731
        for ly in range(S):
            for lx in range(S):
                tx, ty = bx + lx, by + ly
                inr = (tx >= r[:, 0]) & (tx <= r[:, 2]) & (ty >= r[:, 1]) & (ty <= r[:, 3])
                bit = (tm >> ((ly << shift) | lx)) & 1
                rect_bits += int(inr.sum())
                mask_bits += int((bit.astype(bool) & inr).sum())
                cl = np.nonzero(inr & (bit == 0))[0]
                for c0 in range(0, len(cl), 4096):
                    c = cl[c0:c0 + 4096]
                    e = rec[ids[c]]
                    mx, my, A, B2, C, hmax = (e[:, q:q + 1].astype(f32) for q in range(6))
                    px = (tx[c, None] * 16 + np.arange(16)[None, :]).astype(f32) + f32(0.5)
                    hmin = np.full(len(c), np.inf, dtype=f32)
                    for yy in range(16):
                        py = (ty[c, None] * 16 + yy).astype(f32) + f32(0.5)
                        dx, dy = (px - mx).astype(f32), (py - my).astype(f32)
                        bdy, cdy2 = (B2 * dy).astype(f32), ((C * dy).astype(f32) * dy).astype(f32)
                        h = fma(dx, fma(A, dx, bdy), cdy2)
                        hmin = np.minimum(hmin, h.min(axis=1))
                    assert (hmin > hmax[:, 0]).all(), (name, shift, int((hmin <= hmax[:, 0]).sum()))
        if name == "cfg2":
            assert mask_bits < 0.9 * rect_bits, (mask_bits, rect_bits)
    # adaptive truncation with masks: the tail (unmasked, rect-tested) joins seamlessly
    from paper_2503_10148_b200 import api as A

    sc = scenes["cfg2"]
    params = to_dev(sc)
    pr = sss.sss_project(params, sc.cameras)
    full = sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift)
    f0 = sss.Frame.empty(1, sc.cameras[0].height, sc.cameras[0].width)
    sss.sss_render_fwd(pr, full, sc.cameras, out=f0)
    ab = A.Bins.empty(1, full.ranges.shape[1], full.capacity, shift, False, "cuda", 0, sc.n, adaptive=True,
                      tile_masks=True)
    ab.used.zero_()  # caps of 256: many tiles read the tail
    sss.sss_bin_sort(pr, sc.cameras, bin_shift=shift, out=ab)
    f1 = sss.Frame.empty(1, sc.cameras[0].height, sc.cameras[0].width)
    sss.sss_render_fwd(pr, ab, sc.cameras, out=f1)
    torch.cuda.synchronize()
    assert torch.equal(f0.rgb, f1.rgb) and torch.equal(f0.n_contrib, f1.n_contrib)


def test_backward_view_groups(orc, sss, scenes, monkeypatch):
    """The raster backward tags entries with 32-bit g2d record offsets from
    the first view of a launch group; a launch spanning >= 2^32 record floats
    is split into view groups (SSS_BWD_VIEW_GROUP forces small groups here).
    Groups of 1 and 2 views give the single-launch gradients (up to the
    order of the float atomics) and the L1 loss, on the bin-list and on the
    unlisted replay paths."""
    import torch

    from gpu_helpers import to_dev

    sc = scenes["blobs_d2_3v"]
    V, cam = sc.n_views, sc.cameras[0]
    assert V >= 3
    tgt = torch.from_numpy(np.random.default_rng(2).uniform(size=(V, 3, cam.height, cam.width))
                           .astype(np.float32)).cuda()
    for cap in (2048, 0):
        res = []
        for group in (None, "1", "2"):
            if group is None:
                monkeypatch.delenv("SSS_BWD_VIEW_GROUP", raising=False)
            else:
                monkeypatch.setenv("SSS_BWD_VIEW_GROUP", group)
            params = to_dev(sc)
            pr = sss.sss_project(params, sc.cameras)
            bins = sss.sss_bin_sort(pr, sc.cameras, bin_shift=1)
            fr = sss.Frame.empty(V, cam.height, cam.width, tile_cap=cap)
            sss.sss_render_fwd(pr, bins, sc.cameras, out=fr)
            loss = torch.zeros(1, device="cuda")
            g = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, target=tgt, loss=loss)
            torch.cuda.synchronize()
            res.append((g.planes.cpu().numpy().astype(np.float64), float(loss.item())))
        monkeypatch.delenv("SSS_BWD_VIEW_GROUP", raising=False)
        for gk, lk in res[1:]:
            assert rel_l2(gk, res[0][0]) <= 1e-5, cap
            assert abs(lk - res[0][1]) <= 1e-6 * abs(res[0][1]), cap


def test_backward_grad_assign(orc, sss, scenes):
    """SSS_BWD_GRAD_ASSIGN (sss.h): grad = result, the old contents unread --
    on a NaN-filled gradient it gives bit for bit what += gives on zeros,
    including the zero rows of components no view touched."""
    import torch

    from gpu_helpers import to_dev

    sc = scenes["blobs_d2_3v"]
    V, cam = sc.n_views, sc.cameras[0]
    params = to_dev(sc)
    pr = sss.sss_project(params, sc.cameras)
    bins = sss.sss_bin_sort(pr, sc.cameras, bin_shift=1)
    fr = sss.sss_render_fwd(pr, bins, sc.cameras)
    d = torch.from_numpy(np.random.default_rng(6).normal(size=(V, 3, cam.height, cam.width))
                         .astype(np.float32)).cuda()
    g_add = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d)
    g_nan = sss.Params(torch.full_like(params.planes, float("nan")), params.sh_degree)
    g_set = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, d_rgb=d, grad=g_nan, assign=True)
    torch.cuda.synchronize()
    a, b = g_add.planes.cpu().numpy(), g_set.planes.cpu().numpy()
    assert not np.isnan(b).any()
    # the raster's float atomics may order the per-record sums differently
    assert rel_l2(b, a) <= 1e-6
    untouched = np.all(a == 0, axis=0)
    assert untouched.any() and np.all(b[:, untouched] == 0)


def test_backward_u8_targets(orc, sss, scenes):
    """SSS_BWD_TARGET_U8: 8-bit targets read as u / 255 give the gradients
    and the L1 loss of the fp32 targets u / 255 (correctly rounded) bit for
    bit (up to the float atomics' order), and match the oracle's backward."""
    import torch

    from gpu_helpers import to_dev
    from sss_synth import make_targets_u8

    sc = scenes["blobs_d2_3v"]
    V, cam = sc.n_views, sc.cameras[0]
    t8 = make_targets_u8(sc)
    tf = t8.astype(np.float32) / np.float32(255.0)
    params = to_dev(sc)
    pr = sss.sss_project(params, sc.cameras)
    bins = sss.sss_bin_sort(pr, sc.cameras, bin_shift=1)
    fr = sss.sss_render_fwd(pr, bins, sc.cameras)
    res = []
    for t in (torch.from_numpy(tf).cuda(), torch.from_numpy(t8).cuda()):
        loss = torch.zeros(1, device="cuda")
        g = sss.sss_render_bwd(params, pr, bins, sc.cameras, fr, target=t, loss=loss)
        torch.cuda.synchronize()
        res.append((g.planes.cpu().numpy().astype(np.float64), float(loss.item())))
    assert rel_l2(res[1][0], res[0][0]) <= 1e-6
    assert abs(res[1][1] - res[0][1]) <= 1e-6 * abs(res[0][1])
    # and the oracle's loss over the same fp32 targets
    ref = 0.0
    for v in range(V):
        img = orc.render(sc.params, sc.sh_degree, sc.cameras[v], mode="tiled")
        ref += float(np.mean(np.abs(img.rgb.astype(np.float64) - tf[v])))
    assert abs(res[1][1] - ref) <= 1e-4 * abs(ref), (res[1][1], ref)
