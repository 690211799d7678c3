"""NEXT-2 on the GPU (through the C ABI) vs the fp64 oracle: one component
recycling pass (Eqs. 11-12, 1317-1460, 1081).

Bit-exact: which components are relocated and onto which target (the dead
set, the multinomial draws and the groups are integer decisions taken on
identical integer weights).  Floating point: the relocated opacity and
log-scales within 1e-6 relative of the fp64 oracle (fp64 Eq. 12 on both
sides, rounded to fp32 once); copies and resets exact.
"""
import numpy as np
import pytest

from sss_synth import make_custom_scene, make_optimizer_state, make_scene

pytestmark = pytest.mark.gpu


def _with_dead(sc, frac, seed):
    rng = np.random.default_rng(seed)
    pl = sc.params.copy()
    n = pl.shape[1]
    dead = rng.random(n) < frac
    pl[11, dead] = np.arctanh(rng.uniform(-0.0045, 0.0045, dead.sum())).astype(np.float32)
    return pl


def _run(sss, pl, sh, m, v, r, **kw):
    import torch

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    params, mm, vv = sss.Params(dev(pl), sh), sss.Params(dev(m), sh), sss.Params(dev(v), sh)
    rr = dev(r)
    tgt = torch.empty(pl.shape[1], dtype=torch.int32, device="cuda")
    moved = sss.sss_relocate(params, mm, vv, rr, target_of=tgt, **kw)
    torch.cuda.synchronize()
    return (params.planes.cpu().numpy(), mm.planes.cpu().numpy(), vv.planes.cpu().numpy(),
            rr.cpu().numpy(), tgt.cpu().numpy(), int(moved.item()))


def _compare(orc, pl, sh, m, v, r, **kw):
    import paper_2503_10148_b200 as P

    got = _run(P, pl, sh, m, v, r, **kw)
    ref = orc.relocate(pl, sh, m, v, r, **kw)
    g_pl, g_m, g_v, g_r, g_t, g_n = got
    o_pl, o_m, o_v, o_r, o_t, o_n = ref
    assert g_n == o_n
    np.testing.assert_array_equal(g_t, o_t)
    changed = np.flatnonzero(np.any(o_pl != pl, axis=0) | (o_t >= 0))
    changed = np.union1d(changed, o_t[o_t >= 0])
    same = np.setdiff1d(np.arange(pl.shape[1]), changed)
    np.testing.assert_array_equal(g_pl[:, same], pl[:, same])
    np.testing.assert_array_equal(g_m[:, same], m[:, same].astype(np.float32))
    if len(changed):
        np.testing.assert_allclose(g_pl[:, changed], o_pl[:, changed], rtol=1e-6, atol=1e-6)
        assert np.all(g_m[:, changed] == 0) and np.all(g_v[:, changed] == 0)
        assert np.all(g_r[:, changed] == 0)
    return g_n


@pytest.mark.parametrize("sh", [0, 3])
def test_relocate_parity(orc, sss, sh):
    sc = make_custom_scene(30000, sh, 16, 16, seed=50 + sh)
    pl = _with_dead(sc, 0.08, seed=1)
    r, m, v = make_optimizer_state(sc, seed=2)
    moved = _compare(orc, pl, sh, m, v, r, threshold=0.005, cap_frac=0.05, n_max=32, seed=9, step=4)
    assert moved == int(0.05 * pl.shape[1])  # more dead than the cap


def test_relocate_fewer_dead_than_cap(orc, sss):
    sc = make_custom_scene(20000, 1, 16, 16, seed=61)
    pl = _with_dead(sc, 0.01, seed=3)
    r, m, v = make_optimizer_state(sc, seed=4)
    dead = int((np.abs(np.tanh(pl[11].astype(np.float64)).astype(np.float32)) < np.float32(0.005)).sum())
    assert _compare(orc, pl, 1, m, v, r, seed=5, step=1) == dead


def test_relocate_group_cap_single_target(orc, sss):
    sc = make_custom_scene(200, 0, 16, 16, seed=62)
    pl = sc.params.copy()
    pl[11, :] = np.float32(np.arctanh(0.001))
    pl[11, 57] = np.float32(np.arctanh(0.8))
    r, m, v = make_optimizer_state(sc, seed=5)
    assert _compare(orc, pl, 0, m, v, r, cap_frac=1.0, n_max=16, seed=2, step=7) == 15


def test_relocate_nothing_to_do(orc, sss):
    sc = make_custom_scene(5000, 0, 16, 16, seed=63)
    pl = sc.params.copy()
    pl[11] = np.where(np.abs(pl[11]) < 0.01, np.float32(0.5), pl[11])
    r, m, v = make_optimizer_state(sc, seed=6)
    assert _compare(orc, pl, 0, m, v, r) == 0


def test_relocate_config5_scale(orc, sss):
    """3M components (config 5), 2% dead: every decision bit-exact."""
    sc = make_scene(5)
    pl = _with_dead(sc, 0.02, seed=7)
    P, n = pl.shape
    m = np.zeros((P, n), np.float32)
    v = np.zeros((P, n), np.float32)
    r = np.zeros((3, n), np.float32)
    moved = _compare(orc, pl, 3, m, v, r, seed=13, step=100)
    assert moved > 0.015 * n


def test_relocate_arg_errors_and_all_dead(sss):
    import torch

    from paper_2503_10148_b200 import _lib as L

    n = 100
    planes = torch.zeros((15, n), device="cuda")
    p = sss.Params(planes, 0)
    m = sss.Params(torch.zeros((15, n), device="cuda"), 0)
    v = sss.Params(torch.zeros((15, n), device="cuda"), 0)
    r = torch.zeros((3, n), device="cuda")
    with pytest.raises(L.SSSError):
        sss.sss_relocate(p, m, v, r, n_max=1)
    moved = sss.sss_relocate(p, m, v, r)  # all dead, no live target: nothing moves
    assert int(moved.item()) == 0
