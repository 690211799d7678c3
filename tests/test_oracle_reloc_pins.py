"""Pins of the oracle's component recycling (NEXT-2; PAPER.md:168-183 Eqs.
11-12, SM PAPER.md:1317-1460) against things other than itself:
SPEC.md worked examples and beta identities, quadrature of the composited
colour integral (the conservation law Eq. 11 the paper solves), the N = 1
no-op, and the mechanics of one pass (dead set, 5% cap, multinomial
frequencies against the |o| weights, group cap, copies and resets).
"""
import math

import numpy as np
import pytest
from scipy import integrate, special, stats

from helpers import planes_from, raw_o_for


def test_beta_identities(orc):
    """beta(1/2, 3/2) = pi/2, beta(1/2, 1/2) = pi; and scipy."""
    assert orc.beta(0.5, 1.5) == pytest.approx(math.pi / 2, rel=1e-14)
    assert orc.beta(0.5, 0.5) == pytest.approx(math.pi, rel=1e-14)
    for x, y in [(0.5, 2.5), (0.5, 17.0), (1.3, 4.2)]:
        assert orc.beta(x, y) == pytest.approx(special.beta(x, y), rel=1e-13)


def test_new_opacity_worked_examples(orc):
    """N = 1 -> o_old; N = 2, 0.75 -> 0.5; N = 2, -0.2 -> 1 - sqrt(1.2)."""
    assert orc.reloc_opacity(0.37, 1) == pytest.approx(0.37, rel=1e-15)
    assert orc.reloc_opacity(0.75, 2) == pytest.approx(0.5, rel=1e-15)
    assert orc.reloc_opacity(-0.2, 2) == pytest.approx(1 - math.sqrt(1.2), rel=1e-14)
    assert orc.reloc_opacity(-0.2, 2) == pytest.approx(-0.095445, abs=1e-6)
    for o in (0.3, -0.6):
        for N in (2, 5):
            on = orc.reloc_opacity(o, N)
            assert np.sign(on) == np.sign(o)  # PAPER.md:181 sign rule
            assert (1 - on) ** N == pytest.approx(1 - o, rel=1e-13)


@pytest.mark.parametrize("nu", [1.0, 5.0, 100.0])
@pytest.mark.parametrize("o", [0.9, -0.7, 0.3])
def test_K_is_the_integral_of_the_composited_profile(orc, nu, o):
    """K (Eq. 12) = int [1 - (1 - o_new (1+u^2)^{-(nu+3)/2})^N] du
    (the geometric sum of Eq. 7's N terms), by quadrature."""
    for N in (1, 2, 3, 5, 8):
        on = orc.reloc_opacity(o, N)
        f = lambda u: 1.0 - (1.0 - on * (1.0 + u * u) ** (-(nu + 3) / 2)) ** N  # noqa: E731
        val = 2 * integrate.quad(f, 0, np.inf, epsabs=1e-13, epsrel=1e-12, limit=400)[0]
        assert orc.reloc_K(N, on, nu) == pytest.approx(val, rel=1e-8), N


@pytest.mark.parametrize("nu", [1.0, 5.0, 100.0])
@pytest.mark.parametrize("o", [0.9, -0.7])
@pytest.mark.parametrize("N", [2, 3, 5])
def test_relocation_conserves_the_colour_integral(orc, nu, o, N):
    """Eq. 11: with Sigma_new = scale Sigma_old,
    int C_new = int C_old in 1D, C_old = o (1 + x^2/(nu S))^{-(nu+3)/2} and
    C_new = sum_i o_new T (1 - o_new T)^{i-1}, T the new profile."""
    S_old = 0.7
    scale = orc.reloc_scale(o, nu, nu, N)
    S_new = scale * S_old
    on = orc.reloc_opacity(o, N)
    c_old = lambda x: o * (1 + x * x / (nu * S_old)) ** (-(nu + 3) / 2)  # noqa: E731

    def c_new(x):
        T = (1 + x * x / (nu * S_new)) ** (-(nu + 3) / 2)
        return sum(on * T * (1 - on * T) ** (i - 1) for i in range(1, N + 1))

    kw = dict(epsabs=1e-13, epsrel=1e-11, limit=500)
    a = 2 * integrate.quad(c_old, 0, np.inf, **kw)[0]
    b = 2 * integrate.quad(c_new, 0, np.inf, **kw)[0]
    assert b == pytest.approx(a, rel=1e-7)


def test_single_member_group_is_a_no_op(orc):
    """N = 1 -> o_new = o_old, Sigma scale = 1 exactly."""
    for o, nu in [(0.4, 2.0), (-0.8, 7.5), (0.99, 1.0)]:
        assert orc.reloc_scale(o, nu, nu, 1) == pytest.approx(1.0, rel=1e-13)


def _scene(n_live, n_dead, seed=0, sh_degree=1, o_live=None):
    rng = np.random.default_rng(seed)
    comps = []
    for i in range(n_live):
        o = o_live[i] if o_live is not None else float(rng.uniform(0.05, 0.95) * rng.choice([-1, 1]))
        comps.append(dict(mu=tuple(rng.normal(size=3)), log_scale=tuple(rng.normal(-2, 0.3, 3)),
                          q=tuple(rng.normal(size=4)), nu=float(rng.uniform(1.5, 9)), o=o))
    for i in range(n_dead):
        comps.append(dict(mu=tuple(rng.normal(size=3)), log_scale=(-3.0, -3.0, -3.0),
                          o=float(rng.uniform(-0.004, 0.004))))
    perm = rng.permutation(len(comps))
    comps = [comps[i] for i in perm]
    pl = planes_from(comps, sh_degree)
    K = (sh_degree + 1) ** 2
    pl[15:12 + 3 * K] = rng.normal(0, 0.1, size=(3 * K - 3, pl.shape[1]))
    return pl


def _state(pl, seed=1):
    rng = np.random.default_rng(seed)
    P, n = pl.shape
    return rng.normal(size=(P, n)), rng.random((P, n)), rng.normal(size=(3, n))


def test_one_pass_mechanics(orc):
    pl = _scene(400, 60, seed=2)
    P, n = pl.shape
    m, v, r = _state(pl)
    out, m2, v2, r2, tgt, moved = orc.relocate(pl, 1, m, v, r, cap_frac=0.05, seed=7, step=3)
    o = np.tanh(pl[11])
    dead = np.flatnonzero(np.abs(o.astype(np.float32)) < np.float32(0.005))
    cap = int(0.05 * n)
    assert moved == min(len(dead), cap) == np.count_nonzero(tgt >= 0)
    sel = dead[:cap]
    assert set(np.flatnonzero(tgt >= 0)) == set(sel)  # the first dead in index order
    for d in np.flatnonzero(tgt >= 0):
        t = tgt[d]
        assert abs(o[t]) >= 0.005  # a live target
        np.testing.assert_array_equal(out[:, d], out[:, t])  # members copy the target
        assert np.all(m2[:, d] == 0) and np.all(v2[:, d] == 0) and np.all(r2[:, d] == 0)
        assert np.all(m2[:, t] == 0) and np.all(r2[:, t] == 0)
    # groups obey Eq. 12 and the sign rule
    for t in np.unique(tgt[tgt >= 0]):
        N = 1 + int(np.count_nonzero(tgt == t))
        on = orc.reloc_opacity(o[t], N)
        assert math.tanh(out[11, t]) == pytest.approx(on, rel=1e-12)
        assert np.sign(on) == np.sign(o[t])
        nu = orc.nu_of(pl[10, t])
        ls = 0.5 * math.log(orc.reloc_scale(o[t], nu, nu, N))
        np.testing.assert_allclose(out[3:6, t], pl[3:6, t] + ls, rtol=1e-13)
        for p in list(range(0, 3)) + list(range(6, P)):
            if p != 11:
                assert out[p, t] == pl[p, t]
    # untouched components keep their state
    touched = set(np.flatnonzero(tgt >= 0)) | set(tgt[tgt >= 0].tolist())
    keep = np.array([i for i in range(n) if i not in touched])
    np.testing.assert_array_equal(out[:, keep], pl[:, keep])
    np.testing.assert_array_equal(m2[:, keep], m[:, keep])
    # deterministic; another seed draws other targets
    out_b, *_, tgt_b, _ = orc.relocate(pl, 1, m, v, r, cap_frac=0.05, seed=7, step=3)
    np.testing.assert_array_equal(tgt_b, tgt)
    *_, tgt_c, _ = orc.relocate(pl, 1, m, v, r, cap_frac=0.05, seed=8, step=3)
    assert not np.array_equal(tgt_c, tgt)


def test_multinomial_draw_distribution(orc):
    """Draw counts vs |o| weights without group saturation: 4 live targets,
    40 dead per pass (n_max = 64 never binds), 200 passes; chi-square test
    of the 8000 draws against the weights."""
    w = [0.1, -0.2, 0.3, -0.4]
    counts = np.zeros(4)
    total = 0
    for step in range(200):
        pl = _scene(4, 40, seed=5, sh_degree=0, o_live=w)
        m, v, r = _state(pl)
        *_, tg, _ = orc.relocate(pl, 0, m, v, r, cap_frac=1.0, n_max=64, seed=3, step=step)
        lv = np.flatnonzero(np.abs(np.tanh(pl[11])) >= 0.005)
        for k, idx in enumerate(lv):
            counts[k] += np.count_nonzero(tg == idx)
        total += np.count_nonzero(tg >= 0)
    p = np.abs(np.tanh(pl[11, lv]))
    p = p / p.sum()
    assert total == 200 * 40
    chi2 = ((counts - total * p) ** 2 / (total * p)).sum()
    assert stats.chi2.sf(chi2, 3) > 1e-3, (counts, total * p)


def test_group_cap_and_single_live_target(orc):
    """All dead go to the only live component, at most n_max - 1 of them."""
    pl = _scene(1, 100, seed=4, sh_degree=0, o_live=[0.6])
    m, v, r = _state(pl)
    out, *_, tgt, moved = orc.relocate(pl, 0, m, v, r, cap_frac=1.0, n_max=8, seed=1, step=1)
    assert moved == 7
    t = int(np.flatnonzero(np.abs(np.tanh(pl[11])) >= 0.005)[0])
    assert set(tgt[tgt >= 0]) == {t}
    assert math.tanh(out[11, t]) == pytest.approx(orc.reloc_opacity(0.6, 8), rel=1e-12)


def test_nothing_to_do(orc):
    pl = _scene(50, 0, seed=6)
    m, v, r = _state(pl)
    out, m2, *_, tgt, moved = orc.relocate(pl, 1, m, v, r)
    assert moved == 0 and np.all(tgt == -1)
    np.testing.assert_array_equal(out, pl)
    np.testing.assert_array_equal(m2, m)
