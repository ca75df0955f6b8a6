"""Statistical pins of the seeded input generators (SURVEY 8(c) "generator").
CPU tests use synth.gen (numpy Ogata); tests marked gpu use libmdhp_synth.so."""
import numpy as np
import pytest
from scipy import stats

from synth import gen


def rescaled_gaps(t, m, theta, alpha, beta, i):
    """Time-rescaling theorem: for dim i, Lambda_i(t_k) - Lambda_i(t_{k-1}) ~ iid Exp(1), with
    Lambda_i(t) = theta_i t + sum_j sum_{s in j, s < t} (alpha_ij/beta_ij)(1 - e^{-beta_ij (t - s)})."""
    ti = t[m == i]
    lam = theta[i] * ti
    for j in range(len(theta)):
        sj = t[m == j]
        d = ti[:, None] - sj[None, :]
        lam = lam + (alpha[i, j] / beta[i, j] * np.where(d > 0, 1 - np.exp(-beta[i, j] * np.maximum(d, 0)), 0)).sum(1)
    return np.diff(np.concatenate([[0.0], lam]))


def test_poisson_counts():
    """alpha = 0, theta = 3, T = 100: counts over 50 seeds within 4 sigma of Poisson(300)."""
    th, al, be = np.array([3.0]), np.zeros((1, 1)), np.ones((1, 1))
    counts = [len(gen.ogata_window(th, al, be, 100.0, gen.rng_for(1, s))[0]) for s in range(50)]
    assert all(abs(c - 300) <= 4 * np.sqrt(300) for c in counts)
    assert abs(np.mean(counts) - 300) <= 4 * np.sqrt(300 / 50)


def test_zero_intensity_empty():
    t, m = gen.ogata_window(np.zeros(2), np.zeros((2, 2)), np.ones((2, 2)), 10.0, gen.rng_for(2, 0))
    assert len(t) == 0


def test_stationary_rate_symmetric():
    """D = 2, theta = 0.2, alpha = 0.6, beta = 1.5: branching ratio rho = D alpha/beta = 0.8, so the
    stationary rate per dim is theta/(1 - rho) = 1.0; long window, within 15%."""
    D = 2
    th = np.full(D, 0.2); al = np.full((D, D), 0.6); be = np.full((D, D), 1.5)
    t, m = gen.ogata_window(th, al, be, 4000.0, gen.rng_for(3, 0))
    rate = len(t) / 4000.0 / D
    assert abs(rate - 1.0) <= 0.15


def test_time_rescaling_ks():
    """Thinning correctness: rescaled inter-event gaps pass KS vs Exp(1)."""
    rc = gen.Recipe(D=3, T=60.0, total_rate=6.0, beta_lo=0.5, beta_hi=3.0, k_cross=1, attack_frac=0.0)
    gaps = []
    for s in range(5):
        rng = gen.rng_for(4, s)
        th, al, be, _ = gen.recipe_params(rc, rng)
        t, m = gen.ogata_window(th, al, be, rc.T, rng)
        for i in range(3):
            gaps.append(rescaled_gaps(t, m, th, al, be, i))
    g = np.concatenate(gaps)
    assert len(g) > 500
    assert stats.kstest(g, "expon").pvalue > 0.01


def test_determinism_and_window_independence():
    rc = gen.Recipe(D=4, T=1.0, total_rate=50.0)
    a = gen.make_batch(rc, 5, seed=11)
    b = gen.make_batch(rc, 5, seed=11)
    np.testing.assert_array_equal(a["t"], b["t"])
    c = gen.make_batch(rc, 2, seed=11, first_window=3)   # windows 3, 4 alone
    s = a["win_off"][3]
    np.testing.assert_array_equal(c["t"], a["t"][s:])


@pytest.mark.gpu
def test_gpu_generator_statistics():
    """libmdhp_synth.so: Poisson counts, the symmetric stationary rate, time-rescaling KS,
    determinism and independence of a window from its batch."""
    import torch
    from synth import gpu as sg
    W = 400
    p = {"theta": torch.full((W, 1), 3.0), "alpha": torch.zeros(W, 1, 1), "beta": torch.ones(W, 1, 1)}
    b = sg.make_batch_gpu(gen.Recipe(D=1, T=100.0, total_rate=300.0), W, seed=5, params=p)
    cnt = np.diff(b["win_off"].cpu().numpy())
    assert abs(cnt.mean() - 300) <= 4 * np.sqrt(300 / W) and abs(cnt.var() / 300 - 1) < 0.25
    D = 2
    p = {"theta": torch.full((8, D), 0.2), "alpha": torch.full((8, D, D), 0.6), "beta": torch.full((8, D, D), 1.5)}
    b = sg.make_batch_gpu(gen.Recipe(D=2, T=2000.0, total_rate=2.0), 8, seed=6, params=p)
    rate = float(b["win_off"][-1]) / 8 / 2000.0 / D
    assert abs(rate - 1.0) <= 0.1
    rc = gen.Recipe(D=3, T=60.0, total_rate=6.0, beta_lo=0.5, beta_hi=3.0, k_cross=1, attack_frac=0.0)
    b = sg.make_batch_gpu(rc, 6, seed=7)
    gaps = []
    for w in range(6):
        a, z = int(b["win_off"][w]), int(b["win_off"][w + 1])
        t = b["t"][a:z].cpu().numpy(); m = b["mark"][a:z].cpu().numpy()
        th, al, be = (b[k][w].double().cpu().numpy() for k in ("theta", "alpha", "beta"))
        assert np.all(np.diff(t) >= 0) and t.min() >= 0 and t.max() <= 60.0
        for i in range(3):
            gaps.append(rescaled_gaps(t, m, th, al, be, i))
    assert stats.kstest(np.concatenate(gaps), "expon").pvalue > 0.01
    b1 = sg.make_batch_gpu("cfg5", 16, seed=2024)
    b2 = sg.make_batch_gpu("cfg5", 4, seed=2024, first_window=12)
    s = int(b1["win_off"][12])
    assert torch.equal(b1["t"][s:], b2["t"]) and torch.equal(b1["alpha"][12:], b2["alpha"])


# ---- row f2: time-exciting injections (Table II shapes, Algorithm 4 NPP) ----
from scipy import integrate  # noqa: E402

STRATS = ["PLA", "DEA", "ASA", "DAM"]


def _bin_expect(strategy, rate, edges):
    """Expected accepted count per bin: rate * int_bin g / g_max (Algorithm 4 thins a Poisson
    candidate stream of the given rate with acceptance g/g_max)."""
    gmax = gen.attack_rate_max(strategy)
    f = lambda u: float(gen.attack_rate(strategy, u)) / gmax
    return np.array([rate * integrate.quad(f, a, b, points=[0.6])[0] for a, b in zip(edges[:-1], edges[1:])])


def _chi2_ok(counts, expect):
    chi = ((counts - expect) ** 2 / expect).sum()
    return stats.chi2.sf(chi, len(counts) - 1) > 1e-3


@pytest.mark.parametrize("strategy", STRATS)
def test_npp_sampler_integral_proportional(strategy):
    """SPEC's sampler property: quartile-bin counts proportional to int g (chi-square), and the
    total count Poisson with mean rate * int g / g_max (Algorithm 4)."""
    rng = np.random.default_rng(42)
    edges = np.linspace(0, 1, 5)
    runs = [gen.npp_sample(strategy, rng, rate=512.0) for _ in range(200)]
    allu = np.concatenate(runs)
    assert all(np.all(np.diff(r) > 0) for r in runs)
    assert allu.min() > 0 and allu.max() <= 1.0
    counts = np.histogram(allu, edges)[0]
    exp = _bin_expect(strategy, 512.0 * len(runs), edges)
    assert _chi2_ok(counts, exp), (counts, exp)


def test_injection_superposed_on_attack_windows_only():
    rc = gen.Recipe(D=4, T=2.0, total_rate=40.0, attack_frac=0.5, inject="PLA", inj_rate=256.0)
    rc0 = gen.Recipe(D=4, T=2.0, total_rate=40.0, attack_frac=0.5)
    a = gen.make_batch(rc, 30, seed=3)
    b = gen.make_batch(rc0, 30, seed=3)
    for w in range(30):
        na = a["win_off"][w + 1] - a["win_off"][w]
        nb = b["win_off"][w + 1] - b["win_off"][w]
        if a["attack"][w]:
            assert na >= nb
        else:
            assert na == nb
        t = a["t"][a["win_off"][w]:a["win_off"][w + 1]]
        assert np.all(np.diff(t) >= 0) and (len(t) == 0 or t.max() <= rc.T)
    assert sum(a["win_off"][1:] - a["win_off"][:-1]) > sum(b["win_off"][1:] - b["win_off"][:-1])


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", STRATS)
def test_gpu_npp_sampler_integral_proportional(strategy):
    from synth import gpu as sg
    W = 400
    u, off = sg.npp_gpu(strategy, W, seed=9, rate=512.0)
    u = u.cpu().numpy(); off = off.cpu().numpy()
    assert u.min() > 0 and u.max() <= 1.0
    assert all(np.all(np.diff(u[off[w]:off[w + 1]]) > 0) for w in range(W))
    edges = np.linspace(0, 1, 5)
    counts = np.histogram(u, edges)[0]
    assert _chi2_ok(counts, _bin_expect(strategy, 512.0 * W, edges)), counts


@pytest.mark.gpu
def test_gpu_injection_is_exact_superposition():
    """synth_ogata_inject = the Hawkes stream of synth_ogata merged with the NPP stream on one ID,
    in attack windows only (the same Philox streams)."""
    import dataclasses
    from synth import gpu as sg
    rc0 = gen.CONFIGS["cfg2"]
    rc = dataclasses.replace(rc0, inject="DAM")
    W = 64
    a = sg.make_batch_gpu(rc, W, seed=12)
    b = sg.make_batch_gpu(rc0, W, seed=12)
    u, uoff = sg.npp_gpu("DAM", W, seed=12, rate=rc.inj_rate)
    ao, bo, uo = (x.cpu().numpy() for x in (a["win_off"], b["win_off"], uoff))
    att = a["attack"].cpu().numpy()
    assert att.any() and (~att.astype(bool)).any()
    for w in range(W):
        ta = a["t"][ao[w]:ao[w + 1]].cpu().numpy(); ma = a["mark"][ao[w]:ao[w + 1]].cpu().numpy()
        tb = b["t"][bo[w]:bo[w + 1]].cpu().numpy(); mb = b["mark"][bo[w]:bo[w + 1]].cpu().numpy()
        if not att[w]:
            assert np.array_equal(ta, tb) and np.array_equal(ma, mb)
            continue
        ti = u[uoff[w]:uoff[w + 1]].cpu().numpy() * rc.T
        assert len(ta) == len(tb) + len(ti)
        assert np.all(np.diff(ta) >= 0)
        merged = np.sort(np.concatenate([tb, ti]), kind="stable")
        assert np.array_equal(ta, merged)
        inj = np.isin(ta, ti)
        assert len(set(ma[inj].tolist())) == 1
