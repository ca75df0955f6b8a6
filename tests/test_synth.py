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
