"""Seeded synthetic MDHP event generators (CPU, numpy) — input synthesis only.

This module serves both sides of every parity test (the fp64 oracle in ``oracle/`` and the
CUDA path in ``paper_2411_10258_b200``) and imports neither.  It holds none of the
likelihood / gradient / fit arithmetic; it only *simulates* event streams:

* ``ogata_window``   Ogata thinning for the Eq.(2) intensity: propose at the
                     current total intensity (non-increasing between events because
                     alpha >= 0), accept dimension i with probability lambda_i / bound
                     (SPEC S:211).  Pair state is decayed eagerly (O(D^2) per proposal).
* ``recipe_params``  parameter recipe of DESIGN.md "Inputs" (CAN / SOME-IP shaped rates,
                     self + k cross excitations, attack bursts on n_a IDs; 50% attack
                     windows as in STEIA9).
* ``make_batch``     CSR batch (t fp64[E], mark i32[E], win_off i64[W+1], T f64[W]).
* ``attack_rate``, ``npp_sample``  the Table II attack-rate shapes and Algorithm 4
                     (NPP thinning) for time-exciting injections (row f2).
* ``edge_windows``   hand-built edge cases (empty window, empty dims, cross-dim ties,
                     events at t = 0 and t = T, a single event).

The GPU generator used for the 1e9-event bench inputs lives in ``synth/csrc/synth.cu``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def rng_for(seed: int, window: int) -> np.random.Generator:
    """Independent stream per (seed, window): a window's events do not depend on the batch."""
    return np.random.Generator(np.random.Philox(key=[int(seed) & 0xFFFFFFFFFFFFFFFF, int(window)]))


def ogata_window(theta, alpha, beta, T, rng, max_events=2_000_000):
    """Simulate one window on [0, T] with empty history.  Returns (t fp64 ascending, mark i32)."""
    theta = np.asarray(theta, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    D = theta.shape[0]
    exc = np.zeros((D, D))   # exc[i, j] = sum_{k in j, t_k <= now} exp(-beta_ij (now - t_k))
    now = 0.0
    ts, ms = [], []
    while True:
        bound = float(theta.sum() + (alpha * exc).sum())   # total intensity just after `now`
        if bound <= 0.0:
            break
        cand = now + rng.exponential(1.0 / bound)
        if cand > T:
            break
        exc = exc * np.exp(-beta * (cand - now))
        now = cand
        lam = theta + (alpha * exc).sum(axis=1)
        u = rng.uniform() * bound
        cum = np.cumsum(lam)
        if u <= cum[-1]:
            i = min(int(np.searchsorted(cum, u, side="left")), D - 1)
            ts.append(now)
            ms.append(i)
            exc[:, i] += 1.0
            if len(ts) >= max_events:
                raise RuntimeError("max_events exceeded (unstable parameters?)")
    return np.asarray(ts, dtype=np.float64), np.asarray(ms, dtype=np.int32)


@dataclass
class Recipe:
    """per-ID stationary rates r_i (log-uniform, scaled to total_rate),
    branching G = alpha/beta with self terms U(g_self) and k cross terms U(g_cross) per row,
    max row sum of G rescaled to <= rho (a bound on the spectral radius), beta log-uniform,
    theta = (I - G) r (floored at 5% of r).  Attack windows put G_aa = 0.7 (+ one 0.2 cross
    entry) on n_a random IDs and allow rho_attack."""
    D: int = 8
    T: float = 1.0
    total_rate: float = 512.0
    rate_lo: float = 10.0
    rate_hi: float = 200.0
    beta_lo: float = 5.0
    beta_hi: float = 50.0
    g_self: tuple = (0.1, 0.3)
    g_cross: tuple = (0.02, 0.1)
    k_cross: int = 1
    rho: float = 0.6
    attack_frac: float = 0.5
    n_attack: int = 1
    rho_attack: float = 0.9
    inject: str = "none"        # injection strategy in attack windows: none | PLA | DEA | ASA | DAM
    inj_rate: float = 512.0     # Algorithm 4 candidate rate per unit normalised time


CONFIGS = {
    # BASELINE.json configs; DESIGN.md "Inputs" gives the recipe for each.
    "cfg1": Recipe(D=2, T=10.0, total_rate=20.0, rate_lo=10.0, rate_hi=10.0, attack_frac=0.0),
    "cfg2": Recipe(D=8, T=1.0, total_rate=512.0, beta_lo=5.0, beta_hi=50.0, k_cross=1, n_attack=1),
    "cfg3": Recipe(D=32, T=1.0, total_rate=2048.0, beta_lo=10.0, beta_hi=200.0, k_cross=2, n_attack=3),
    "cfg4": Recipe(D=16, T=1000.0, total_rate=1000.0, beta_lo=5.0, beta_hi=50.0, k_cross=2, rho=0.5,
                   attack_frac=0.0),
    "cfg5": Recipe(D=16, T=1.0, total_rate=1024.0, beta_lo=5.0, beta_hi=50.0, k_cross=2, n_attack=2),
}

CFG1_PARAMS = dict(  # BASELINE cfg1 / SURVEY 8(d): rho = 0.612, stationary E[N] = 200 on T = 10 s
    theta=np.array([3.875, 3.875]),
    alpha=np.array([[0.8, 0.4], [0.3, 0.9]]),
    beta=np.array([[2.0, 1.5], [1.5, 2.5]]),
)


STRATEGIES = {"none": 0, "PLA": 1, "DEA": 2, "ASA": 3, "DAM": 4}


def attack_rate(strategy: str, u):
    """Table II attack-rate shapes on the normalised window u in [0, 1] with
    the constants of DESIGN.md R23."""
    u = np.asarray(u, dtype=np.float64)
    if strategy == "PLA":                      # a t^b
        return 1.0 * u ** 2
    if strategy == "DEA":                      # W1 a1 t^(a1-1) | W2 a2 e^{gamma (t - t1)}
        return np.where(u < 0.6, 1.0 * 2.0 * u, 1.0 * 1.2 * np.exp(4.0 * (u - 0.6)))
    if strategy == "ASA":                      # C e^{gamma t} / (1 + e^{gamma (t - t0)})^2
        return np.exp(10.0 * u) / (1.0 + np.exp(10.0 * (u - 0.5))) ** 2
    if strategy == "DAM":                      # w a1 t^(a1-1) + (1 - w) a2 e^{a2 t}
        return 0.5 * 3.0 * u ** 2 + 0.5 * 4.0 * np.exp(4.0 * u)
    raise ValueError(strategy)


def attack_rate_max(strategy: str) -> float:
    """max of g on [0, 1] by dense evaluation (Algorithm 6's "max(evaluate g(t))")."""
    return float(attack_rate(strategy, np.arange(4097) / 4096.0).max()) * (1.0 + 1e-9)


def npp_sample(strategy: str, rng: np.random.Generator, rate: float = 512.0, t_min=0.0, t_max=1.0):
    """Algorithm 4: candidate gaps Exponential(mean 1/rate), accept a candidate t
    with u ~ Uniform(0, g_max) < g(t).  Returns the accepted times (ascending)."""
    gmax = attack_rate_max(strategy)
    t, out = t_min, []
    while t < t_max:
        t += rng.exponential(1.0 / rate)
        if t > t_max:
            break
        if rng.uniform(0.0, gmax) < float(attack_rate(strategy, t)):
            out.append(t)
    return np.asarray(out, dtype=np.float64)


def recipe_params(rc: Recipe, rng: np.random.Generator):
    """-> (theta[D], alpha[D,D], beta[D,D], is_attack) in seconds (RAW time)."""
    D = rc.D
    if rc.rate_hi > rc.rate_lo:
        r = np.exp(rng.uniform(np.log(rc.rate_lo), np.log(rc.rate_hi), D))
    else:
        r = np.full(D, rc.rate_lo)
    r *= rc.total_rate / r.sum()
    G = np.zeros((D, D))
    G[np.arange(D), np.arange(D)] = rng.uniform(*rc.g_self, D)
    for i in range(D):
        if D > 1 and rc.k_cross > 0:
            others = [j for j in range(D) if j != i]
            for j in rng.choice(others, size=min(rc.k_cross, D - 1), replace=False):
                G[i, j] = rng.uniform(*rc.g_cross)
    attack = bool(rng.uniform() < rc.attack_frac)
    rho = rc.rho
    if attack:
        rho = rc.rho_attack
        for a in rng.choice(D, size=min(rc.n_attack, D), replace=False):
            G[a, a] = 0.7
            if D > 1:
                b = int(rng.choice([j for j in range(D) if j != a]))
                G[a, b] = 0.2
    rs = G.sum(axis=1).max()
    if rs > rho:
        G *= rho / rs
    beta = np.exp(rng.uniform(np.log(rc.beta_lo), np.log(rc.beta_hi), (D, D)))
    alpha = G * beta
    theta = np.maximum(r - G @ r, 0.05 * r)
    return theta, alpha, beta, attack


def make_batch(rc: Recipe, W: int, seed: int = 2024, first_window: int = 0, params=None):
    """Simulate W windows (global indices first_window ...).  Returns dict with CSR arrays,
    the true parameters (theta [W,D], alpha [W,D,D], beta [W,D,D]) and attack flags."""
    D = rc.D
    ts, ms, offs = [], [], [0]
    TH = np.zeros((W, D)); AL = np.zeros((W, D, D)); BE = np.zeros((W, D, D))
    att = np.zeros(W, dtype=bool)
    for w in range(W):
        rng = rng_for(seed, first_window + w)
        if params is None:
            th, al, be, a = recipe_params(rc, rng)
        else:
            th, al, be = (np.asarray(params[k], dtype=np.float64) for k in ("theta", "alpha", "beta"))
            a = False
        t, m = ogata_window(th, al, be, rc.T, rng)
        if a and rc.inject != "none":
            # injections superposed on the Hawkes traffic, on one random ID
            k = int(rng.integers(D))
            ti = npp_sample(rc.inject, rng, rc.inj_rate) * rc.T
            t = np.concatenate([t, ti]); m = np.concatenate([m, np.full(len(ti), k, np.int32)])
            o = np.argsort(t, kind="stable"); t, m = t[o], m[o]
        ts.append(t); ms.append(m); offs.append(offs[-1] + len(t))
        TH[w], AL[w], BE[w], att[w] = th, al, be, a
    return {
        "D": D, "t": np.concatenate(ts) if ts else np.zeros(0), "mark": np.concatenate(ms).astype(np.int32)
        if ms else np.zeros(0, np.int32), "win_off": np.asarray(offs, dtype=np.int64),
        "T": np.full(W, rc.T, dtype=np.float64), "theta": TH, "alpha": AL, "beta": BE, "attack": att,
    }


def poisson_window(rates, T, rng):
    """Homogeneous Poisson events per dim (alpha = 0 ground truth), merged and sorted."""
    ts, ms = [], []
    for i, r in enumerate(rates):
        n = rng.poisson(r * T)
        ts.append(rng.uniform(0.0, T, n)); ms.append(np.full(n, i, dtype=np.int32))
    t = np.concatenate(ts); m = np.concatenate(ms)
    o = np.argsort(t, kind="stable")
    return t[o], m[o]


def edge_windows(D: int, T: float = 1.0):
    """Hand-built windows exercising the degenerate cases the method has (R9-R15).
    Times are multiples of 1/64 so that they are exact in fp32 and cross-dim ties survive
    rounding.  Returns a list of (t, mark)."""
    q = T / 64.0
    out = []
    out.append((np.zeros(0), np.zeros(0, np.int32)))                          # empty window
    out.append((np.array([0.0]), np.array([0], np.int32)))                     # single event at 0
    out.append((np.array([T]), np.array([D - 1], np.int32)))                   # single event at T
    if D >= 2:
        out.append((np.array([8 * q, 8 * q, 9 * q]), np.array([0, 1, 0], np.int32)))   # cross-dim tie
        ts = np.array([0.0, 0.0, 3 * q, 5 * q, 5 * q, 5 * q, 64 * q])
        ms = np.array([0, 1, 1, 0, 1, D - 1, 1], np.int32)
        if D == 2:
            ms = np.array([0, 1, 1, 0, 1, 0, 1], np.int32)
            ts = np.array([0.0, 0.0, 3 * q, 5 * q, 5 * q, 6 * q, 64 * q])
        out.append((ts, ms))                                                   # ties at 0, ties, event at T
        # only dim 0 active; every other dim empty
        out.append((np.arange(1, 20) * q, np.zeros(19, np.int32)))
    return out
