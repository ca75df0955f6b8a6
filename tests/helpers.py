"""Shared test helpers: batch construction (from synth/, the seeded generators), oracle
references on the same inputs, and the tolerance definitions of DESIGN.md R17."""
from __future__ import annotations

import numpy as np

import oracle
from synth import gen


def batch_from_windows(wins, T):
    """wins: list of (t fp64, mark i32).  -> CSR dict."""
    ts = [w[0] for w in wins]
    ms = [w[1] for w in wins]
    off = np.zeros(len(wins) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in ts])
    return {"t": np.concatenate(ts) if ts else np.zeros(0), "mark": np.concatenate(ms).astype(np.int32),
            "win_off": off, "T": np.full(len(wins), float(T)) if np.isscalar(T) else np.asarray(T, float)}


def small_batch(D, W, seed=2024, total_rate=None, T=1.0, edges=True, beta_range=(5.0, 50.0)):
    """W recipe windows (Ogata) of D marks plus the edge windows of synth.gen.edge_windows."""
    rc = gen.Recipe(D=D, T=T, total_rate=total_rate or 24.0 * D, beta_lo=beta_range[0],
                    beta_hi=beta_range[1], k_cross=min(2, D - 1) if D > 1 else 0, n_attack=1)
    b = gen.make_batch(rc, W, seed=seed)
    wins = [(b["t"][b["win_off"][w]:b["win_off"][w + 1]], b["mark"][b["win_off"][w]:b["win_off"][w + 1]])
            for w in range(W)]
    truth = (b["theta"], b["alpha"], b["beta"])
    if edges:
        e = gen.edge_windows(D, T)
        wins = wins + e
        th, al, be = (np.concatenate([x, np.repeat(x[:1], len(e), 0)]) for x in truth)
        truth = (th, al, be)
    return batch_from_windows(wins, T), truth


def random_params(rng, W, D, scale_theta=(0.5, 30.0), alpha=(0.0, 8.0), beta=(0.5, 60.0)):
    th = rng.uniform(*scale_theta, (W, D))
    al = rng.uniform(*alpha, (W, D, D))
    be = rng.uniform(*beta, (W, D, D))
    return th, al, be


def oracle_times(b, D, time_mode=oracle.TIME_RAW, lo=0.0, hi=1.0, tie_policy=oracle.TIE_NUDGE):
    """Oracle's own packing of every window -> (t32 concat, T32 per window, status per window)."""
    W = len(b["win_off"]) - 1
    t32 = np.zeros(len(b["t"]), np.float32)
    T32 = np.zeros(W)
    st = np.zeros(W, np.int32)
    for w in range(W):
        a, z = b["win_off"][w], b["win_off"][w + 1]
        o, T_, s = oracle.convert_window(D, b["t"][a:z], b["mark"][a:z], b["T"][w], time_mode, lo, hi,
                                         tie_policy)
        t32[a:z] = o
        T32[w] = T_
        st[w] = s
    return t32, T32, st


def compensator_terms(t32, mark, T, beta, D):
    """C_ij = sum_{k in j} (1 - e^{-b_ij u_k}) and F_ij = sum_k u_k e^{-b_ij u_k} (fp64), used only
    to build the fp32 error scale of a gradient entry (sum of |terms|), never as a reference."""
    u = T - t32.astype(np.float64)
    C = np.zeros((D, D)); F = np.zeros((D, D))
    for j in range(D):
        uj = u[mark == j]
        if len(uj) == 0:
            continue
        e = np.exp(-beta[:, j][:, None] * uj[None, :])
        C[:, j] = (1 - e).sum(1)
        F[:, j] = (uj[None, :] * e).sum(1)
    return C, F


def grad_scales(t32, mark, T, theta, alpha, beta, ref):
    """Per-entry 'gross' scale of each gradient: the sum of the absolute values of the terms
    whose signed sum is the gradient (R17).  fp32 rounding error is bounded by a small
    multiple of eps * gross; cancellation near an optimum makes |g| << gross."""
    D = len(theta)
    C, F = compensator_terms(t32, mark, T, beta, D)
    sth = (ref["g_theta"] + T) + T
    Eb = -C / beta
    sal = np.abs(ref["g_alpha"] - Eb) + np.abs(Eb)
    t2 = alpha * C / beta ** 2          # -alpha E / beta^2
    t3 = alpha * F / beta               # alpha F / beta
    sbe = np.abs(ref["g_beta"] - t2 + t3) + np.abs(t2) + np.abs(t3)
    return sth, sal, sbe


def assert_grad_close(got, ref, scale, rel=1e-3, gross_rel=1e-4, what=""):
    """|got - ref| <= rel * |ref| + gross_rel * gross  (entrywise)."""
    got = np.asarray(got, np.float64); ref = np.asarray(ref, np.float64)
    tol = rel * np.abs(ref) + gross_rel * scale + 1e-30
    bad = np.abs(got - ref) > tol
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} entries out of tolerance, e.g. "
                             + "; ".join(f"{tuple(i)} got {got[tuple(i)]:.9g} ref {ref[tuple(i)]:.9g} "
                                         f"scale {np.broadcast_to(scale, ref.shape)[tuple(i)]:.3g}" for i in idx))
