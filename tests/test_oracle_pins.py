"""Pins for the fp64 oracle (CPU only).  Each test checks the oracle against something that is
not the oracle: hand-evaluated worked examples, SPEC examples, closed forms, an independent
quadrature route for Eq.(4), Ozaki's univariate recursion, finite differences, exact
identities, and torch.optim.Adam for the optimizer.  A plausible slip anywhere in the oracle (a
dropped "-1", a transposed alpha/beta index, <= instead of <, a wrong sign in a gradient, a
wrong bias correction) fails at least one of these; see the comment on each test."""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import torch

import oracle
from synth import gen
from tests import pins

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand_case(rng, D, n_per_dim=6, T=1.0, ties=False):
    """Random small window: times rounded to fp32 (the oracle's input type)."""
    ts, ms = [], []
    for j in range(D):
        k = rng.integers(0, n_per_dim + 1)
        ts.append(rng.uniform(0, T, k)); ms.append(np.full(k, j))
    t = np.concatenate(ts); m = np.concatenate(ms).astype(np.int32)
    if ties and len(t) >= 2 and D >= 2:
        # force a cross-dim tie: copy the time of an event of another dim
        a = rng.integers(0, len(t)); b = rng.integers(0, len(t))
        if m[a] != m[b]:
            t[b] = t[a]
    t = t.astype(np.float32).astype(np.float64)
    o = np.lexsort((m, t)); t, m = t[o], m[o]
    # drop accidental same-dim duplicates after rounding
    keep = np.ones(len(t), bool)
    for j in range(D):
        idx = np.where(m == j)[0]
        d = np.diff(t[idx]) == 0
        keep[idx[1:][d]] = False
    t, m = t[keep], m[keep]
    theta = rng.uniform(0.2, 2.0, D)
    alpha = rng.uniform(0.0, 1.5, (D, D))
    beta = rng.uniform(0.5, 6.0, (D, D))
    return t.astype(np.float32), m, T, theta, alpha, beta


# ---------------------------------------------------------------- worked examples / SPEC


def test_hand_values():
    """Hand expansions of Eq.(5) (tests/golden/hand_values.json).  Catches: missing '-1' in
    Part3, transposed alpha/beta (the D=2 cases have asymmetric matrices), <= vs < (tie case),
    wrong Part3 horizon (event at T case)."""
    g = json.load(open(os.path.join(GOLD, "hand_values.json")))
    env = {"log": mpmath.log, "exp": mpmath.exp}
    with mpmath.workdps(30):
        for c in g["cases"]:
            ref = float(eval(c["expr"], env))
            for fn in (oracle.loglik_def, oracle.loglik_rec):
                r = fn(c["D"], np.array(c["t"], np.float32), c["mark"], c["T"], c["theta"], c["alpha"], c["beta"])
                assert abs(r["lnl"] - ref) <= 1e-13 * max(1.0, abs(ref)), (c["name"], fn.__name__, r["lnl"], ref)


def test_spec_examples():
    """SPEC S:53-54 (intensity), S:63-64 (Poisson / empty), S:83 (Gamma with alpha = 0)."""
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for c in g["loglik"]:
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            r = fn(c["D"], np.array(c["t"], np.float32), c["mark"], c["T"], c["theta"], c["alpha"], c["beta"])
            assert r["lnl"] == pytest.approx(c["value"], abs=1e-14), c["cite"]
    for c in g["gamma"]:
        r = oracle.loglik_def(c["D"], np.array(c["t"], np.float32), c["mark"], c["T"], c["theta"], c["alpha"], c["beta"])
        assert r["gamma"] == pytest.approx(c["value"], abs=1e-14), c["cite"]
    # intensity at a query point = d lnL / d(theta_i) contributions are not exposed; use a
    # one-event-at-query trick: lnL(window + event of dim i at t_q) - lnL(window) - [Part3 term of
    # the new event] = ln lambda_i(t_q).  With alpha_.i = 0 for the query dim's column the
    # Part3 term vanishes, so ln lambda = lnL(with) - lnL(without).
    for c in g["intensity"]:
        D = c["D"]
        al = np.array(c["alpha"], float)
        T = max([c["query_t"]] + c["t"]) + 1.0
        t0 = np.array(c["t"], np.float32); m0 = np.array(c["mark"], np.int32)
        # add a new dimension D whose column has alpha = 0 and whose theta equals theta_i,
        # and whose row copies row i: its intensity equals lambda_i at every time.
        D2 = D + 1
        th2 = np.append(np.array(c["theta"], float), c["theta"][c["query_dim"]])
        al2 = np.zeros((D2, D2)); al2[:D, :D] = al; al2[D, :D] = al[c["query_dim"]]
        be2 = np.ones((D2, D2)); be2[:D, :D] = c["beta"]; be2[D, :D] = np.array(c["beta"])[c["query_dim"]]
        t1 = np.append(t0, np.float32(c["query_t"])); m1 = np.append(m0, D)
        o = np.argsort(t1, kind="stable"); t1, m1 = t1[o], m1[o]
        with_ = oracle.loglik_def(D2, t1, m1, T, th2, al2, be2)["lnl"]
        without = oracle.loglik_def(D2, t0, m0, T, th2, al2, be2)["lnl"]
        lam = math.exp(with_ - without)
        ref = c["value"] if "value" in c else eval(c["value_expr"], {"exp": math.exp})
        assert lam == pytest.approx(ref, rel=1e-12), c["cite"]


def test_standardize_examples():
    """Eq.(6) with joint min/max across dims, T_span = Max."""
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for c in g["standardize"]:
        out, T32, st = oracle.convert_window(c["D"], c["t"], c["mark"], c["T"], oracle.TIME_EQ6, c["lo"], c["hi"])
        assert st == oracle.OK, c["cite"]
        np.testing.assert_array_equal(out, np.array(c["out"], np.float32))
        assert T32 == c["T_out"]


def test_convert_validation_statuses():
    """Validation and the RAW / UNIT conversions (fp32 round-to-nearest)."""
    cw = oracle.convert_window
    assert cw(2, [0.1, 0.2], [0, 1], 1.0)[2] == oracle.OK
    assert cw(2, [], [], 1.0)[2] == oracle.EMPTY
    assert cw(2, [0.2, 0.1], [0, 1], 1.0)[2] & oracle.UNSORTED
    assert cw(2, [0.1, 1.5], [0, 1], 1.0)[2] & oracle.OUT_OF_RANGE
    assert cw(2, [-0.1, 0.5], [0, 1], 1.0)[2] & oracle.OUT_OF_RANGE
    assert cw(2, [0.1, float("nan")], [0, 1], 1.0)[2] & oracle.OUT_OF_RANGE
    assert cw(2, [0.1, 0.5], [0, 2], 1.0)[2] & oracle.BAD_MARK
    assert cw(2, [0.1, 0.5], [-1, 0], 1.0)[2] & oracle.BAD_MARK
    assert cw(2, [0.5, 0.5], [0, 0], 1.0)[2] & oracle.SAME_DIM_TIE
    assert cw(2, [0.5, 0.5], [0, 1], 1.0)[2] == oracle.OK            # cross-dim tie is fine
    # distinct in fp64, equal after fp32 rounding -> same-dim tie (R19)
    assert cw(1, [0.5, 0.5 + 1e-12], [0, 0], 1.0)[2] & oracle.SAME_DIM_TIE
    assert cw(2, [0.3, 0.3], [0, 1], 1.0, oracle.TIME_EQ6)[2] & oracle.DEGENERATE
    assert cw(2, [0.1], [0], 0.0)[2] & oracle.BAD_T
    # NUDGE: y_k = max(fl32(x_k), y_{k-1}); a tie with the previous event of the
    # same mark moves to the next float.  Hand example: marks 0,0,1,1 all at x = 0.5:
    # 0.5, 0.5+u, then mark 1 starts at max(0.5, 0.5+u) = 0.5+u, its second event ties -> 0.5+2u.
    x = np.float32(0.5)
    u1 = np.nextafter(x, np.float32(2)); u2 = np.nextafter(u1, np.float32(2))
    out, _, st = cw(2, [0.5, 0.5, 0.5, 0.5], [0, 0, 1, 1], 1.0, tie_policy=oracle.TIE_NUDGE)
    assert st == oracle.OK
    np.testing.assert_array_equal(out, np.array([x, u1, u1, u2], np.float32))
    out, _, st = cw(2, [0.25, 0.5, 0.5 + 1e-12, 0.75], [1, 0, 0, 1], 1.0, tie_policy=oracle.TIE_NUDGE)
    np.testing.assert_array_equal(out, np.array([0.25, x, u1, 0.75], np.float32))
    assert cw(2, [0.5, 0.5], [0, 0], 1.0, tie_policy=oracle.TIE_NUDGE)[2] == oracle.OK
    out, T32, st = cw(1, [0.1, 0.3], [0, 0], 3.0, oracle.TIME_UNIT)
    np.testing.assert_array_equal(out, np.array([0.1 / 3.0, 0.3 / 3.0], np.float32))
    assert T32 == 1.0
    out, T32, st = cw(1, [0.1, 0.3], [0, 0], 3.0, oracle.TIME_RAW)
    np.testing.assert_array_equal(out, np.array([0.1, 0.3], np.float32))
    assert T32 == np.float32(3.0)


# ---------------------------------------------------------------- closed forms / brute force


def test_poisson_closed_form():
    """alpha = 0: lnL = sum_i (N_i ln theta_i - theta_i T), d theta_i = N_i/theta_i - T.
    Catches: Part2 sign/scale, theta gradient."""
    rng = np.random.default_rng(1)
    for D in (1, 3, 5):
        t, m, T, th, al, be = _rand_case(rng, D, 8, T=2.5)
        al = np.zeros((D, D))
        N = np.bincount(m, minlength=D)
        ref = float(np.sum(N * np.log(th) - th * T))
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            r = fn(D, t, m, T, th, al, be)
            assert r["lnl"] == pytest.approx(ref, rel=1e-13, abs=1e-13)
            np.testing.assert_allclose(r["g_theta"], N / th - T, rtol=1e-13, atol=1e-13)


def test_eq4_quadrature_brute_force():
    """Oracle (Eq.(5), App. B closed form) vs Eq.(4) by direct Eq.(2) evaluation + mpmath
    quadrature of Gamma.  Independent route for Part3/Gamma and for Part1's strict
    inequality and index orientation.  Includes cross-dim ties and an event at T."""
    rng = np.random.default_rng(7)
    for k in range(6):
        D = 1 + k % 3
        t, m, T, th, al, be = _rand_case(rng, D, 4, T=1.5, ties=(k % 2 == 0))
        if k == 5 and len(t):
            t[-1] = np.float32(T)
        lnl_q, gam_q = pins.loglik_eq4_quad(th, al, be, t.astype(float), m, T)
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            r = fn(D, t, m, T, th, al, be)
            assert r["lnl"] == pytest.approx(lnl_q, rel=1e-9, abs=1e-9), (k, fn.__name__)
            assert r["gamma"] == pytest.approx(gam_q, rel=1e-9, abs=1e-9)


def test_ozaki_univariate():
    """D = 1 reduces to Ozaki's textbook recursion."""
    rng = np.random.default_rng(3)
    for _ in range(5):
        n = int(rng.integers(1, 40))
        t = np.sort(rng.uniform(0, 4.0, n)).astype(np.float32)
        t = np.unique(t)
        th, al, be = rng.uniform(0.2, 2), rng.uniform(0.1, 2), rng.uniform(0.5, 5)
        ref = pins.ozaki_d1(th, al, be, t.astype(float), 4.0)
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            r = fn(1, t, np.zeros(len(t), np.int32), 4.0, [th], [[al]], [[be]])
            assert r["lnl"] == pytest.approx(ref, rel=1e-12)


def test_def_vs_rec_random():
    """The O(N^2) definition and the eager recursion agree (ties, empty dims, events at 0/T)."""
    rng = np.random.default_rng(11)
    for k in range(40):
        D = int(rng.integers(1, 6))
        t, m, T, th, al, be = _rand_case(rng, D, 10, T=float(rng.uniform(0.5, 3)), ties=(k % 3 == 0))
        a = oracle.loglik_def(D, t, m, T, th, al, be)
        b = oracle.loglik_rec(D, t, m, T, th, al, be)
        assert b["lnl"] == pytest.approx(a["lnl"], rel=1e-12, abs=1e-12)
        for key in ("g_theta", "g_alpha", "g_beta"):
            np.testing.assert_allclose(b[key], a[key], rtol=1e-11, atol=1e-11)
    for D in (2, 3):
        for t, m in gen.edge_windows(D):
            t = t.astype(np.float32); th = np.full(D, 0.7); al = np.full((D, D), 0.4); be = np.full((D, D), 2.0)
            be[0, -1] = 5.0
            a = oracle.loglik_def(D, t, m, 1.0, th, al, be)
            b = oracle.loglik_rec(D, t, m, 1.0, th, al, be)
            assert b["lnl"] == pytest.approx(a["lnl"], rel=1e-13, abs=1e-13)


# ---------------------------------------------------------------- gradients / identities


def test_finite_differences():
    """Analytic gradients vs central differences of lnL.  Catches any sign or
    factor slip in d/d theta, d/d alpha, d/d beta (including the -alpha F / beta term)."""
    rng = np.random.default_rng(5)
    for k in range(8):
        D = 1 + k % 3
        t, m, T, th, al, be = _rand_case(rng, D, 6, T=2.0, ties=(k % 2 == 1))
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            r = fn(D, t, m, T, th, al, be)
            f = lambda th_, al_, be_: fn(D, t, m, T, th_, al_, be_, grads=False)["lnl"]
            for name, arr, g in (("theta", th, r["g_theta"]), ("alpha", al, r["g_alpha"]), ("beta", be, r["g_beta"])):
                flat = arr.reshape(-1)
                for q in range(flat.size):
                    h = 1e-6 * max(1.0, abs(flat[q]))
                    p1 = arr.copy().reshape(-1); p1[q] += h
                    p0 = arr.copy().reshape(-1); p0[q] -= h
                    args1 = [th, al, be]; args0 = [th, al, be]
                    idx = {"theta": 0, "alpha": 1, "beta": 2}[name]
                    args1[idx] = p1.reshape(arr.shape); args0[idx] = p0.reshape(arr.shape)
                    fd = (f(*args1) - f(*args0)) / (2 * h)
                    an = g.reshape(-1)[q]
                    assert an == pytest.approx(fd, rel=1e-6, abs=1e-6), (k, name, q, an, fd)


def test_euler_identity():
    """lambda is homogeneous of degree 1 in (theta, alpha) and Gamma is linear in them, so
    sum theta d_theta + sum alpha d_alpha = N - Gamma exactly (DESIGN.md pins)."""
    rng = np.random.default_rng(9)
    for k in range(20):
        D = int(rng.integers(1, 6))
        t, m, T, th, al, be = _rand_case(rng, D, 10, T=1.7, ties=(k % 2 == 0))
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            r = fn(D, t, m, T, th, al, be)
            lhs = float(np.sum(th * r["g_theta"]) + np.sum(al * r["g_alpha"]))
            assert lhs == pytest.approx(len(t) - r["gamma"], rel=1e-12, abs=1e-11)


def test_time_rescaling():
    """lnL(c t, c T; theta/c, alpha/c, beta/c) = lnL - N ln c (exact); c = 4 keeps fp32 times exact.
    Catches a beta that multiplies the wrong time difference, or a Part3 with a wrong 1/beta."""
    rng = np.random.default_rng(13)
    c = 4.0
    for k in range(10):
        D = int(rng.integers(1, 5))
        t, m, T, th, al, be = _rand_case(rng, D, 8, T=1.0, ties=True)
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            a = fn(D, t, m, T, th, al, be)
            b = fn(D, (t * np.float32(c)).astype(np.float32), m, T * c, th / c, al / c, be / c)
            assert b["lnl"] == pytest.approx(a["lnl"] - len(t) * math.log(c), rel=1e-12, abs=1e-11)
            np.testing.assert_allclose(b["g_theta"], a["g_theta"] * c, rtol=1e-10, atol=1e-10)
            np.testing.assert_allclose(b["g_beta"], a["g_beta"] * c, rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(b["g_alpha"], a["g_alpha"] * c, rtol=1e-9, atol=1e-9)


def test_small_beta_part3():
    """Part3 at beta -> 0: (alpha/beta) sum_k (e^{-beta u_k} - 1) -> -alpha sum_k u_k.  The
    oracle uses expm1, so this limit is exact to fp64 (R20)."""
    t = np.array([0.125, 0.25, 0.5], np.float32); m = np.zeros(3, np.int32)
    T = 1.0
    for b in (1e-4, 1e-7, 1e-10):
        r = oracle.loglik_def(1, t, m, T, [1.0], [[0.5]], [[b]])
        part1 = np.log(1.0) + np.log(1 + 0.5 * np.exp(-b * 0.125)) + np.log(1 + 0.5 * (np.exp(-b * 0.25) + np.exp(-b * 0.375)))
        ref = part1 - 1.0 - 0.5 * (0.875 + 0.75 + 0.5)
        # the next Taylor term of (a/b)(e^{-bu}-1) + a u is a b u^2 / 2 (alternating-series bound)
        bound = 0.5 * b * (0.875 ** 2 + 0.75 ** 2 + 0.5 ** 2) * 0.5
        assert 0.0 <= r["lnl"] - ref <= bound * 1.0001 + 1e-15


# ---------------------------------------------------------------- fit


def _fitcfg(**kw):
    c = oracle.FitConfig(**kw)
    return c


def test_fit_poisson_theta_only():
    """alpha frozen at 0, fit theta only: the MLE is theta_i = N_i / T (north_star pin)."""
    rng = np.random.default_rng(2)
    for D in (1, 4):
        t, m = gen.poisson_window(rng.uniform(5, 40, D), 2.0, rng)
        t = t.astype(np.float32)
        N = np.bincount(m, minlength=D)
        cfg = _fitcfg(max_iters=4000, optimizer="adam", lr=0.2, tol_rel=0.0, fit_mask=1)
        r = oracle.fit(D, t, m, 2.0, np.full(D, 1.0), np.zeros((D, D)), np.ones((D, D)), cfg)
        np.testing.assert_allclose(r["theta"], np.maximum(N / 2.0, 1e-4), rtol=1e-9)
        assert np.all(r["alpha"] == 0.0)
        if D == 1:
            # GD on the mean loss, started near the optimum with lr = theta*^2 / 4 (curvature
            # of -lnL/N at theta* is 1/theta*^2): contraction 3/4 per step.
            ts = N[0] / 2.0
            cfg = _fitcfg(max_iters=300, optimizer="gd", lr=ts * ts / 4, loss="mean", tol_rel=0.0, fit_mask=1)
            r = oracle.fit(D, t, m, 2.0, [0.9 * ts], np.zeros((D, D)), np.ones((D, D)), cfg)
            np.testing.assert_allclose(r["theta"], [ts], rtol=1e-10)


def test_fit_empty_window_floor():
    """Empty window: lnL = -T sum theta, so theta collapses to the floor."""
    cfg = _fitcfg(max_iters=400, optimizer="adam", lr=0.05, tol_rel=0.0)
    r = oracle.fit(2, np.zeros(0, np.float32), np.zeros(0, np.int32), 1.0, [0.1, 0.1],
                   np.full((2, 2), 0.5), np.ones((2, 2)), cfg)
    np.testing.assert_allclose(r["theta"], 1e-4)
    assert r["lnl"] == pytest.approx(-2e-4)


def test_fit_gd_ascent_and_projection():
    """Small-lr GD: the lnL trace never decreases, and every iterate satisfies the projection
    invariants alpha >= 0, beta, theta >= floor."""
    rng = np.random.default_rng(4)
    b = gen.make_batch(gen.Recipe(D=3, T=1.0, total_rate=60.0), 1, seed=5)
    t = b["t"].astype(np.float32); m = b["mark"]
    cfg = _fitcfg(max_iters=200, optimizer="gd", lr=2e-3, loss="mean", tol_rel=0.0)
    r = oracle.fit(3, t, m, 1.0, np.full(3, 0.1), np.full((3, 3), 0.5), np.ones((3, 3)), cfg, trace=True)
    tr = r["trace"]
    assert len(tr) == 200
    assert np.all(np.diff(tr) >= -1e-12 * np.abs(tr[1:]))
    assert np.all(r["alpha"] >= 0) and np.all(r["beta"] >= 1e-4) and np.all(r["theta"] >= 1e-4)
    assert r["lnl"] >= tr[-1]


def test_fit_adam_matches_torch():
    """The oracle's Adam (with projection after each step) equals torch.optim.Adam run with the
    oracle's gradient, in fp64 (library routine as the pin for the optimizer arithmetic)."""
    rng = np.random.default_rng(6)
    D = 2
    t, m, T, th, al, be = _rand_case(rng, D, 12, T=1.0)
    cfg = _fitcfg(max_iters=60, optimizer="adam", lr=0.05, tol_rel=0.0)
    r = oracle.fit(D, t, m, T, th, al, be, cfg)
    p = [torch.tensor(th, dtype=torch.float64, requires_grad=True),
         torch.tensor(al, dtype=torch.float64, requires_grad=True),
         torch.tensor(be, dtype=torch.float64, requires_grad=True)]
    opt = torch.optim.Adam(p, lr=0.05, betas=(0.9, 0.999), eps=1e-8)
    for _ in range(60):
        g = oracle.loglik_def(D, t, m, T, p[0].detach().numpy(), p[1].detach().numpy(), p[2].detach().numpy())
        p[0].grad = torch.tensor(-g["g_theta"]); p[1].grad = torch.tensor(-g["g_alpha"]); p[2].grad = torch.tensor(-g["g_beta"])
        opt.step()
        with torch.no_grad():
            p[0].clamp_(min=1e-4); p[1].clamp_(min=0.0); p[2].clamp_(min=1e-4)
    np.testing.assert_allclose(r["theta"], p[0].detach().numpy(), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r["alpha"], p[1].detach().numpy(), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r["beta"], p[2].detach().numpy(), rtol=1e-9, atol=1e-12)


def test_fit_fixed_beta_kkt():
    """lnL is concave in (theta, alpha) at fixed beta; at the optimum the KKT conditions hold and,
    by the Euler identity, Gamma = N - sum_{theta at floor} theta d_theta.  A long (theta, alpha)
    fit must satisfy both (catches an optimizer that stalls, a wrong projection, or a gradient
    that is not the gradient of the evaluated lnL)."""
    b = gen.make_batch(gen.Recipe(D=2, T=1.0, total_rate=80.0), 1, seed=8)
    t = b["t"].astype(np.float32); m = b["mark"]; D = 2
    be = b["beta"][0]
    cfg = _fitcfg(max_iters=20000, optimizer="adam", lr=0.05, tol_rel=0.0, fit_mask=3)
    r = oracle.fit(D, t, m, 1.0, np.full(D, 10.0), np.full((D, D), 1.0), be, cfg)
    g = oracle.loglik_def(D, t, m, 1.0, r["theta"], r["alpha"], r["beta"])
    N = len(t)
    at_floor = r["theta"] <= 1e-4
    assert g["gamma"] == pytest.approx(N - float(np.sum((r["theta"] * g["g_theta"])[at_floor])), abs=1e-9)
    assert np.all(np.abs(g["g_theta"][~at_floor]) < 1e-8) and np.all(g["g_theta"][at_floor] <= 0)
    pos = r["alpha"] > 0
    assert np.all(np.abs(g["g_alpha"][pos]) < 1e-8)
    assert np.all(g["g_alpha"][~pos] <= 1e-12)


def test_fit_nonfinite_rollback():
    """A step that produces non-finite parameters is rolled back and lr halved; with the
    halving budget exhausted the window is DIVERGED and keeps its last finite point."""
    t = np.array([0.1, 0.2, 0.3], np.float32); m = np.zeros(3, np.int32)
    cfg = _fitcfg(max_iters=50, optimizer="gd", lr=1e308, tol_rel=0.0, max_halvings=3)
    r = oracle.fit(1, t, m, 1.0, [0.5], [[0.5]], [[1.0]], cfg)
    assert r["status"] & oracle.DIVERGED
    assert np.isfinite(r["lnl"])
    cfg = _fitcfg(max_iters=50, optimizer="gd", lr=1e308, tol_rel=0.0, max_halvings=2000)
    r = oracle.fit(1, t, m, 1.0, [0.5], [[0.5]], [[1.0]], cfg)
    assert not (r["status"] & oracle.DIVERGED)
    assert r["iters"] == 50 and np.isfinite(r["lnl"])


def test_fit_convergence_stop():
    """tol_rel / patience stop rule: the fit stops early with CONVERGED."""
    b = gen.make_batch(gen.Recipe(D=2, T=1.0, total_rate=60.0), 1, seed=12)
    t = b["t"].astype(np.float32); m = b["mark"]
    cfg = _fitcfg(max_iters=3000, optimizer="adam", lr=0.05, tol_rel=1e-6, patience=10)
    r = oracle.fit(2, t, m, 1.0, np.full(2, 0.1), np.full((2, 2), 0.5), np.ones((2, 2)), cfg, trace=True)
    assert r["status"] & oracle.CONVERGED
    assert r["iters"] < 3000
    tr = r["trace"]
    last = np.abs(np.diff(tr[-11:])) <= 1e-6 * np.maximum(np.abs(tr[-11:-1]), 1.0)
    assert last.all()


def test_batch_equals_single():
    """Thread-pool batch = per-window calls, bit for bit (determinism)."""
    b = gen.make_batch(gen.Recipe(D=3, T=1.0, total_rate=40.0), 6, seed=21)
    D = 3; W = 6
    t32 = b["t"].astype(np.float32)
    th = np.full((W, D), 0.3); al = np.full((W, D, D), 0.2); be = np.full((W, D, D), 3.0)
    rb = oracle.loglik_batch(D, t32, b["mark"], b["win_off"], b["T"], th, al, be, nthreads=3)
    for w in range(W):
        a, z = b["win_off"][w], b["win_off"][w + 1]
        r = oracle.loglik_rec(D, t32[a:z], b["mark"][a:z], 1.0, th[w], al[w], be[w])
        assert rb["lnl"][w] == r["lnl"]
        assert np.array_equal(rb["g_beta"][w], r["g_beta"])
    cfg = _fitcfg(max_iters=20, optimizer="adam")
    fb = oracle.fit_batch(D, t32, b["mark"], b["win_off"], b["T"], th, al, be, cfg, nthreads=4)
    for w in (0, 5):
        a, z = b["win_off"][w], b["win_off"][w + 1]
        r = oracle.fit(D, t32[a:z], b["mark"][a:z], 1.0, th[w], al[w], be[w], cfg)
        assert fb["lnl"][w] == r["lnl"] and np.array_equal(fb["alpha"][w], r["alpha"])


def test_mark_relabeling_invariance():
    """Relabelling the marks by a permutation pi (and theta, alpha, beta with it:
    theta'[pi i] = theta[i], alpha'[pi i][pi j] = alpha[i][j]) leaves lnL unchanged and permutes
    the gradients the same way.  Catches any index that mixes target and source (alpha[i][j]
    used as alpha[j][i]) on non-symmetric parameters, in both routes."""
    rng = np.random.default_rng(21)
    for k in range(12):
        D = int(rng.integers(2, 6))
        t, m, T, th, al, be = _rand_case(rng, D, 8, T=1.3, ties=(k % 2 == 0))
        pi = rng.permutation(D)
        inv = np.argsort(pi)
        m2 = pi[m].astype(np.int32)
        th2 = th[inv]
        al2 = al[np.ix_(inv, inv)]
        be2 = be[np.ix_(inv, inv)]
        for fn in (oracle.loglik_def, oracle.loglik_rec):
            a = fn(D, t, m, T, th, al, be)
            b = fn(D, t, m2, T, th2, al2, be2)
            assert b["lnl"] == pytest.approx(a["lnl"], rel=1e-13, abs=1e-13)
            np.testing.assert_allclose(b["g_theta"], a["g_theta"][inv], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(b["g_alpha"], a["g_alpha"][np.ix_(inv, inv)], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(b["g_beta"], a["g_beta"][np.ix_(inv, inv)], rtol=1e-11, atol=1e-11)
