"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one
mdhp_pack_windows + the persistent mdhp_fit / mdhp_loglik_grad over the whole batch), checked
on sampled windows the fp64 oracle computes one by one."""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_10258_b200 as M
from synth import gen
from synth import gpu as sg
from tests import helpers as H

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _host(b, w):
    a, z = int(b["win_off"][w]), int(b["win_off"][w + 1])
    return b["t"][a:z].cpu().numpy(), b["mark"][a:z].cpu().numpy()


def _check_ll(D, b, r, windows, th, al, be, time_mode=1):
    for w in windows:
        t, m = _host(b, w)
        T = float(b["T"][w])
        t32, T32, st = oracle.convert_window(D, t, m, T, time_mode, tie_policy=oracle.TIE_NUDGE)
        assert st in (0, 1)
        p = (th[w].double().cpu().numpy(), al[w].double().cpu().numpy(), be[w].double().cpu().numpy())
        ref = oracle.loglik_rec(D, t32, m, T32, *p)
        got = float(r["lnl"][w])
        assert abs(got - ref["lnl"]) <= 1e-4 * abs(ref["lnl"]), (w, got, ref["lnl"])
        sth, sal, sbe = H.grad_scales(t32, m, T32, *p, ref)
        H.assert_grad_close(r["g_theta"][w].cpu().numpy(), ref["g_theta"], sth, what=f"w{w} theta")
        H.assert_grad_close(r["g_alpha"][w].cpu().numpy(), ref["g_alpha"], sal, what=f"w{w} alpha")
        H.assert_grad_close(r["g_beta"][w].cpu().numpy(), ref["g_beta"], sbe, what=f"w{w} beta")


def _check_fit(D, b, fr, windows, th0, al0, be0, cfg_kw, time_mode=1):
    for w in windows:
        t, m = _host(b, w)
        T = float(b["T"][w])
        t32, T32, st = oracle.convert_window(D, t, m, T, time_mode, tie_policy=oracle.TIE_NUDGE)
        o = oracle.fit(D, t32, m, T32, th0[w].double().cpu().numpy(), al0[w].double().cpu().numpy(),
                       be0[w].double().cpu().numpy(), oracle.FitConfig(**cfg_kw))
        assert int(fr["iters"][w]) == o["iters"]
        for k in ("theta", "alpha", "beta"):
            got = fr[k][w].cpu().numpy().astype(np.float64)
            ref = o[k]
            s = 1e-2 * np.mean(np.abs(ref))
            bad = np.abs(got - ref) > 1e-3 * np.maximum(np.abs(ref), s)
            assert not bad.any(), (w, k, got[bad][:4], ref[bad][:4])
        assert abs(float(fr["lnl"][w]) - o["lnl"]) <= 1e-4 * abs(o["lnl"])


def _run(cfg, W, loglik_sample, fit_sample, fit_iters):
    b = sg.make_batch_gpu(cfg, W, seed=2024)
    D = b["D"]
    pk = M.pack_windows(D, b["t"], b["mark"], b["win_off"], b["T"], time_mode=1)
    st = pk.status[:W].cpu().numpy()
    assert np.all((st & M.mdhp.ST_INVALID) == 0)
    th, al, be = b["theta"], b["alpha"], b["beta"]
    r = M.loglik_grad(pk, th, al, be)
    torch.cuda.synchronize()
    lnl = r["lnl"].cpu().numpy()
    assert np.all(np.isfinite(lnl))
    rng = np.random.default_rng(7)
    sample = sorted(set(rng.choice(W, size=min(loglik_sample, W), replace=False).tolist()) | {0, W - 1})
    _check_ll(D, b, r, sample, th, al, be)
    # fit in the bench's configuration (SPEC init, Adam lr 0.05), a few iterations, full batch
    th0 = torch.full((W, D), 0.1, device=DEV); al0 = torch.full((W, D, D), 0.5, device=DEV)
    be0 = torch.full((W, D, D), 1.0, device=DEV)
    kw = dict(max_iters=fit_iters, optimizer="adam", lr=0.05, tol_rel=0.0)
    th1, al1, be1 = th0.clone(), al0.clone(), be0.clone()
    fr = M.fit(pk, th1, al1, be1, M.FitConfig(**kw))
    torch.cuda.synchronize()
    assert np.all(fr["iters"].cpu().numpy() == fit_iters)
    fsample = sample[:fit_sample]
    _check_fit(D, b, {"theta": th1, "alpha": al1, "beta": be1, "lnl": fr["lnl"], "iters": fr["iters"]},
               fsample, th0, al0, be0, kw)


def test_cfg2_full():
    """4,096 windows, D = 8, ~512 events: every window's lnL checked is too slow in Python
    loops, so 256 sampled windows + the first and last, and a 5-iteration fit on 32."""
    _run("cfg2", 4096, 256, 32, 5)


def test_cfg3_full():
    """65,536 windows, D = 32, ~2,048 events (134M events)."""
    _run("cfg3", 65536, 24, 8, 3)


def test_cfg5_full():
    """1,048,576 windows, D = 16, ~1,024 events (1.07e9 events): the bench workload."""
    _run("cfg5", 1 << 20, 48, 16, 3)


def test_cfg1_500_gd():
    """Config 1: one window, D = 2, ~200 events, T = 10 s, 500 GD iterations (mean loss) from
    the SPEC init: fitted parameters within 1e-3 of the oracle's."""
    D = 2
    b = gen.make_batch(gen.CONFIGS["cfg1"], 1, seed=2024, params=gen.CFG1_PARAMS)
    t, m = b["t"], b["mark"]
    assert 120 < len(t) < 320
    bb = H.batch_from_windows([(t, m)], 10.0)
    pk = M.pack_windows(D, torch.tensor(bb["t"], device=DEV), torch.tensor(bb["mark"], device=DEV),
                        torch.tensor(bb["win_off"], device=DEV), torch.tensor(bb["T"], device=DEV))
    kw = dict(max_iters=500, optimizer="gd", lr=0.5, loss="mean", tol_rel=0.0)
    th = torch.full((1, D), 0.1, device=DEV); al = torch.full((1, D, D), 0.5, device=DEV)
    be = torch.full((1, D, D), 1.0, device=DEV)
    fr = M.fit(pk, th, al, be, M.FitConfig(**kw), trace=True)
    torch.cuda.synchronize()
    t32, T32, st = oracle.convert_window(D, t, m, 10.0, tie_policy=oracle.TIE_NUDGE)
    o = oracle.fit(D, t32, m, T32, [0.1, 0.1], np.full((2, 2), 0.5), np.ones((2, 2)), oracle.FitConfig(**kw),
                   trace=True)
    for got, ref in ((th[0], o["theta"]), (al[0], o["alpha"]), (be[0], o["beta"])):
        got = got.cpu().numpy()
        assert np.all(np.abs(got - ref) <= 1e-3 * np.maximum(np.abs(ref), 1e-2 * np.mean(np.abs(ref)))), (got, ref)
    np.testing.assert_allclose(fr["trace"][0].cpu().numpy(), o["trace"], rtol=1e-4)


def test_cfg5_full_bench_fit_500():
    """The bench step itself: 1,048,576 cfg5 windows, SPEC init, Adam lr 0.05, 500 fixed
    iterations in one persistent mdhp_fit launch; the fitted lnL of sampled windows (first,
    last, 6 random) equals the fp64 oracle's 500-iteration fit within 1e-4 relative (R18: long
    Adam runs are compared through lnL)."""
    W, D = 1 << 20, 16
    b = sg.make_batch_gpu("cfg5", W, seed=2024)
    pk = M.pack_windows(D, b["t"], b["mark"], b["win_off"], b["T"], time_mode=1)
    th0 = torch.full((W, D), 0.1, device=DEV); al0 = torch.full((W, D, D), 0.5, device=DEV)
    be0 = torch.full((W, D, D), 1.0, device=DEV)
    kw = dict(max_iters=500, optimizer="adam", lr=0.05, tol_rel=0.0)
    th, al, be = th0.clone(), al0.clone(), be0.clone()
    fr = M.fit(pk, th, al, be, M.FitConfig(**kw))
    torch.cuda.synchronize()
    assert np.all(fr["iters"].cpu().numpy() == 500)
    lnl = fr["lnl"].cpu().numpy()
    assert np.all(np.isfinite(lnl))
    rng = np.random.default_rng(11)
    for w in sorted({0, W - 1} | set(rng.choice(W, 6, replace=False).tolist())):
        t, m = _host(b, w)
        t32, T32, st = oracle.convert_window(D, t, m, float(b["T"][w]), 1, tie_policy=oracle.TIE_NUDGE)
        o = oracle.fit(D, t32, m, T32, np.full(D, 0.1), np.full((D, D), 0.5), np.full((D, D), 1.0),
                       oracle.FitConfig(**kw))
        assert o["iters"] == 500
        assert abs(lnl[w] - o["lnl"]) <= 1e-4 * abs(o["lnl"]), (w, lnl[w], o["lnl"])
