"""GPU parity of the long-sequence path (row a7: chunked parallel scan) against the fp64 oracle on
the sequence's fp64 times (the GPU stores chunk-relative fp32 times; R19)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_10258_b200 as M
from paper_2411_10258_b200 import mdhp
from synth import gen
from tests import helpers as H

pytestmark = pytest.mark.gpu
DEV = "cuda"


def f32(x):
    return np.asarray(x, np.float32)


def seq_case(D, T, rate, seed, ties=False):
    rc = gen.Recipe(D=D, T=T, total_rate=rate, beta_lo=0.5, beta_hi=5.0, k_cross=min(2, D - 1),
                    attack_frac=0.0)
    b = gen.make_batch(rc, 1, seed=seed)
    t, m = b["t"], b["mark"]
    if ties and len(t) > 10:
        # equal times across marks at several places (incl. around chunk boundaries)
        for k in range(5, len(t) - 1, 37):
            if m[k] != m[k + 1]:
                t[k + 1] = t[k]
    return t, m, (b["theta"][0], b["alpha"][0], b["beta"][0])


def gpu_seq(D, t, m, T, th, al, be, ce=64, grads=True):
    ps = M.seq_pack(D, torch.tensor(t, dtype=torch.float64, device=DEV),
                    torch.tensor(m, dtype=torch.int32, device=DEV), T, chunk_events=ce)
    r = M.seq_loglik_grad(ps, torch.tensor(f32(th), device=DEV), torch.tensor(f32(al), device=DEV),
                          torch.tensor(f32(be), device=DEV), grads=grads)
    torch.cuda.synchronize()
    out = {k: (v.cpu().numpy() if v is not None else None) for k, v in r.items()}
    out["status"] = int(ps.status.cpu()[0])
    return out


def check(D, t, m, T, th, al, be, ce, what, use_def=True):
    out = gpu_seq(D, t, m, T, th, al, be, ce)
    p = (f32(th).astype(float), f32(al).astype(float), f32(be).astype(float))
    fn = oracle.loglik_def if use_def else oracle.loglik_rec
    ref = fn(D, t, m, T, *p)
    rel = abs(out["lnl"][0] - ref["lnl"]) / abs(ref["lnl"])
    assert rel <= 1e-4, (what, out["lnl"][0], ref["lnl"], rel)
    sth, sal, sbe = H.grad_scales(t, m, T, *p, ref)
    H.assert_grad_close(out["g_theta"], ref["g_theta"], sth, what=f"{what} theta")
    H.assert_grad_close(out["g_alpha"], ref["g_alpha"], sal, what=f"{what} alpha")
    H.assert_grad_close(out["g_beta"], ref["g_beta"], sbe, what=f"{what} beta")
    return out, ref, rel


@pytest.mark.parametrize("D", [1, 3, 8, 12, 16, 20])
def test_seq_vs_definition(D):
    """Several hundred chunks; lnL within 1e-4 (expected ~1e-6) of Eq.(5) written out."""
    t, m, p = seq_case(D, 60.0, 40.0, seed=10 + D)
    check(D, t, m, 60.0, *p, ce=16, what=f"D{D}")


@pytest.mark.parametrize("ce", [8, 64, 256, 100000])
def test_seq_chunk_size_invariance_and_ties(ce):
    """Cross-mark ties (some straddling nominal chunk boundaries, which are moved past tie
    groups) and chunk sizes from 8 events to a single chunk."""
    D = 4
    t, m, p = seq_case(D, 40.0, 50.0, seed=3, ties=True)
    check(D, t, m, 40.0, *p, ce=ce, what=f"ce{ce}")


def test_seq_matches_window_path():
    """The same sequence through mdhp_loglik_grad as one window (RAW time, T small enough for
    absolute fp32 times) and through the chunked scan agree to fp32 rounding."""
    D = 5
    t, m, (th, al, be) = seq_case(D, 8.0, 60.0, seed=21)
    s = gpu_seq(D, t, m, 8.0, th, al, be, ce=32)
    b = H.batch_from_windows([(t, m)], 8.0)
    pk = M.pack_windows(D, torch.tensor(b["t"], device=DEV), torch.tensor(b["mark"], device=DEV),
                        torch.tensor(b["win_off"], device=DEV), torch.tensor(b["T"], device=DEV))
    r = M.loglik_grad(pk, torch.tensor(f32(th)[None], device=DEV), torch.tensor(f32(al)[None], device=DEV),
                      torch.tensor(f32(be)[None], device=DEV))
    lw = float(r["lnl"][0])
    assert abs(s["lnl"][0] - lw) <= 1e-5 * abs(lw)
    np.testing.assert_allclose(s["g_alpha"], r["g_alpha"][0].cpu().numpy(), rtol=2e-3, atol=1e-3)


def test_seq_invalid_and_empty():
    D = 2
    o = gpu_seq(D, np.array([0.5, 0.25]), np.array([0, 1], np.int32), 1.0, [1, 1], np.ones((2, 2)),
                np.ones((2, 2)))
    assert o["status"] & mdhp.ST_UNSORTED and np.isnan(o["lnl"][0])
    o = gpu_seq(D, np.array([0.25, 0.25]), np.array([1, 1], np.int32), 1.0, [1, 1], np.ones((2, 2)),
                np.ones((2, 2)))
    assert o["status"] & mdhp.ST_SAME_DIM_TIE
    o = gpu_seq(D, np.zeros(0), np.zeros(0, np.int32), 3.0, [0.5, 0.25], np.ones((2, 2)), np.ones((2, 2)))
    assert o["status"] == mdhp.ST_EMPTY
    assert o["lnl"][0] == pytest.approx(-3.0 * 0.75)
    np.testing.assert_allclose(o["g_theta"], [-3.0, -3.0])


@pytest.mark.parametrize("opt", ["gd", "adam"])
def test_seq_fit_parity(opt):
    D = 3
    t, m, _ = seq_case(D, 30.0, 30.0, seed=31)
    th0 = np.full(D, 2.0); al0 = np.full((D, D), 0.5); be0 = np.full((D, D), 2.0)
    kw = dict(max_iters=25, optimizer=opt, lr=0.05 if opt == "adam" else 0.2, loss="mean" if opt == "gd" else "sum",
              tol_rel=0.0)
    ps = M.seq_pack(D, torch.tensor(t, device=DEV), torch.tensor(m, dtype=torch.int32, device=DEV), 30.0,
                    chunk_events=32)
    th = torch.tensor(f32(th0), device=DEV); al = torch.tensor(f32(al0), device=DEV)
    be = torch.tensor(f32(be0), device=DEV)
    r = M.seq_fit(ps, th, al, be, M.FitConfig(**kw), trace=True)
    torch.cuda.synchronize()
    o = oracle.fit(D, t, m, 30.0, th0, al0, be0, oracle.FitConfig(**kw), trace=True)
    assert int(r["iters"][0]) == o["iters"] == 25
    for got, ref in ((th, o["theta"]), (al, o["alpha"]), (be, o["beta"])):
        got = got.cpu().numpy()
        s = 1e-2 * np.mean(np.abs(ref))
        assert np.all(np.abs(got - ref) <= 1e-3 * np.maximum(np.abs(ref), s)), (got, ref)
    assert abs(float(r["lnl"][0]) - o["lnl"]) <= 1e-4 * abs(o["lnl"])
    np.testing.assert_allclose(r["trace"].cpu().numpy(), o["trace"], rtol=1e-4)


def test_seq_cfg4_full_size():
    """BASELINE config 4 at full size: one sequence, D = 16, ~1e6 events over 1000 s, generated
    on the GPU (synth), chunked scan vs the eager fp64 oracle recursion on the same fp64 times."""
    from synth import gpu as sg
    b = sg.make_batch_gpu("cfg4", 1, seed=2024)
    D = 16
    t = b["t"].cpu().numpy(); m = b["mark"].cpu().numpy()
    assert len(t) > 500_000
    th, al, be = (b[k][0].cpu().numpy() for k in ("theta", "alpha", "beta"))
    out, ref, rel = check(D, t, m, 1000.0, th, al, be, ce=256, what="cfg4", use_def=False)
    assert rel < 1e-5


def test_seq_fit_resume_is_exact():
    """Long-sequence fit: fit(15) + fit(10, opt_state, adam_step0=15) == fit(25) bit for bit."""
    D = 3
    t, m, _ = seq_case(D, 30.0, 30.0, seed=32)
    ps = M.seq_pack(D, torch.tensor(t, device=DEV), torch.tensor(m, dtype=torch.int32, device=DEV), 30.0,
                    chunk_events=32)
    P = D + 2 * D * D
    init = (torch.full((D,), 2.0, device=DEV), torch.full((D, D), 0.5, device=DEV),
            torch.full((D, D), 2.0, device=DEV))
    kw = dict(optimizer="adam", lr=0.05, tol_rel=0.0)
    a = [x.clone() for x in init]
    oa = torch.zeros(2 * P, device=DEV)
    ra = M.seq_fit(ps, *a, M.FitConfig(max_iters=25, **kw), opt_state=oa)
    c = [x.clone() for x in init]
    oc = torch.zeros(2 * P, device=DEV)
    M.seq_fit(ps, *c, M.FitConfig(max_iters=15, **kw), opt_state=oc)
    rc = M.seq_fit(ps, *c, M.FitConfig(max_iters=10, adam_step0=15, **kw), opt_state=oc)
    torch.cuda.synchronize()
    for x, y in zip(a, c):
        assert torch.equal(x, y)
    assert torch.equal(oa, oc) and torch.equal(ra["lnl"], rc["lnl"])
