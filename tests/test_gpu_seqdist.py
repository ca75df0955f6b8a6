"""f1: one sequence split over R ranks with the map exchange, emulated in one process
on one GPU (LocalComm: every kernel completes before the exchange), against the single-GPU
chunked-scan path and the fp64 oracle."""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_10258_b200 as M
from paper_2411_10258_b200 import seqdist
from tests import helpers as H
from tests.test_gpu_seq import seq_case

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _slices(D, t, m, T, R, ce=32, cfg=None):
    td = torch.tensor(t, dtype=torch.float64, device=DEV)
    md = torch.tensor(m, dtype=torch.int32, device=DEV)
    ctxs = []
    for r, (lo, hi) in enumerate(seqdist.slice_bounds(t, R)):
        t0 = float(t[lo - 1]) if lo > 0 else 0.0
        ctxs.append(seqdist.make_slice(D, td[lo:hi].contiguous(), md[lo:hi].contiguous(), T, t0, r,
                                       chunk_events=ce, cfg=cfg))
    return ctxs


@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_dist_loglik_matches_single_and_oracle(R):
    D = 4
    t, m, (th, al, be) = seq_case(D, 50.0, 40.0, seed=41, ties=True)
    f = lambda x: torch.tensor(np.asarray(x, np.float32), device=DEV)
    ctxs = _slices(D, t, m, 50.0, R)
    d = seqdist.loglik_grad(ctxs, seqdist.LocalComm(R), f(th), f(al), f(be), n_total=len(t))
    ps = M.seq_pack(D, torch.tensor(t, device=DEV), torch.tensor(m, dtype=torch.int32, device=DEV), 50.0,
                    chunk_events=32)
    s = M.seq_loglik_grad(ps, f(th), f(al), f(be))
    torch.cuda.synchronize()
    assert float(d["lnl"][0]) == pytest.approx(float(s["lnl"][0]), rel=2e-6)
    np.testing.assert_allclose(d["g_alpha"].cpu().numpy(), s["g_alpha"].cpu().numpy(), rtol=1e-3, atol=1e-3)
    p = [np.asarray(x, np.float32).astype(float) for x in (th, al, be)]
    ref = oracle.loglik_def(D, t, m, 50.0, *p)
    assert abs(float(d["lnl"][0]) - ref["lnl"]) <= 1e-4 * abs(ref["lnl"])
    sth, sal, sbe = H.grad_scales(t, m, 50.0, *p, ref)
    H.assert_grad_close(d["g_theta"].cpu().numpy(), ref["g_theta"], sth, what="theta")
    H.assert_grad_close(d["g_alpha"].cpu().numpy(), ref["g_alpha"], sal, what="alpha")
    H.assert_grad_close(d["g_beta"].cpu().numpy(), ref["g_beta"], sbe, what="beta")


def test_dist_with_empty_slice():
    D = 2
    t = np.sort(np.random.default_rng(1).uniform(0, 5.0, 6)); m = np.array([0, 1, 0, 1, 1, 0], np.int32)
    th, al, be = [0.7, 0.4], np.full((D, D), 0.5), np.full((D, D), 2.0)
    f = lambda x: torch.tensor(np.asarray(x, np.float32), device=DEV)
    ctxs = _slices(D, t, m, 5.0, 8, ce=8)          # 8 ranks for 6 events: some slices empty
    d = seqdist.loglik_grad(ctxs, seqdist.LocalComm(8), f(th), f(al), f(be), n_total=len(t))
    ref = oracle.loglik_def(D, t, m, 5.0, *[np.asarray(x, np.float32).astype(float) for x in (th, al, be)])
    assert abs(float(d["lnl"][0]) - ref["lnl"]) <= 1e-5 * abs(ref["lnl"])


@pytest.mark.parametrize("opt", ["gd", "adam"])
def test_dist_fit_matches_single(opt):
    D = 3
    t, m, _ = seq_case(D, 30.0, 30.0, seed=31)
    kw = dict(max_iters=20, optimizer=opt, lr=0.05 if opt == "adam" else 0.2, loss="mean" if opt == "gd" else "sum",
              tol_rel=0.0)
    cfg = M.FitConfig(**kw)
    R = 3
    ctxs = _slices(D, t, m, 30.0, R, cfg=cfg)
    init = (np.full(D, 2.0, np.float32), np.full((D, D), 0.5, np.float32), np.full((D, D), 2.0, np.float32))
    params = [{"theta": torch.tensor(init[0], device=DEV), "alpha": torch.tensor(init[1], device=DEV),
               "beta": torch.tensor(init[2], device=DEV)} for _ in range(R)]
    outs = seqdist.fit(ctxs, seqdist.LocalComm(R), params, cfg, n_total=len(t))
    ps = M.seq_pack(D, torch.tensor(t, device=DEV), torch.tensor(m, dtype=torch.int32, device=DEV), 30.0,
                    chunk_events=32)
    th, al, be = (torch.tensor(x, device=DEV) for x in init)
    r = M.seq_fit(ps, th, al, be, cfg)
    torch.cuda.synchronize()
    for p in params:   # every rank holds the same parameters
        np.testing.assert_allclose(p["alpha"].cpu().numpy(), al.cpu().numpy(), rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(p["beta"].cpu().numpy(), be.cpu().numpy(), rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(p["theta"].cpu().numpy(), th.cpu().numpy(), rtol=1e-4, atol=1e-6)
    assert int(outs[0]["iters"][0]) == int(r["iters"][0]) == 20
    assert float(outs[0]["lnl"][0]) == pytest.approx(float(r["lnl"][0]), rel=1e-6)


def _fit_once(D, t, m, T, R, cfg, comm, graph, init):
    ctxs = _slices(D, t, m, T, R, cfg=cfg)
    params = [{"theta": torch.tensor(init[0], device=DEV), "alpha": torch.tensor(init[1], device=DEV),
               "beta": torch.tensor(init[2], device=DEV)} for _ in range(R)]
    outs = seqdist.fit(ctxs, comm, params, cfg, n_total=len(t), graph=graph)
    torch.cuda.synchronize()
    return params, outs


def test_dist_fit_graph_replay_equals_eager():
    """The distributed fit replayed as one captured CUDA graph per iteration (kernels and the two
    exchanges) gives bit-identical parameters, lnL and iteration counts to the eager loop."""
    D, T, R = 4, 30.0, 3
    t, m, _ = seq_case(D, T, 30.0, seed=41)
    cfg = M.FitConfig(max_iters=25, optimizer="adam", lr=0.05, tol_rel=0.0)
    init = (np.full(D, 2.0, np.float32), np.full((D, D), 0.5, np.float32), np.full((D, D), 2.0, np.float32))
    pe, oe = _fit_once(D, t, m, T, R, cfg, seqdist.LocalComm(R), False, init)
    pg, og = _fit_once(D, t, m, T, R, cfg, seqdist.LocalComm(R), True, init)
    for a, b in zip(pe, pg):
        for k in ("theta", "alpha", "beta"):
            np.testing.assert_array_equal(a[k].cpu().numpy(), b[k].cpu().numpy())
    assert float(oe[0]["lnl"][0]) == float(og[0]["lnl"][0])
    assert int(oe[0]["iters"][0]) == int(og[0]["iters"][0]) == 25


def test_dist_fit_nccl_single_rank_graph():
    """TorchComm over a real NCCL process group (world size 1 on this GPU): the collectives are
    captured in the iteration graph; the result equals the single-GPU sequence fit."""
    import os
    import socket
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        D, T = 3, 30.0
        t, m, _ = seq_case(D, T, 30.0, seed=43)
        cfg = M.FitConfig(max_iters=20, optimizer="adam", lr=0.05, tol_rel=0.0)
        init = (np.full(D, 2.0, np.float32), np.full((D, D), 0.5, np.float32), np.full((D, D), 2.0, np.float32))
        comm = seqdist.TorchComm()
        assert comm.graph_safe
        pg, og = _fit_once(D, t, m, T, 1, cfg, comm, None, init)
        ps = M.seq_pack(D, torch.tensor(t, device=DEV), torch.tensor(m, dtype=torch.int32, device=DEV), T,
                        chunk_events=32)
        th, al, be = (torch.tensor(x, device=DEV) for x in init)
        r = M.seq_fit(ps, th, al, be, cfg)
        torch.cuda.synchronize()
        np.testing.assert_allclose(pg[0]["alpha"].cpu().numpy(), al.cpu().numpy(), rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(pg[0]["beta"].cpu().numpy(), be.cpu().numpy(), rtol=1e-4, atol=1e-6)
        assert int(og[0]["iters"][0]) == 20
        assert float(og[0]["lnl"][0]) == pytest.approx(float(r["lnl"][0]), rel=1e-6)
    finally:
        dist.destroy_process_group()
