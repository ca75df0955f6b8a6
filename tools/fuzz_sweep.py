"""Extended randomised parity sweep (evidence run, not part of the test suite): N random batches
(D uniform in 1..32, ragged/empty/long windows, ties, events at 0 and T, random parameters) through
mdhp_pack_windows + mdhp_loglik_grad vs the fp64 oracle; prints the number of windows over the
plain 1e-4 relative lnL bar, the worst relative lnL error and the worst gradient error in units
of the R17 tolerance.  usage: python tools/fuzz_sweep.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2411_10258_b200 as M  # noqa: E402
from tests import helpers as H  # noqa: E402
from tests.test_gpu_fuzz import fuzz_params, fuzz_windows, f32  # noqa: E402


def grad_ratio(got, ref, scale, rel=1e-3, gross_rel=1e-4):
    tol = rel * np.abs(ref) + gross_rel * scale + 1e-30
    return float(np.max(np.abs(np.asarray(got, float) - ref) / tol))


def main(n):
    worst_lnl, worst_g, windows, events, bad = 0.0, 0.0, 0, 0, 0
    for k in range(n):
        rng = np.random.default_rng(50000 + k)
        D = int(rng.integers(1, 33))
        W = int(rng.integers(1, 40))
        b = fuzz_windows(rng, D, W)
        th, al, be = fuzz_params(rng, W, D)
        dev = (torch.tensor(b["t"], dtype=torch.float64, device="cuda"),
               torch.tensor(b["mark"], dtype=torch.int32, device="cuda"),
               torch.tensor(b["win_off"], dtype=torch.int64, device="cuda"),
               torch.tensor(b["T"], dtype=torch.float64, device="cuda"))
        pk = M.pack_windows(D, *dev)
        r = M.loglik_grad(pk, *(torch.tensor(f32(x), device="cuda") for x in (th, al, be)))
        out = {q: v.cpu().numpy() for q, v in r.items() if v is not None}
        t32, T32, _ = H.oracle_times(b, D)
        for w in range(W):
            a, z = b["win_off"][w], b["win_off"][w + 1]
            p = (f32(th[w]).astype(float), f32(al[w]).astype(float), f32(be[w]).astype(float))
            ref = oracle.loglik_rec(D, t32[a:z], b["mark"][a:z], T32[w], *p)
            e = abs(out["lnl"][w] - ref["lnl"]) / max(abs(ref["lnl"]), 1e-300)
            if e > 1e-4:
                bad += 1
                print(f"  lnL out of bar: batch {k} D={D} window {w} n={z - a} T={T32[w]} "
                      f"gpu={out['lnl'][w]!r} oracle={ref['lnl']!r} rel={e:.3g} "
                      f"sum|ln lambda| scale: N={z - a}", flush=True)
            worst_lnl = max(worst_lnl, e)
            sth, sal, sbe = H.grad_scales(t32[a:z], b["mark"][a:z], T32[w], *p, ref)
            worst_g = max(worst_g, grad_ratio(out["g_theta"][w], ref["g_theta"], sth),
                          grad_ratio(out["g_alpha"][w], ref["g_alpha"], sal),
                          grad_ratio(out["g_beta"][w], ref["g_beta"], sbe))
            windows += 1
            events += z - a
    print(f"{n} batches, {windows} windows, {events} events: {bad} windows over the plain lnL bar, "
          f"worst lnL rel err {worst_lnl:.3g} (bar 1e-4), "
          f"worst gradient error {worst_g:.3g} x the R17 tolerance (bar 1)")
    return 0 if worst_lnl <= 1e-4 and worst_g <= 1.0 else 1




def fit_sweep(n, iters=5, latency=False):
    """Random-start Adam fits (lr 0.02, `iters` iterations) vs the oracle's: parameters within
    R17 (1e-3 relative, floor 1e-2 of the group mean); prints the worst ratio to that bar.
    latency: mdhp_fit latency mode (one window per warp in time chunks; D <= 8 only)."""
    worst, windows = 0.0, 0
    for k in range(n):
        rng = np.random.default_rng(70000 + k)
        D = int(rng.integers(1, 33))
        if latency:
            D = 1 + (D - 1) % 8
        W = int(rng.integers(1, 16))
        b = fuzz_windows(rng, D, W)
        th, al, be = fuzz_params(rng, W, D)
        be = np.clip(be, 0.05, None)
        dev = (torch.tensor(b["t"], dtype=torch.float64, device="cuda"),
               torch.tensor(b["mark"], dtype=torch.int32, device="cuda"),
               torch.tensor(b["win_off"], dtype=torch.int64, device="cuda"),
               torch.tensor(b["T"], dtype=torch.float64, device="cuda"))
        pk = M.pack_windows(D, *dev)
        tt = [torch.tensor(f32(x), device="cuda") for x in (th, al, be)]
        M.fit(pk, *tt, M.FitConfig(max_iters=iters, optimizer="adam", lr=0.02, tol_rel=0.0, latency_mode=latency))
        g = [x.cpu().numpy() for x in tt]
        t32, T32, _ = H.oracle_times(b, D)
        ocfg = oracle.FitConfig(max_iters=iters, optimizer="adam", lr=0.02, tol_rel=0.0)
        for w in range(W):
            a, z = b["win_off"][w], b["win_off"][w + 1]
            o = oracle.fit(D, t32[a:z], b["mark"][a:z], T32[w], f32(th[w]).astype(float),
                           f32(al[w]).astype(float), f32(be[w]).astype(float), ocfg)
            for got, key in zip(g, ("theta", "alpha", "beta")):
                ref = o[key]
                s = 1e-2 * max(np.mean(np.abs(ref)), 1e-4)
                r = float(np.max(np.abs(got[w] - ref) / (1e-3 * np.maximum(np.abs(ref), s))))
                if r > 1:
                    print(f"  fit out of bar: batch {k} D={D} window {w} n={z - a} {key} ratio {r:.3g}", flush=True)
                worst = max(worst, r)
            windows += 1
    print(f"fit sweep{' (latency mode)' if latency else ''}: {n} batches, {windows} windows, {iters} Adam iterations: worst parameter error "
          f"{worst:.3g} x the R17 tolerance (bar 1)")
    return 0 if worst <= 1 else 1


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] in ("fit", "fit-latency"):
        sys.exit(fit_sweep(int(sys.argv[2]) if len(sys.argv) > 2 else 200, latency=sys.argv[1] == "fit-latency"))
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 300))
