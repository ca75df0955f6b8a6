"""Ablation f3: the paper's all-pairs evaluation vs the recurrence, same packed batch, same GPU.
Prints one JSON line per config: event-evaluations/s of mdhp_loglik_dense (lnL only),
mdhp_loglik_grad lnL-only and lnL+gradients.  Usage: python tools/ablation_dense.py [cfg ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_10258_b200 as M  # noqa: E402
from synth import gpu as sg  # noqa: E402

SIZES = {"cfg2": 4096, "cfg3": 65536, "cfg5": 1 << 20}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main(cfgs):
    for cfg in cfgs:
        W = SIZES[cfg]
        b = sg.make_batch_gpu(cfg, W, seed=2024)
        D = b["D"]
        pk = M.pack_windows(D, b["t"], b["mark"], b["win_off"], b["T"], time_mode=1)
        E = int(b["win_off"][-1])
        th, al, be = b["theta"], b["alpha"], b["beta"]
        out = torch.empty(W, dtype=torch.float64, device="cuda")
        td = timed(lambda: M.mdhp.loglik_dense(pk, th, al, be, out=out), reps=1 if cfg == "cfg5" else 3)
        tr = timed(lambda: M.loglik_grad(pk, th, al, be, grads=False))
        tg = timed(lambda: M.loglik_grad(pk, th, al, be, grads=True))
        dl = M.mdhp.loglik_dense(pk, th, al, be)
        rl = M.loglik_grad(pk, th, al, be, grads=False)["lnl"]
        rel = float(((dl - rl).abs() / rl.abs()).max())
        print(json.dumps({"config": cfg, "windows": W, "events": E, "D": D,
                          "dense_lnl_event_evals_per_s": E / td, "recurrence_lnl_event_evals_per_s": E / tr,
                          "recurrence_lnl_grad_event_evals_per_s": E / tg, "speedup_lnl": td / tr,
                          "max_rel_diff_dense_vs_recurrence": rel}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg5"])
