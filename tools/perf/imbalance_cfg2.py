"""How much of the cfg2 fit time is set by its longest windows (one wave of warps: the kernel
ends with the slowest warp).  Times mdhp_fit on the whole cfg2 batch, on the windows at or below
the p-th length percentile, and on the rest.  python tools/perf/imbalance_cfg2.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2411_10258_b200 as M  # noqa: E402
from synth import gpu as sg  # noqa: E402


def subset(b, sel):
    off = b["win_off"].cpu().numpy()
    idx = np.concatenate([np.arange(off[w], off[w + 1]) for w in sel])
    n = off[1:] - off[:-1]
    o2 = np.zeros(len(sel) + 1, np.int64)
    o2[1:] = np.cumsum(n[sel])
    it = torch.from_numpy(idx).cuda()
    return b["t"][it], b["mark"][it], torch.from_numpy(o2).cuda(), b["T"][torch.from_numpy(sel).cuda()]


def timed(D, t, m, off, T, cfg, reps=3):
    W = T.numel()
    pk = M.pack_windows(D, t.contiguous(), m.contiguous(), off.contiguous(), T.contiguous(), time_mode=1)
    best = 1e9
    for _ in range(reps):
        th = torch.full((W, D), 0.1, device="cuda")
        al = torch.full((W, D, D), 0.5, device="cuda")
        be = torch.full((W, D, D), 1.0, device="cuda")
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        M.fit(pk, th, al, be, cfg)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


b = sg.make_batch_gpu("cfg2", 4096, seed=2024)
D = b["D"]
n = (b["win_off"][1:] - b["win_off"][:-1]).cpu().numpy()
cfg = M.FitConfig(max_iters=500, optimizer="adam", lr=0.05, tol_rel=0.0)
allw = np.arange(len(n))
print(f"windows {len(n)} events mean {n.mean():.1f} max {n.max()}")
print(f"all: {timed(D, *subset(b, allw), cfg):.2f} ms")
for p in (50, 90, 99):
    thr = np.percentile(n, p)
    lo, hi = allw[n <= thr], allw[n > thr]
    print(f"p{p} (n <= {thr:.0f}): {len(lo)} windows {timed(D, *subset(b, lo), cfg):.2f} ms, max {n[lo].max()};"
          f" rest {len(hi)} windows {timed(D, *subset(b, hi), cfg):.2f} ms")
