"""Strong scaling (bench.py default at N > 1): one batch cut into balanced window
ranges, each range packed and fitted on its own, must give the N = 1 results bit for bit -- a
window's fit never depends on which other windows share its launch.  The cfg2 8192-window
cases also pin the two k_fit<8> builds against each other: the full batch (2,048 warp units)
runs the 16-warps/SM kernel, its ranges (<= 1,184 units) the one-wave LAT kernel (fit.cu) with
the static sub-partition-aware unit order (<= 7 units per SM); cfg2 4500 (1,125 units) runs the
LAT kernel with the dynamic order, its ranges the static one."""
import numpy as np
import pytest
import torch

import paper_2411_10258_b200 as M
from paper_2411_10258_b200 import shard
from synth import gpu as sg

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _fit(D, t, m, off, T, cfg):
    W = T.numel()
    pk = M.pack_windows(D, t.contiguous(), m.contiguous(), off.contiguous(), T.contiguous(), time_mode=1)
    th = torch.full((W, D), 0.1, device=DEV); al = torch.full((W, D, D), 0.5, device=DEV)
    be = torch.full((W, D, D), 1.0, device=DEV)
    r = M.fit(pk, th, al, be, cfg)
    return th, al, be, r["lnl"], r["iters"], r["status"][:W].clone()


@pytest.mark.parametrize("cfg_name,W,tol", [("cfg5", 8192, 0.0), ("cfg2", 4096, 0.0), ("cfg5", 4096, 1e-4),
                                              ("cfg2", 8192, 0.0), ("cfg2", 8192, 1e-4), ("cfg2", 4500, 0.0)])
def test_ranges_concat_equal_single_gpu(cfg_name, W, tol):
    b = sg.make_batch_gpu(cfg_name, W, seed=2024)
    D = b["D"]
    cfg = M.FitConfig(max_iters=30, optimizer="adam", lr=0.05, tol_rel=tol, patience=3)
    ref = shard.pack_records(*_fit(D, b["t"], b["mark"], b["win_off"], b["T"], cfg))
    counts = (b["win_off"][1:] - b["win_off"][:-1]).cpu().numpy()
    for world in (2, 4, 8):
        ranges = shard.balanced_ranges(counts, world)
        n_max = max(z - a for a, z in ranges)
        recs = []
        for lo, hi in ranges:
            rec = torch.zeros(n_max, shard.record_width(D), device=DEV)
            res = _fit(D, *shard.slice_csr(b["t"], b["mark"], b["win_off"], b["T"], lo, hi), cfg)
            shard.pack_records(*res, out=rec[: hi - lo])
            recs.append(rec)
        got = torch.cat([r[: hi - lo] for r, (lo, hi) in zip(recs, ranges)])
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int32), ref.view(torch.int32)), (cfg_name, world)
        loads = [int(counts[lo:hi].sum()) for lo, hi in ranges]
        assert max(loads) - min(loads) <= 2 * int(counts.max())
