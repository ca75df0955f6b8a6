"""Run-to-run spread of the cfg4 fit (500 iterations): 12 timed fits, CUDA events, printed each.
python tools/perf/seq_variance.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2411_10258_b200 as M  # noqa: E402
from synth import gen, gpu as sgpu  # noqa: E402

rc = gen.CONFIGS["cfg4"]
b = sgpu.make_batch_gpu(rc, 1, seed=2024, first_window=0, device="cuda")
N = int(b["win_off"][-1])
ce = M.seq_chunk_hint(rc.D, N)
ps = M.seq_pack(rc.D, b["t"], b["mark"], rc.T, chunk_events=ce)
th0, al0, be0 = b["theta"][0].clone(), b["alpha"][0].clone(), b["beta"][0].clone()
cfg = M.FitConfig(max_iters=500, optimizer="adam", lr=0.05, tol_rel=0.0)
out = []
for k in range(12):
    th, al, be = th0.clone(), al0.clone(), be0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    M.seq_fit(ps, th, al, be, cfg)
    e1.record()
    torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1))
print("chunk", ce, "fit ms:", " ".join(f"{x:.1f}" for x in out))
