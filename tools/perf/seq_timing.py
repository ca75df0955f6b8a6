"""Time the cfg4 sequence path pieces (pack, fit at several iteration counts) with CUDA events and
wall clock, to separate fixed per-call cost from per-iteration cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2411_10258_b200 as M  # noqa: E402
from synth import gen, gpu as sgpu  # noqa: E402


def ev_time(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        w1 = time.perf_counter()
        torch.cuda.synchronize()
        w2 = time.perf_counter()
        out.append((e0.elapsed_time(e1), (w1 - w0) * 1e3, (w2 - w0) * 1e3))
    return min(out)


rc = gen.CONFIGS["cfg4"]
b = sgpu.make_batch_gpu(rc, 1, seed=2024, first_window=0, device="cuda")
ce = int(os.environ.get("CHUNK", "256"))
ps = M.seq_pack(rc.D, b["t"], b["mark"], rc.T, chunk_events=ce)
th0, al0, be0 = b["theta"][0].clone(), b["alpha"][0].clone(), b["beta"][0].clone()
print("N", int(b["win_off"][-1]), "chunk", ce)
print("pack  gpu_ms %.3f  enqueue_ms %.3f  total_ms %.3f" % ev_time(
    lambda: M.seq_pack(rc.D, b["t"], b["mark"], rc.T, chunk_events=ce, out=ps)))
for it in (1, 2, 10, 100, 500):
    cfg = M.FitConfig(max_iters=it, optimizer="adam", lr=0.05, tol_rel=0.0)

    def f():
        th, al, be = th0.clone(), al0.clone(), be0.clone()
        M.seq_fit(ps, th, al, be, cfg)
    print("fit iters %4d  gpu_ms %.3f  enqueue_ms %.3f  total_ms %.3f" % ((it,) + ev_time(f)))
th, al, be = th0.clone(), al0.clone(), be0.clone()
print("loglik_grad  gpu_ms %.3f  enqueue_ms %.3f  total_ms %.3f" % ev_time(lambda: M.seq_loglik_grad(ps, th, al, be)))
