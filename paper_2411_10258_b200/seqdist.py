"""One long sequence over several GPUs (include/mdhp.h "f1").

Rank r owns a contiguous slice of the events (cut between tie groups, ~equal counts).  Each
evaluation exchanges the slices' composite affine maps of the decayed-sum state (all_gather,
2 D^2 + 1 floats per rank), lets every rank compose the state carried into its slice, evaluates
its chunks, and all-reduces the fp64 partial sums (2 D^2 + D + 1) before an identical epilogue /
optimizer step on every rank.  The collectives go through a small Comm interface:

* TorchComm  torch.distributed (NCCL over NVLink on GPUs; one slice per process)
* LocalComm  R emulated ranks in one process (tests on one GPU; every kernel runs to completion
             before the exchange, no kernel waits on another)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import mdhp
from .mdhp import FitConfig, SeqDesc, _check, _ptr, _stream, lib


def slice_bounds(t: np.ndarray, R: int):
    """Contiguous [lo, hi) index ranges, ~equal counts, never splitting equal times."""
    N = len(t)
    cuts = [0]
    for r in range(1, R):
        b = max(cuts[-1], (N * r) // R)
        while 0 < b < N and t[b] == t[b - 1]:
            b += 1
        cuts.append(b)
    cuts.append(N)
    return [(cuts[r], cuts[r + 1]) for r in range(R)]


@dataclass
class SliceCtx:
    rank: int
    ps: mdhp.PackedSeq
    work: torch.Tensor
    D: int


def make_slice(D, t_slice, m_slice, T, t0, rank, chunk_events=256, cfg: FitConfig | None = None, stream=None):
    ps = mdhp.seq_pack(D, t_slice, m_slice, T, chunk_events=chunk_events, t0=t0, has_history=rank > 0,
                       stream=stream)
    nb = int(lib().mdhp_seq_work_bytes(ctypes.byref(ps.desc)))
    work = torch.empty(nb, dtype=torch.uint8, device=t_slice.device)
    c = cfg.c() if cfg is not None else None
    _check(lib().mdhp_seq_work_init(ctypes.byref(ps.desc), _ptr(work), ctypes.byref(c) if c else None,
                                    _stream(stream)), "mdhp_seq_work_init")
    return SliceCtx(rank, ps, work, D)


class LocalComm:
    """All R ranks live in this process: collectives are stacks and sums of the per-rank lists."""

    graph_safe = True

    def __init__(self, R):
        self.R = R

    def all_gather(self, xs):
        if len(xs) == 1:            # one emulated rank: a view, no copy kernel
            return xs[0].unsqueeze(0)
        return torch.stack(xs)

    def all_reduce_sum(self, xs):
        if len(xs) == 1:
            return xs[0]
        return torch.stack(xs).sum(0)


class TorchComm:
    """One slice per process; torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.R = dist.get_world_size(group)
        # NCCL collectives can be captured in CUDA graphs; gloo ones cannot
        self.graph_safe = dist.get_backend(group) == "nccl"

    def all_gather(self, xs):
        (x,) = xs
        out = torch.empty(self.R * x.numel(), dtype=x.dtype, device=x.device)   # flat: NCCL and gloo
        self.dist.all_gather_into_tensor(out, x.contiguous().reshape(-1), group=self.group)
        return out.view((self.R,) + tuple(x.shape))

    def all_reduce_sum(self, xs):
        """In place: the callers pass freshly written temporaries."""
        (x,) = xs
        self.dist.all_reduce(x, group=self.group)
        return x


def _stats(ctxs, comm, stream=None):
    D = ctxs[0].D
    Dp = 1 << (D - 1).bit_length()
    S = 2 * Dp + 17 * Dp + 1
    loc = []
    for c in ctxs:
        st = torch.empty(S, dtype=torch.float64, device=c.work.device)
        _check(lib().mdhp_seq_stats(ctypes.byref(c.ps.desc), _ptr(c.ps.buf), _ptr(st), _stream(stream)), "mdhp_seq_stats")
        loc.append(st)
    g = comm.all_gather(loc).contiguous()
    comb = torch.empty(S, dtype=torch.float64, device=g.device)
    _check(lib().mdhp_seq_stats_combine(D, g.shape[0], _ptr(g), _ptr(comb), _stream(stream)), "mdhp_seq_stats_combine")
    return comb


def _parts(ctxs, comm, theta, alpha, beta, grad, fit, stream=None):
    """One distributed evaluation: maps -> all_gather -> parts -> all_reduce (two collectives).
    Returns (reduced parts, global final state).  theta/alpha/beta are per-context lists
    (identical).  The final state (the last slice's) rides in the all-reduce: every other rank
    contributes exact zeros, so the sum is that state bit for bit."""
    D = ctxs[0].D
    DD = D * D
    R = comm.R
    bufs = []
    for c, be in zip(ctxs, beta):
        mb = torch.empty(2 * DD + 1, dtype=torch.float32, device=c.work.device)   # [maps | span]
        _check(lib().mdhp_seq_maps(ctypes.byref(c.ps.desc), _ptr(c.ps.buf), _ptr(be), _ptr(c.work), _ptr(mb),
                                   _ptr(mb[2 * DD:]), int(fit), _stream(stream)), "mdhp_seq_maps")
        bufs.append(mb)
    G = comm.all_gather(bufs)                          # [R, 2 D^2 + 1]
    M = G[:, :2 * DD].contiguous()                     # [R][D*D] float2
    Sp = G[:, 2 * DD].contiguous()                     # [R]
    NP = 2 * DD + D + 1
    red = []
    for c, th, al, be in zip(ctxs, theta, alpha, beta):
        pb = torch.empty(NP + 2 * DD, dtype=torch.float64, device=c.work.device)   # [parts | final state]
        fn = torch.empty(DD, 2, dtype=torch.float32, device=c.work.device)
        _check(lib().mdhp_seq_parts(ctypes.byref(c.ps.desc), _ptr(c.ps.buf), _ptr(th), _ptr(al), _ptr(be), _ptr(M),
                                    _ptr(Sp), c.rank, _ptr(c.work), _ptr(pb), _ptr(fn), int(grad), int(fit),
                                    _stream(stream)), "mdhp_seq_parts")
        if c.rank == R - 1:
            pb[NP:].copy_(fn.reshape(-1))
        else:
            pb[NP:].zero_()
        red.append(pb)
    S = comm.all_reduce_sum(red)
    P = S[:NP].contiguous()
    F = S[NP:].to(torch.float32).reshape(DD, 2).contiguous()
    return P, F


def loglik_grad(ctxs, comm, theta, alpha, beta, n_total, grads=True, stream=None):
    """Distributed lnL (+ gradients) of one sequence.  theta/alpha/beta: CUDA tensors (the same
    values on every rank; here one set per local context).  Returns the first local context's
    outputs (every rank computes the same)."""
    th = [theta] * len(ctxs); al = [alpha] * len(ctxs); be = [beta] * len(ctxs)
    stats = _stats(ctxs, comm, stream)
    P, F = _parts(ctxs, comm, th, al, be, grad=int(grads), fit=0, stream=stream)
    c = ctxs[0]
    D = c.D
    dev = c.work.device
    lnl = torch.empty(1, dtype=torch.float64, device=dev)
    gt = torch.empty(D, device=dev) if grads else None
    ga = torch.empty(D, D, device=dev) if grads else None
    gb = torch.empty(D, D, device=dev) if grads else None
    _check(lib().mdhp_seq_finish(ctypes.byref(c.ps.desc), int(n_total), _ptr(stats), _ptr(P), _ptr(F), _ptr(theta),
                                 _ptr(alpha), _ptr(beta), _ptr(lnl), _ptr(gt), _ptr(ga), _ptr(gb), None, _ptr(c.work),
                                 None, None, None, None, 0, _ptr(c.ps.buf), _stream(stream)), "mdhp_seq_finish")
    return {"lnl": lnl, "g_theta": gt, "g_alpha": ga, "g_beta": gb}


def fit(ctxs, comm, params, cfg: FitConfig, n_total, stream=None, graph=None):
    """Distributed fit of one sequence: the DESIGN.md "Fit" loop with one exchange pair per
    iteration.  params: per-local-context dicts of CUDA tensors theta [D], alpha/beta [D,D]
    (updated in place, identical on all ranks).  ctxs must have been made with cfg.
    graph (default: when the comm is graph-safe and no explicit stream is given): replay one
    captured iteration (kernels + collectives) as a CUDA graph."""
    stats = _stats(ctxs, comm, stream)
    c = cfg.c()
    outs = []
    dev = ctxs[0].work.device
    for x in ctxs:
        outs.append({"lnl": torch.empty(1, dtype=torch.float64, device=dev),
                     "iters": torch.zeros(1, dtype=torch.int32, device=dev),
                     "status": torch.zeros(1, dtype=torch.int32, device=dev)})
    th = [p["theta"] for p in params]; al = [p["alpha"] for p in params]; be = [p["beta"] for p in params]

    def iteration(final):
        P, F = _parts(ctxs, comm, th, al, be, grad=0 if final else 1, fit=0 if final else 1, stream=stream)
        for x, p, o in zip(ctxs, params, outs):
            _check(lib().mdhp_seq_finish(ctypes.byref(x.ps.desc), int(n_total), _ptr(stats), _ptr(P), _ptr(F),
                                         _ptr(p["theta"]), _ptr(p["alpha"]), _ptr(p["beta"]), _ptr(o["lnl"]), None,
                                         None, None, ctypes.byref(c), _ptr(x.work), None, None, _ptr(o["status"]),
                                         _ptr(o["iters"]), int(final), _ptr(x.ps.buf), _stream(stream)),
                   "mdhp_seq_finish")

    if graph is None:
        graph = stream is None and getattr(comm, "graph_safe", False)
    if graph and cfg.max_iters > 1:
        # iteration 0 runs eagerly (it also initialises the communicator), the rest replay one
        # captured iteration: kernels and collectives, no host round trip; the device-side control
        # block stops the updates once the loop is done (as in mdhp_seq_fit)
        iteration(False)
        # capture_begin/end directly: the torch.cuda.graph context manager also runs gc.collect()
        # and empties the allocator cache on entry (tens of ms, and every later allocation pays
        # cudaMalloc again), which made a fit's wall time vary 4x from call to call
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            g.capture_begin()
            try:
                iteration(False)
            finally:
                g.capture_end()
        torch.cuda.current_stream(dev).wait_stream(side)
        for _ in range(cfg.max_iters - 1):
            g.replay()
        iteration(True)
    else:
        for it in range(cfg.max_iters + 1):
            iteration(it == cfg.max_iters)
    return outs
