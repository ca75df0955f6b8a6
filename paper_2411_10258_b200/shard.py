"""Window sharding across GPUs and the final gather (row a8 of DESIGN.md section 4).

Windows are independent, so there is no collective on the data path: every rank packs and
fits its own shard, and one gather of fixed-size per-window records ends the step.  This module
is the host-side logic: shard ranges (weak: W windows per rank at global offset rank*W;
strong: one global batch cut into contiguous ranges with ~equal event counts, balanced_ranges),
CSR slicing, the record layout, the gather over a torch.distributed process group (NCCL on
GPUs, gloo in the CPU tests; padded to equal shapes for unequal strong ranges) and the
reassembly in global window order on rank 0.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def weak_range(windows_per_rank: int, rank: int):
    """Global window indices [first, first + W) of `rank` under weak scaling."""
    return rank * windows_per_rank, windows_per_rank


def balanced_ranges(events_per_window, world: int):
    """Contiguous window ranges [(lo, hi)] per rank with ~equal event totals: cut the prefix sum
    of the per-window counts at k/world of the total (work is ~ proportional to events)."""
    c = np.asarray(events_per_window, dtype=np.int64)
    W = len(c)
    pre = np.concatenate([[0], np.cumsum(c)])
    tot = pre[-1]
    cuts = [0]
    for k in range(1, world):
        target = tot * k / world
        cuts.append(int(np.searchsorted(pre, target, side="left")))
    cuts.append(W)
    cuts = np.maximum.accumulate(np.minimum(np.asarray(cuts), W))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def slice_csr(t, mark, win_off, T, lo: int, hi: int):
    """Windows [lo, hi) of a CSR batch as a batch of its own: the event range is contiguous, the
    offsets are rebased to 0 (works for numpy arrays and torch tensors on any device)."""
    a, z = int(win_off[lo]), int(win_off[hi])
    off = win_off[lo:hi + 1] - win_off[lo]
    return t[a:z], mark[a:z], off, T[lo:hi]


def record_width(D: int) -> int:
    """fp32 slots per window: theta (D), alpha (D^2), beta (D^2), lnL (fp64 in 2 slots), iters,
    status (int32 bit-cast)."""
    return D + 2 * D * D + 4


def pack_records(theta, alpha, beta, lnl, iters, status, out=None):
    """-> float32 tensor [W, record_width(D)] (lnL, iters, status stored bit-exactly)."""
    W, D = theta.shape
    R = record_width(D)
    rec = out if out is not None else torch.empty(W, R, dtype=torch.float32, device=theta.device)
    rec[:, :D] = theta
    rec[:, D:D + D * D] = alpha.reshape(W, -1)
    rec[:, D + D * D:D + 2 * D * D] = beta.reshape(W, -1)
    rec[:, D + 2 * D * D:D + 2 * D * D + 2] = lnl.to(torch.float64).contiguous().view(torch.float32).view(W, 2)
    rec[:, -2] = iters.to(torch.int32).view(torch.float32)
    rec[:, -1] = status[:W].to(torch.int32).view(torch.float32)
    return rec


def unpack_records(rec, D: int):
    W = rec.shape[0]
    k = D + 2 * D * D
    return {"theta": rec[:, :D], "alpha": rec[:, D:D + D * D].reshape(W, D, D),
            "beta": rec[:, D + D * D:k].reshape(W, D, D),
            "lnl": rec[:, k:k + 2].contiguous().view(torch.float64).reshape(W),
            "iters": rec[:, -2].contiguous().view(torch.int32), "status": rec[:, -1].contiguous().view(torch.int32)}


def gather_ranges(rec, n_max: int, world: int, rank: int, group=None, out=None):
    """Gather per-rank record tensors of DIFFERENT lengths (strong scaling: balanced_ranges) to
    rank 0: every rank sends a tensor padded to n_max rows (collectives need equal shapes).
    Returns the padded list on rank 0, else None."""
    if rec.shape[0] < n_max:
        pad = torch.zeros(n_max - rec.shape[0], rec.shape[1], dtype=rec.dtype, device=rec.device)
        rec = torch.cat([rec, pad])
    return gather_records(rec, world, rank, group=group, out=out)


def reassemble(gathered, ranges, D: int):
    """Rank 0: the gathered (padded) records of every rank -> results in global window order
    (rank r's rows 0..hi_r-lo_r-1 are windows lo_r..hi_r-1)."""
    parts = [g[: hi - lo] for g, (lo, hi) in zip(gathered, ranges)]
    return unpack_records(torch.cat(parts), D)


def gather_step(theta, alpha, beta, lnl, iters, status, rec, ranges, world: int, rank: int,
                gathered=None, group=None):
    """The end of a strong-scaling step (a8): this rank's results (windows ranges[rank]) into its
    record buffer `rec` ([max range length, record_width] preallocated, so every rank sends the
    same shape), one gather to rank 0, and the reassembly in global window order there.
    Returns the global results dict on rank 0 (world 1: this rank's), else None."""
    lo, hi = ranges[rank]
    D = theta.shape[1]
    pack_records(theta, alpha, beta, lnl, iters, status, out=rec[: hi - lo])
    g = gather_records(rec, world, rank, group=group, out=gathered)
    return reassemble(g, ranges, D) if g is not None else None


def gather_records(rec, world: int, rank: int, group=None, out=None):
    """Gather equally-shaped record tensors to rank 0 (returns the list on rank 0, else None)."""
    if world == 1:
        return [rec]
    lst = out if (rank == 0 and out is not None) else ([torch.empty_like(rec) for _ in range(world)]
                                                      if rank == 0 else None)
    dist.gather(rec, lst, dst=0, group=group)
    return lst
