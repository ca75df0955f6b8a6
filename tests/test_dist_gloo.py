"""Multi-process (world size 2, gloo, CPU) coverage of the sharding/gather host logic (row a8).
The data path itself has no collective; this checks what crosses processes."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_10258_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_results(rank, W, D):
    g = torch.Generator().manual_seed(100 + rank)
    th = torch.rand(W, D, generator=g)
    al = torch.rand(W, D, D, generator=g)
    be = torch.rand(W, D, D, generator=g)
    lnl = torch.randn(W, generator=g, dtype=torch.float64) * 1e4
    it = torch.arange(W, dtype=torch.int32) + 7 * rank
    st = torch.full((W,), 256 * rank + 1, dtype=torch.int32)
    return th, al, be, lnl, it, st


def _worker(rank, world, port, W, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, n = shard.weak_range(W, rank)
    rec = shard.pack_records(*_fake_results(rank, W, D))
    got = shard.gather_records(rec, world, rank)
    if rank == 0:
        ok = True
        for r in range(world):
            u = shard.unpack_records(got[r], D)
            ref = _fake_results(r, W, D)
            ok &= torch.equal(u["theta"], ref[0]) and torch.equal(u["alpha"], ref[1])
            ok &= torch.equal(u["beta"], ref[2]) and torch.equal(u["lnl"], ref[3])
            ok &= torch.equal(u["iters"], ref[4]) and torch.equal(u["status"], ref[5])
        q.put(("ok" if ok else "mismatch", first, n))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    W, D = 37, 5
    ps = [ctx.Process(target=_worker, args=(r, 2, port, W, D, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    status, first, n = q.get(timeout=5)
    assert status == "ok" and first == 0 and n == W


def test_records_roundtrip_bit_exact():
    th, al, be, lnl, it, st = _fake_results(3, 11, 4)
    u = shard.unpack_records(shard.pack_records(th, al, be, lnl, it, st), 4)
    assert torch.equal(u["lnl"], lnl) and torch.equal(u["status"], st) and torch.equal(u["beta"], be)


def test_balanced_ranges():
    rng = np.random.default_rng(0)
    c = rng.poisson(1000, 10000)
    for world in (1, 2, 4, 8):
        rr = shard.balanced_ranges(c, world)
        assert rr[0][0] == 0 and rr[-1][1] == len(c)
        assert all(rr[k][1] == rr[k + 1][0] for k in range(world - 1))
        loads = [c[a:b].sum() for a, b in rr]
        assert max(loads) - min(loads) <= 2 * c.max()
    assert shard.balanced_ranges([5, 0, 0], 4)[-1] == (3, 3) or shard.balanced_ranges([5, 0, 0], 4)[-1][1] == 3


def _comm_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_10258_b200 import seqdist
    c = seqdist.TorchComm()
    g = c.all_gather([torch.full((3, 2), float(rank))])
    s = c.all_reduce_sum([torch.arange(4, dtype=torch.float64) * (rank + 1)])
    if rank == 0:
        ok = g.shape == (world, 3, 2) and all(torch.all(g[r] == r) for r in range(world))
        ok = ok and torch.equal(s, torch.arange(4, dtype=torch.float64) * sum(r + 1 for r in range(world)))
        q.put("ok" if ok else "bad")
    dist.barrier()
    dist.destroy_process_group()


def test_seqdist_torchcomm_gloo():
    """The f1 exchange wrapper (all_gather of maps, all_reduce of partial sums) over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_comm_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) == "ok"


def test_slice_bounds_never_split_ties():
    from paper_2411_10258_b200 import seqdist
    t = np.array([0.0, 1.0, 1.0, 1.0, 2.0, 3.0, 3.0, 4.0, 5.0, 6.0])
    for R in (1, 2, 3, 4, 7, 12):
        b = seqdist.slice_bounds(t, R)
        assert b[0][0] == 0 and b[-1][1] == len(t) and all(b[k][1] == b[k + 1][0] for k in range(R - 1))
        for lo, hi in b:
            assert lo == 0 or lo == len(t) or t[lo] != t[lo - 1]


def _fake_fit(t, mark, win_off, T, D):
    """A deterministic per-window stand-in for pack + fit (CPU): results depend only on the
    window's own events, so any split of the batch must reassemble to the unsplit results."""
    W = len(T)
    th = torch.zeros(W, D); al = torch.zeros(W, D, D); be = torch.zeros(W, D, D)
    lnl = torch.zeros(W, dtype=torch.float64)
    for w in range(W):
        a, z = int(win_off[w]), int(win_off[w + 1])
        cnt = torch.bincount(mark[a:z].long(), minlength=D).float()
        th[w] = cnt / float(T[w])
        al[w] = torch.outer(cnt, cnt) / (1.0 + (z - a) % 7)
        be[w] = float(t[a:z].sum()) + torch.arange(D * D, dtype=torch.float32).view(D, D)
        lnl[w] = float(t[a:z].double().sum()) - 1e-3 * (z - a)
    it = (win_off[1:] - win_off[:-1]).to(torch.int32)
    st = torch.where(it == 0, 1, 0).to(torch.int32)
    return th, al, be, lnl, it, st


def _strong_batch(W=53, D=4, seed=3):
    g = torch.Generator().manual_seed(seed)
    n = torch.randint(0, 30, (W,), generator=g)
    off = torch.zeros(W + 1, dtype=torch.int64)
    off[1:] = torch.cumsum(n, 0)
    E = int(off[-1])
    t = torch.rand(E, generator=g, dtype=torch.float64)
    mark = torch.randint(0, D, (E,), generator=g, dtype=torch.int32)
    T = torch.ones(W, dtype=torch.float64)
    return t, mark, off, T


def _strong_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = 4
    t, mark, off, T = _strong_batch(D=D)
    ranges = shard.balanced_ranges((off[1:] - off[:-1]).numpy(), world)
    lo, hi = ranges[rank]
    res = _fake_fit(*shard.slice_csr(t, mark, off, T, lo, hi), D)
    n_max = max(z - a for a, z in ranges)
    rec = torch.zeros(n_max, shard.record_width(D))
    out = shard.gather_step(*res, rec, ranges, world, rank)
    if rank == 0:
        ref = _fake_fit(t, mark, off, T, D)
        ok = all(torch.equal(out[k], v) for k, v in zip(("theta", "alpha", "beta", "lnl", "iters", "status"), ref))
        q.put(("ok" if ok else "mismatch", ranges))
    dist.barrier()
    dist.destroy_process_group()


def test_strong_step_world2_gloo():
    """The strong-scaling step logic of bench.py on CPU, world size 2: balanced ranges of ONE
    batch -> CSR slices -> per-rank (stand-in) fits -> padded records -> gather -> reassembly in
    global window order on rank 0 == the unsplit batch's results bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_strong_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    status, ranges = q.get(timeout=5)
    assert status == "ok" and ranges[0][0] == 0 and ranges[-1][1] == 53 and ranges[0][1] == ranges[1][0]


def test_slice_csr_and_reassemble_single_process():
    D = 3
    t, mark, off, T = _strong_batch(W=40, D=D, seed=9)
    ref = _fake_fit(t, mark, off, T, D)
    for world in (1, 3, 5, 8):
        ranges = shard.balanced_ranges((off[1:] - off[:-1]).numpy(), world)
        n_max = max(z - a for a, z in ranges)
        recs = []
        for r, (lo, hi) in enumerate(ranges):
            res = _fake_fit(*shard.slice_csr(t, mark, off, T, lo, hi), D)
            rec = torch.zeros(n_max, shard.record_width(D))
            shard.pack_records(*res, out=rec[: hi - lo])
            recs.append(rec)
        out = shard.reassemble(recs, ranges, D)
        for k, v in zip(("theta", "alpha", "beta", "lnl", "iters", "status"), ref):
            assert torch.equal(out[k], v), (world, k)
