"""A/B check that two builds of libmdhp.so give bit-identical fits (run once per build with
MDHP_LIB set, then compare): python tools/ab_bitexact.py save out.pt [config] [W] [iters]
                              python tools/ab_bitexact.py cmp a.pt b.pt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def save(out, cfg="cfg2", W=4096, iters=20):
    import paper_2411_10258_b200 as M
    from synth import gpu as sg
    b = sg.make_batch_gpu(cfg, W, seed=2024)
    D = b["D"]
    pk = M.pack_windows(D, b["t"], b["mark"], b["win_off"], b["T"], time_mode=1)
    r = M.loglik_grad(pk, b["theta"], b["alpha"], b["beta"])
    th = torch.full((W, D), 0.1, device="cuda"); al = torch.full((W, D, D), 0.5, device="cuda")
    be = torch.full((W, D, D), 1.0, device="cuda")
    f = M.fit(pk, th, al, be, M.FitConfig(max_iters=iters, tol_rel=0.0))
    torch.save({k: v.cpu() for k, v in {**{"l_" + a: b for a, b in r.items()}, "theta": th, "alpha": al, "beta": be,
                                        "lnl": f["lnl"]}.items()}, out)


def cmp(a, b):
    A, B = torch.load(a), torch.load(b)
    bad = [k for k in A if not torch.equal(A[k].view(torch.int32) if A[k].dtype == torch.float32 else A[k],
                                           B[k].view(torch.int32) if B[k].dtype == torch.float32 else B[k])]
    print("bit-identical" if not bad else f"DIFFER: {bad}")
    return 1 if bad else 0


if __name__ == "__main__":
    if sys.argv[1] == "save":
        save(sys.argv[2], *(sys.argv[3:4] or ["cfg2"]), *[int(x) for x in sys.argv[4:6]])
    else:
        sys.exit(cmp(sys.argv[2], sys.argv[3]))
