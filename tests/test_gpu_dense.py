"""The dense all-pairs ablation kernel computes the same Eq.(5) lnL: checked
against the oracle definition and against the recurrence path on the same packed batch."""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_10258_b200 as M
from paper_2411_10258_b200 import mdhp
from tests import helpers as H

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("D", [1, 3, 8, 16, 32])
def test_dense_vs_oracle_and_recurrence(D):
    b, (th, al, be) = H.small_batch(D, 16, seed=900 + D)
    pk = M.pack_windows(D, torch.tensor(b["t"], device=DEV), torch.tensor(b["mark"], dtype=torch.int32, device=DEV),
                        torch.tensor(b["win_off"], device=DEV), torch.tensor(b["T"], device=DEV))
    f = lambda x: torch.tensor(np.asarray(x, np.float32), device=DEV)
    dense = M.mdhp.loglik_dense(pk, f(th), f(al), f(be)).cpu().numpy()
    rec = M.loglik_grad(pk, f(th), f(al), f(be), grads=False)["lnl"].cpu().numpy()
    t32, T32, st = H.oracle_times(b, D)
    for w in range(len(b["T"])):
        a, z = b["win_off"][w], b["win_off"][w + 1]
        p = [np.asarray(x[w], np.float32).astype(float) for x in (th, al, be)]
        ref = oracle.loglik_def(D, t32[a:z], b["mark"][a:z], T32[w], *p, grads=False)["lnl"]
        assert abs(dense[w] - ref) <= 1e-4 * abs(ref), (w, dense[w], ref)
        assert abs(dense[w] - rec[w]) <= 1e-4 * abs(ref)
