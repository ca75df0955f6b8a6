"""Row f4: the MDHP-LSTM Hawkes gate hks = tanh(A alpha - B (beta T) + C theta)
(Eq.(7) third line) on the tcgen05 tensor-core kernel vs the fp64 oracle.

Tolerance (R22): both operands enter the tensor core as TF32 (10 explicit mantissa
bits).  The TMA path hands it raw fp32 (the hardware keeps the top 19 bits: |rel err| < 2^-10
per operand), the register-staged path rounds to nearest first (2^-11); so each product carries
< 2^-9 + 2^-20 relative error, fp32 accumulation over K <= 2080 terms (plus the acc0 - T acc1
combine) adds <= (K + 2) 2^-24 of the gross sum, and tanh' <= 1:
|hks_gpu - hks_ref| <= (2^-9 + 2^-20 + 2082 * 2^-24) * gross + 1e-6 ~ 2.1e-3 * gross + 1e-6,
gross = sum_k |W_hk X_wk| (computed by the oracle)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2411_10258_b200 import hawkes_features

pytestmark = pytest.mark.gpu

TOL_G = 2.0 ** -9 + 2.0 ** -20 + 2082 * 2.0 ** -24


def _inputs(D, W, H, seed, wscale=None):
    """Fitted-parameter-like inputs (alpha in [0, 2], beta log-uniform in [1, 60], theta
    log-uniform in [0.05, 50], T in [0.5, 2]) and weights N(0, s^2) with s = 1/sqrt(K) so the
    pre-activation is O(1) (f4 recipe)."""
    rng = np.random.default_rng(seed)
    al = rng.uniform(0, 2, (W, D, D)).astype(np.float32)
    be = np.exp(rng.uniform(np.log(1), np.log(60), (W, D, D))).astype(np.float32)
    th = np.exp(rng.uniform(np.log(0.05), np.log(50), (W, D))).astype(np.float32)
    T = rng.uniform(0.5, 2.0, W).astype(np.float32)
    K = 2 * D * D + D
    s = wscale if wscale is not None else 1.0 / np.sqrt(K) / 10.0
    A = rng.normal(0, s, (H, D * D)).astype(np.float32)
    B = rng.normal(0, s, (H, D * D)).astype(np.float32)
    C = rng.normal(0, s, (H, D)).astype(np.float32)
    return th, al, be, T, A, B, C


def _run(th, al, be, T, A, B, C):
    dev = "cuda"
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    out = hawkes_features(t(th), t(al), t(be), t(T), t(A), t(B), t(C))
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _check(D, W, H, seed, rows=None, wscale=None):
    th, al, be, T, A, B, C = _inputs(D, W, H, seed, wscale)
    got = _run(th, al, be, T, A, B, C)
    idx = np.arange(W) if rows is None else rows
    ref, gross = oracle.hawkes_features(D, th[idx], al[idx], be[idx], T[idx], A, B, C, gross=True)
    err = np.abs(got[idx] - ref)
    bound = TOL_G * gross + 1e-6
    assert np.all(err <= bound), (D, W, H, float((err / bound).max()))
    return got, ref


@pytest.mark.parametrize("D", [1, 2, 3, 5, 8, 16, 32])
def test_features_vs_oracle_all_D(D):
    # 129 windows: one full 128-row tile + a ragged tail of 1
    _check(D, 129, 32, seed=D)


@pytest.mark.parametrize("H", [16, 48, 128, 256, 512])
def test_features_hidden_sizes(H):
    _check(16, 300, H, seed=100 + H)


@pytest.mark.parametrize("W", [1, 127, 128, 257, 1000])
def test_features_ragged_windows(W):
    _check(8, W, 64, seed=200 + W)


def test_features_saturation_and_sign():
    """Large weights: tanh saturates to +-1; the sign of every entry must match the oracle."""
    got, ref = _check(4, 200, 32, seed=7, wscale=1.0)
    sat = np.abs(ref) > 0.999
    assert sat.any() and np.all(np.sign(got[sat]) == np.sign(ref[sat]))


def test_features_selector_weights_exact_tf32():
    """Unit-vector weights pick single parameters: hks = tanh(tf32(x)) up to tanhf's error
    (|tf32(x) - x| < 2^-10 |x| under truncation)."""
    D, W = 4, 130
    th, al, be, T, _, _, _ = _inputs(D, W, 16, seed=9)
    K = 2 * D * D + D
    H = 48   # first 36 columns select X entries, the rest zero
    Wt = np.zeros((H, K), np.float32)
    Wt[np.arange(K), np.arange(K)] = 1.0
    got = _run(th, al, be, T, Wt[:, :D * D].copy(), Wt[:, D * D:2 * D * D].copy(), Wt[:, 2 * D * D:].copy())
    ref = oracle.hawkes_features(D, th, al, be, T, Wt[:, :D * D], Wt[:, D * D:2 * D * D], Wt[:, 2 * D * D:])
    X = np.concatenate([al.reshape(W, -1), -be.reshape(W, -1) * T[:, None], th], axis=1).astype(np.float64)
    assert np.all(np.abs(got - ref) <= 2.0 ** -10 * np.abs(np.concatenate([X, np.zeros((W, H - K))], 1)) + 1e-6)
    assert np.all(got[:, K:] == 0.0)


def test_features_empty_batch():
    th, al, be, T, A, B, C = _inputs(4, 1, 16, seed=1)
    out = hawkes_features(*(torch.from_numpy(x[:0] if i < 4 else x).cuda()
                            for i, x in enumerate((th, al, be, T, A, B, C))))
    assert out.shape == (0, 16)


def test_features_full_size_sampled():
    """cfg5 size: 1,048,576 windows, D = 16, H = 128; 2,000 sampled windows vs the oracle."""
    D, W, H = 16, 1 << 20, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    al = torch.rand(W, D, D, device="cuda", generator=g) * 2
    be = torch.exp(torch.rand(W, D, D, device="cuda", generator=g) * np.log(60))
    th = torch.exp(torch.log(torch.tensor(0.05)) + torch.rand(W, D, device="cuda", generator=g) * np.log(1000))
    T = 0.5 + 1.5 * torch.rand(W, device="cuda", generator=g)
    s = 1.0 / np.sqrt(2 * D * D + D) / 10.0
    A = torch.randn(H, D * D, device="cuda", generator=g) * s
    B = torch.randn(H, D * D, device="cuda", generator=g) * s
    C = torch.randn(H, D, device="cuda", generator=g) * s
    out = hawkes_features(th, al, be, T, A, B, C)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(0).choice(W, 2000, replace=False))
    ri = torch.from_numpy(rows).cuda()
    c = lambda x: x.cpu().numpy()
    ref, gross = oracle.hawkes_features(D, c(th[ri]), c(al[ri]), c(be[ri]), c(T[ri]), c(A), c(B), c(C), gross=True)
    err = np.abs(out[ri].cpu().numpy() - ref)
    assert np.all(err <= TOL_G * gross + 1e-6), float((err / (TOL_G * gross + 1e-6)).max())
    assert torch.isfinite(out).all()


@pytest.mark.parametrize("D", [4, 16])
def test_features_register_path_matches_oracle(D, monkeypatch):
    """The register-staged kernel (used when TMA cannot address the arrays, e.g. D % 4 != 0)
    forced for D % 4 == 0 too."""
    monkeypatch.setenv("MDHP_FEAT_NO_TMA", "1")
    _check(D, 300, 128, seed=300 + D)
    _check(D, 129, 48, seed=301 + D)
