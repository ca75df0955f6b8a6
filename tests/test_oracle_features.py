"""Pins of oracle.hawkes_features (Eq.(7) third line) against things
other than its own formula: SPEC's stated examples, selector weights that reduce the gate to
tanh of single parameters (math.tanh), linearity of atanh(hks) in the weights, and an
independent numpy matmul on random inputs."""
import json
import math
import os

import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def test_spec_examples():
    for ex in json.load(open(GOLD))["hawkes_gate"]:
        D, H = ex["D"], ex["H"]
        rng = np.random.default_rng(0)
        if ex.get("zero_weights"):
            A = np.zeros((H, D * D)); B = np.zeros((H, D * D)); C = np.zeros((H, D))
            th, al, be, T = rng.random((1, D)), rng.random((1, D, D)), rng.random((1, D, D)), [1.7]
        else:
            A, B, C = np.array(ex["A"]), np.array(ex["B"]), np.array(ex["C"])
            th = np.array([ex["theta"]]); al = np.array([ex["alpha"]]); be = np.array([ex["beta"]])
            T = [ex["T"]]
        out = oracle.hawkes_features(D, th, al, be, T, A, B, C)
        assert np.all(out == ex["value"]), ex["cite"]


def test_selector_weights_reduce_to_tanh_of_each_parameter():
    """Row h of [A|B|C] = unit vector e_h: hks_h = tanh(alpha_ij), tanh(-beta_ij T), tanh(theta_j)
    with the row-major (i*D + j) flattening.  Asymmetric alpha/beta catch a transposed index,
    distinct T per window a missing or misplaced T_span, the B rows a sign error."""
    D, W = 3, 4
    rng = np.random.default_rng(1)
    al = rng.uniform(0, 2, (W, D, D)); be = rng.uniform(0.1, 3, (W, D, D))
    th = rng.uniform(0.05, 2, (W, D)); T = rng.uniform(0.2, 1.5, W)
    K = 2 * D * D + D
    Wt = np.eye(K)
    A, B, C = Wt[:, :D * D], Wt[:, D * D:2 * D * D], Wt[:, 2 * D * D:]
    out = oracle.hawkes_features(D, th, al, be, T, A, B, C)
    for w in range(W):
        for i in range(D):
            for j in range(D):
                assert out[w, i * D + j] == math.tanh(al[w, i, j])
                assert abs(out[w, D * D + i * D + j] - math.tanh(-be[w, i, j] * T[w])) <= 1e-16
        for j in range(D):
            assert out[w, 2 * D * D + j] == math.tanh(th[w, j])


def test_atanh_is_linear_in_the_weights():
    D, W, H = 4, 5, 6
    rng = np.random.default_rng(2)
    al = rng.uniform(0, 1, (W, D, D)); be = rng.uniform(0.5, 5, (W, D, D))
    th = rng.uniform(0.1, 1, (W, D)); T = rng.uniform(0.5, 2, W)
    s = 0.02
    W1 = [rng.normal(0, s, (H, D * D)), rng.normal(0, s, (H, D * D)), rng.normal(0, s, (H, D))]
    W2 = [rng.normal(0, s, (H, D * D)), rng.normal(0, s, (H, D * D)), rng.normal(0, s, (H, D))]
    z1 = np.arctanh(oracle.hawkes_features(D, th, al, be, T, *W1))
    z2 = np.arctanh(oracle.hawkes_features(D, th, al, be, T, *W2))
    z12 = np.arctanh(oracle.hawkes_features(D, th, al, be, T, *[a + b for a, b in zip(W1, W2)]))
    assert np.allclose(z12, z1 + z2, rtol=1e-12, atol=1e-12)


def test_random_vs_numpy_matmul_and_gross():
    D, W, H = 5, 7, 16
    rng = np.random.default_rng(3)
    al = rng.uniform(0, 1, (W, D, D)); be = rng.uniform(0.5, 5, (W, D, D))
    th = rng.uniform(0.1, 1, (W, D)); T = rng.uniform(0.5, 2, W)
    A, B = rng.normal(0, 0.1, (H, D * D)), rng.normal(0, 0.1, (H, D * D))
    C = rng.normal(0, 0.1, (H, D))
    X = np.concatenate([al.reshape(W, -1), -be.reshape(W, -1) * T[:, None], th], axis=1)
    Wt = np.concatenate([A, B, C], axis=1)
    ref = np.tanh(X @ Wt.T)
    out, gross = oracle.hawkes_features(D, th, al, be, T, A, B, C, gross=True)
    assert np.allclose(out, ref, rtol=1e-13, atol=1e-14)
    assert np.allclose(gross, np.abs(X) @ np.abs(Wt).T, rtol=1e-13)
