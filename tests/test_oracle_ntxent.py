"""Pins of the NT-Xent oracle (oracle/ntxent.py) against things other than itself: a pure-Python
brute force of the definition (tests/brute.py), central finite differences, closed forms (identical views:
L = log(2b - 1); one-hot classes), swap symmetry, the sampled-row large-b helper, and mutations."""
import math

import numpy as np
import pytest

from oracle import ntxent as N
from tests import brute


def rand(b, d, seed):
    x = np.random.default_rng(seed).standard_normal((b, d))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


@pytest.mark.parametrize("b,d,s,seed", [(1, 4, 1.0, 0), (3, 5, 14.2857, 1), (6, 8, 2.0, 2), (5, 3, 100.0, 3)])
def test_loss_vs_bruteforce(b, d, s, seed):
    A, B = rand(b, d, seed), rand(b, d, seed + 10)
    s32 = float(np.float32(s))
    assert N.forward(A, B, s)["loss"] == pytest.approx(brute.ntxent_loss(A.tolist(), B.tolist(), s32), rel=1e-12,
                                                       abs=1e-13)


@pytest.mark.parametrize("b,d,s,seed", [(2, 3, 1.0, 4), (4, 5, 7.0, 5)])
def test_grads_vs_finite_differences(b, d, s, seed):
    A, B = rand(b, d, seed), rand(b, d, seed + 10)
    s32 = float(np.float32(s))
    dA, dB = N.backward(A, B, s)
    fA, fB = brute.ntxent_fd_grads(A.tolist(), B.tolist(), s32)
    assert np.allclose(dA, fA, rtol=1e-5, atol=1e-8) and np.allclose(dB, fB, rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("b", [1, 2, 7, 64])
def test_identical_views_log_2b_minus_1(b):
    u = rand(1, 16, 9)[0]
    A = np.tile(u, (b, 1))
    f = N.forward(A, A.copy(), 14.2857)
    assert f["loss"] == pytest.approx(math.log(2 * b - 1), abs=1e-12)
    dA, dB = N.backward(A, A.copy(), 14.2857)
    assert np.abs(dA).max() < 1e-12 and np.abs(dB).max() < 1e-12


@pytest.mark.parametrize("s", [1.0, 5.0, 14.2857])
def test_onehot_closed_form_matches_definition(s):
    b, K, d = 24, 4, 6
    A = np.zeros((b, d))
    A[np.arange(b), np.arange(b) % K] = 1.0
    cf = N.onehot_closed_form(b, K, d, s)
    f = N.forward(A, A.copy(), s)
    dA, dB = N.backward(A, A.copy(), s)
    assert f["loss"] == pytest.approx(cf["loss"], rel=1e-13)
    assert np.allclose(f["r_a"], cf["r_a"], atol=1e-13) and np.allclose(f["r_b"], cf["r_b"], atol=1e-13)
    assert np.allclose(dA, cf["dA"], atol=1e-14) and np.allclose(dB, cf["dB"], atol=1e-14)


def test_swap_symmetry_and_sampled_rows():
    b, d, s = 30, 8, 14.2857
    A, B = rand(b, d, 21), rand(b, d, 22)
    f1, f2 = N.forward(A, B, s), N.forward(B, A, s)
    assert f1["loss"] == pytest.approx(f2["loss"], rel=1e-13)
    assert np.allclose(f1["r_a"], f2["r_b"]) and np.allclose(f1["r_b"], f2["r_a"])
    dA, dB = N.backward(A, B, s, 0.7)
    eB, eA = N.backward(B, A, s, 0.7)
    assert np.allclose(dA, eA, atol=1e-15) and np.allclose(dB, eB, atol=1e-15)
    rows = np.array([0, 3, 29])
    sA, sB = N.sampled_rows(A, B, s, f1["r_a"], f1["r_b"], rows, 0.7)
    assert np.allclose(sA, dA[rows], atol=1e-15) and np.allclose(sB, dB[rows], atol=1e-15)


def test_mutations_are_caught():
    """Plausible mistakes (self-similarity not masked; positive at the own index; G not symmetrised) change
    the result by far more than the GPU gates."""
    b, d, s = 8, 6, 5.0
    A, B = rand(b, d, 31), rand(b, d, 32)
    ref = brute.ntxent_loss(A.tolist(), B.tolist(), float(np.float32(s)))
    Z = np.concatenate([A, B])
    X = float(np.float32(s)) * Z @ Z.T
    r_nomask = np.log(np.exp(X).sum(1))
    pos = np.concatenate([np.einsum("ij,ij->i", A, B)] * 2) * float(np.float32(s))
    assert abs(np.mean(r_nomask - pos) - ref) > 1e-2
    dA, _ = N.backward(A, B, s)
    fA, _ = brute.ntxent_fd_grads(A.tolist(), B.tolist(), float(np.float32(s)))
    f = N.forward(A, B, s)
    r = np.concatenate([f["r_a"], f["r_b"]])
    G = np.exp(np.where(np.eye(2 * b, dtype=bool), -np.inf, X) - r[:, None]) / (2 * b)
    G[np.arange(2 * b), (np.arange(2 * b) + b) % (2 * b)] -= 1 / (2 * b)
    wrong = float(np.float32(s)) * (G @ Z)[:b]  # missing G^T
    assert np.abs(wrong - np.asarray(fA)).max() > 1e-3
    assert np.allclose(dA, fA, rtol=1e-5, atol=1e-8)
