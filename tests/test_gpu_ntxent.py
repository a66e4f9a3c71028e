"""GPU parity of the NT-Xent (SimCLR) second workload (include/infcl.h infcl_ntxent_*) against
the fp64 oracle (oracle/ntxent.py) on the same seeded bf16 views, at the north-star gates: loss relative
<= 1e-4 (+ 2^-20 max(1, s) at L ~ 0), LSEs max-abs <= 2e-3, gradients normwise relative <= 2e-3."""
import math

import numpy as np
import pytest
import torch

from oracle import ntxent as N
from synth import make_features
from paper_2410_17243_b200 import loss as K

pytestmark = pytest.mark.gpu


def grad_ok(got, want, rtol=2e-3):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert np.linalg.norm(want) > rtol * np.linalg.norm(want)  # zero fails this gate
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err <= rtol, err


def loss_ok(got, ref, s):
    return abs(got - ref) <= 1e-4 * abs(ref) + 2.0 ** -20 * max(1.0, s)


def run(A, B, s, g=1.0):
    Ad, Bd = A.cuda(), B.cuda()
    b = A.shape[0]
    loss, la, lb, pos = K.ntxent_forward(Ad, Bd, b, s)
    dA, dB = K.ntxent_backward(Ad, Bd, b, s, la, lb, pos, torch.tensor(g, device="cuda"))
    torch.cuda.synchronize()
    return loss.item(), la.cpu().numpy(), lb.cpu().numpy(), pos.cpu().numpy(), dA.cpu().numpy(), dB.cpu().numpy()


@pytest.mark.parametrize("b,d", [(64, 32), (300, 128), (1000, 512), (2048, 768), (777, 256), (130, 40)])
@pytest.mark.parametrize("s", [1.0, 14.2857])
def test_ntxent_parity(b, d, s):
    A, B = make_features(b, d, seed=b + d + 1, dist="paired")
    loss, la, lb, pos, dA, dB = run(A, B, s, 0.7)
    ref = N.forward(A, B, s)
    rdA, rdB = N.backward(A, B, s, 0.7)
    assert loss_ok(loss, ref["loss"], s), (loss, ref["loss"])
    assert np.abs(la - ref["r_a"]).max() <= 2e-3 and np.abs(lb - ref["r_b"]).max() <= 2e-3
    assert np.abs(pos - ref["pos"]).max() <= 2e-3
    grad_ok(dA, rdA)
    grad_ok(dB, rdB)


@pytest.mark.parametrize("s", [0.0, 100.0])
def test_ntxent_scales(s):
    A, B = make_features(1024, 256, seed=7, dist="paired")
    loss, la, lb, pos, dA, dB = run(A, B, s)
    ref = N.forward(A, B, s)
    assert loss_ok(loss, ref["loss"], s), (loss, ref["loss"])
    assert np.abs(la - ref["r_a"]).max() <= 2e-3 and np.abs(lb - ref["r_b"]).max() <= 2e-3
    rdA, rdB = N.backward(A, B, s)
    if s == 0.0:  # uniform softmax: dZ_k = (s g / 2b) ... = 0 at s = 0
        assert np.abs(dA).max() == 0.0 and np.abs(dB).max() == 0.0
    else:
        # s = 100 with paired views: every negative is ~e^-50 below its positive, the exact gradient is ~1e-24,
        # below the fp32 resolution of the LSEs it is evaluated from (one ulp of r ~ 70 moves P_kk - 1 by ~1e-5):
        # the same absolute gate as the CLIP tests' zero-gradient cases
        for got, want in ((dA, rdA), (dB, rdB)):
            assert np.linalg.norm(want) <= 1e-9
            assert np.abs(got).max() <= 1e-6 * s


def test_ntxent_identical_views():
    """All 2b views equal: L = log(2b - 1) exactly and zero gradients (oracle pin)."""
    A, _ = make_features(512, 64, seed=0, dist="identical")
    loss, la, lb, pos, dA, dB = run(A, A.clone(), 14.2857)
    assert abs(loss - math.log(2 * 512 - 1)) <= 1e-4 * math.log(1023)
    assert np.abs(dA).max() <= 1e-6 * 14.2857 and np.abs(dB).max() <= 1e-6 * 14.2857


@pytest.mark.parametrize("s", [1.0, 3.0])
def test_ntxent_onehot_closed_form(s):
    b, K_, d = 1024, 32, 64
    A, _ = make_features(b, d, dist="onehot", K=K_)
    cf = N.onehot_closed_form(b, K_, d, s)
    loss, la, lb, pos, dA, dB = run(A, A.clone(), s)
    assert loss_ok(loss, cf["loss"], s)
    assert np.abs(la - cf["r_a"]).max() <= 2e-3 and np.abs(lb - cf["r_b"]).max() <= 2e-3
    grad_ok(dA, cf["dA"])
    grad_ok(dB, cf["dB"])


def test_ntxent_autograd():
    A, B = make_features(512, 128, seed=4, dist="paired")
    Ad = A.cuda().requires_grad_(True)
    Bd = B.cuda().requires_grad_(True)
    loss = K.ntxent_loss(Ad, Bd, 14.2857)
    (2.0 * loss).backward()
    rdA, rdB = N.backward(A, B, 14.2857, 2.0)
    grad_ok(Ad.grad.float().cpu().numpy(), rdA, 2e-3 + 2.0 ** -8)  # grads returned in bf16
    grad_ok(Bd.grad.float().cpu().numpy(), rdB, 2e-3 + 2.0 ** -8)


def test_ntxent_errors():
    from paper_2410_17243_b200._lib import InfclError
    A, B = make_features(64, 32, seed=1, dtype=torch.float32)
    with pytest.raises(InfclError):  # bf16 views only
        K.ntxent_forward(A.cuda(), B.cuda(), 64, 1.0)


def test_ntxent_cfg2_views_sampled_protocol():
    """cfg2's 65536 views (b = 32768 examples, d = 512) by the large-b protocol: exact fp64 LSEs of 256
    stratified views per side (O(b d) each), the loss from the GPU's LSEs and the exact positives, and 256
    exact gradient rows per side (oracle.ntxent.sampled_rows with the exact LSEs at the sampled views)."""
    b, d, s = 32768, 512, 14.2857
    A, B = make_features(b, d, seed=17, dist="paired")
    loss, la, lb, pos, dA, dB = run(A, B, s)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([[0, 1, 127, 128, 255, 256, b - 1, b - 129], rng.integers(0, b, 248)]))
    Z = N.views(A, B)
    s32 = float(np.float32(s))
    ex = {}
    for half, name in ((0, "a"), (1, "b")):
        ks = rows + half * b
        X = s32 * (Z[ks] @ Z.T)
        X[np.arange(len(ks)), ks] = -np.inf
        m = X.max(1)
        ex[name] = m + np.log(np.exp(X - m[:, None]).sum(1))
    assert np.abs(la[rows] - ex["a"]).max() <= 2e-3 and np.abs(lb[rows] - ex["b"]).max() <= 2e-3
    pos_ex = s32 * np.einsum("ij,ij->i", Z[:b], Z[b:])
    assert np.abs(pos - pos_ex).max() <= 2e-3
    L = math.fsum(np.concatenate([la.astype(np.float64) - pos_ex, lb.astype(np.float64) - pos_ex])) / (2 * b)
    assert abs(loss - L) <= 1e-4 * abs(L)
    ra = la.astype(np.float64)
    rb = lb.astype(np.float64)
    ra[rows], rb[rows] = ex["a"], ex["b"]
    wA, wB = N.sampled_rows(A, B, s, ra, rb, rows)
    grad_ok(dA[rows], wA)
    grad_ok(dB[rows], wB)
