"""Pins of the fp64 oracle against things other than itself (SURVEY.md 8(c) "What pins each part").

Every oracle function is checked against at least one of: the SPEC's worked examples (golden file),
a pure-Python brute force written from Eq.1 (tests/brute.py), closed forms (identical / one-hot /
codebook inputs), central finite differences, exact gradient identities, swap symmetry, and tiling /
ring invariance.  A mutation section checks that plausible mistakes are caught.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import infonce as O
from synth import make_features, codebook_assignment, codebook_vectors
from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def golden():
    out = {}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        name, val, *_ = line.split()
        out[name] = float(val)
    return out


def rand_feats(b, d, seed, dtype=np.float64, unit=True):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, d))
    if unit:
        x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(dtype)


# ------------------------------------------------------------------ SPEC worked examples (golden)
def test_spec_tile_lse_examples():
    g = golden()
    assert O.tile_lse([[0.0, 0.0, 0.0, 0.0]])[0] == pytest.approx(g["tile_lse_row_of_4_zeros"], abs=1e-15)
    assert O.tile_lse([[3.7]])[0] == pytest.approx(g["tile_lse_single_col_3.7"], abs=1e-15)
    v = O.tile_lse([[1000.0, 1000.0]])[0]
    assert math.isfinite(v) and v == pytest.approx(g["tile_lse_1000_1000"], abs=1e-12)


def test_spec_merge_examples():
    g = golden()
    assert O.merge_lse(O.NEG_INF, 2.5) == pytest.approx(g["merge_identity_2.5"], abs=0)
    assert O.merge_lse(math.log(2), math.log(2)) == pytest.approx(g["merge_log2_log2"], abs=1e-15)
    assert O.merge_lse(0.3, 1.9) == pytest.approx(g["merge_0.3_1.9"], abs=1e-15)
    assert O.merge_lse(1.9, 0.3) == pytest.approx(g["merge_0.3_1.9"], abs=1e-15)
    assert O.merge_lse(O.NEG_INF, O.NEG_INF) == O.NEG_INF  # (-inf)-(-inf) guard (Q1)


def test_spec_loss_examples():
    g = golden()
    one = np.array([[0.6, 0.8]])
    assert O.loss_only(one, one, 3.0) == pytest.approx(g["loss_b1"], abs=1e-15)
    eye = np.eye(2)
    f = O.forward(eye, eye, 1.0)
    assert f["loss"] == pytest.approx(g["loss_2x2_identity_s1"], abs=1e-15)
    assert f["loss_i"] == pytest.approx(g["loss_2x2_identity_s1"], abs=1e-15)
    dI, dT = O.backward(one, one, 3.0)
    assert np.abs(dI).max() == 0 and np.abs(dT).max() == 0


def test_uniform_similarity_lse():
    # all similarities equal to s -> every LSE = s + log b
    b = 8
    X = np.full((b, b), 2.5)
    assert np.allclose(O.lse_rows(X), 2.5 + math.log(b), atol=1e-14)
    assert np.allclose(O.lse_cols(X), 2.5 + math.log(b), atol=1e-14)


# ------------------------------------------------------------------ brute force (pure Python, Eq.1)
@pytest.mark.parametrize("b,d,s,seed", [(1, 3, 2.0, 0), (2, 2, 1.0, 1), (3, 4, 14.2857, 2), (5, 3, 0.7, 3),
                                        (8, 6, 100.0, 4), (7, 5, 0.0, 5)])
def test_loss_vs_bruteforce(b, d, s, seed):
    I = rand_feats(b, d, seed)
    T = rand_feats(b, d, seed + 100)
    ref = brute.loss(I.tolist(), T.tolist(), float(np.float32(s)))
    got = O.loss_only(I, T, s)
    assert got == pytest.approx(ref, rel=1e-13, abs=1e-14)


@pytest.mark.parametrize("b,d,s,seed", [(2, 2, 1.0, 10), (4, 3, 5.0, 11), (6, 4, 14.2857, 12), (5, 2, 30.0, 13)])
def test_grads_vs_finite_differences(b, d, s, seed):
    I = rand_feats(b, d, seed)
    T = rand_feats(b, d, seed + 100)
    s32 = float(np.float32(s))
    fdI, fdT = brute.fd_grads(I.tolist(), T.tolist(), s32)
    dI, dT = O.backward(I, T, s)
    fdI = np.array(fdI)
    fdT = np.array(fdT)
    # central differences h=1e-6, 1e-5 relative or 1e-8 absolute
    assert np.allclose(dI, fdI, rtol=1e-5, atol=1e-8)
    assert np.allclose(dT, fdT, rtol=1e-5, atol=1e-8)


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("b,d", [(1, 4), (8, 16), (64, 32), (333, 8)])
def test_identical_features_log_b(b, d):
    u = rand_feats(1, d, 7)
    I = np.repeat(u, b, axis=0)
    for s in (0.0, 1.0, 14.2857, 100.0):
        f = O.forward(I, I, s)
        assert f["loss"] == pytest.approx(math.log(b), abs=1e-12)
        dI, dT = O.backward(I, I, s)
        assert np.abs(dI).max() < 1e-12 and np.abs(dT).max() < 1e-12


@pytest.mark.parametrize("s", [0.0, 1.0, 14.2857, 100.0])
def test_onehot_closed_form_matches_definition(s):
    b, K, d = 96, 8, 16
    I = np.zeros((b, d))
    I[np.arange(b), np.arange(b) % K] = 1.0
    f = O.loss_and_grads(I, I, s)
    cf = O.onehot_closed_form(b, K, d, s)
    assert f["loss"] == pytest.approx(cf["loss"], rel=1e-12, abs=1e-14)
    assert np.allclose(f["r"], cf["r"], atol=1e-11) and np.allclose(f["c"], cf["c"], atol=1e-11)
    assert np.allclose(f["dI"], cf["dI"], atol=1e-14)
    assert np.allclose(f["dT"], cf["dT"], atol=1e-14)


def test_onehot_orthonormal_2x2_is_spec_value():
    cf = O.onehot_closed_form(2, 2, 2, 1.0)
    assert cf["loss"] == pytest.approx(golden()["loss_2x2_identity_s1"], abs=1e-15)


@pytest.mark.parametrize("s", [1.0, 14.2857, 100.0])
def test_codebook_closed_form_matches_definition(s):
    b, d, K, seed = 200, 32, 12, 3
    ci, ct = codebook_vectors(d, K, seed)
    ai, at = codebook_assignment(b, K, seed)
    I, T = make_features(b, d, seed=seed, dist="codebook", K=K)
    f = O.loss_and_grads(I, T, s)
    cf = O.codebook_closed_form(ci, ct, ai, at, s)
    assert f["loss"] == pytest.approx(cf["loss"], rel=1e-12)
    assert np.allclose(f["r"], cf["r"], atol=1e-10) and np.allclose(f["c"], cf["c"], atol=1e-10)
    assert np.allclose(f["diag"], cf["diag"], atol=1e-12)
    assert np.allclose(f["dI"], cf["dI"], atol=1e-13) and np.allclose(f["dT"], cf["dT"], atol=1e-13)


# ------------------------------------------------------------------ identities and symmetry
@pytest.mark.parametrize("s", [0.5, 14.2857, 100.0])
def test_scale_identity(s):
    """sum_i <dI_i, I_i> = sum_j <dT_j, T_j> = s dL/ds (x is bilinear in s, I, T); dL/ds by central FD."""
    b, d = 24, 8
    I = rand_feats(b, d, 21)
    T = rand_feats(b, d, 22)
    s32 = float(np.float32(s))
    dI, dT, ds = O.backward(I, T, s, want_ds=True)
    lhs = (dI * I).sum()
    rhs = (dT * T).sum()
    h = 1e-5 * max(1.0, s32)
    fd = (brute.loss(I.tolist(), T.tolist(), s32 + h) - brute.loss(I.tolist(), T.tolist(), s32 - h)) / (2 * h)
    assert lhs == pytest.approx(rhs, rel=1e-10, abs=1e-13)
    assert lhs == pytest.approx(s32 * ds, rel=1e-10, abs=1e-13)
    assert ds == pytest.approx(fd, rel=1e-6, abs=1e-9)


@pytest.mark.parametrize("s", [1.0, 14.2857, 100.0])
def test_streamed_grad_scale(s):
    """streamed_grad_scale (the large-b ds oracle) against central finite differences of the brute-force loss
    (tests/brute.py, Eq.1 written out) and the s dL/ds = sum_i <dI_i, I_i> identity, across chunkings."""
    b, d = 20, 8
    I = rand_feats(b, d, 23)
    T = rand_feats(b, d, 24)
    s32 = float(np.float32(s))
    f = O.forward(I, T, s)
    h = 1e-5 * max(1.0, s32)
    fd = (brute.loss(I.tolist(), T.tolist(), s32 + h) - brute.loss(I.tolist(), T.tolist(), s32 - h)) / (2 * h)
    dI, _ = O.backward(I, T, s, 0.7)
    for chunk in (1, 7, 64):
        ds = O.streamed_grad_scale(I, T, s, f["r"], f["c"], 0.7, chunk=chunk)
        assert ds == pytest.approx(0.7 * fd, rel=1e-6, abs=1e-9)
        assert s32 * ds == pytest.approx((dI * I).sum(), rel=1e-10, abs=1e-13)


def test_swap_symmetry():
    b, d = 40, 12
    I = rand_feats(b, d, 31)
    T = rand_feats(b, d, 32)
    f1 = O.loss_and_grads(I, T, 14.2857)
    f2 = O.loss_and_grads(T, I, 14.2857)
    assert f1["loss"] == pytest.approx(f2["loss"], rel=1e-13)
    assert np.allclose(f1["r"], f2["c"]) and np.allclose(f1["c"], f2["r"])
    assert np.allclose(f1["dI"], f2["dT"], atol=1e-15) and np.allclose(f1["dT"], f2["dI"], atol=1e-15)


def test_softmax_rows_sum_to_one_and_loss_nonneg():
    b, d = 50, 16
    I = rand_feats(b, d, 41)
    T = rand_feats(b, d, 42)
    X = O.similarity(I, T, 14.2857)
    f = O.forward(I, T, 14.2857)
    assert np.allclose(np.exp(X - f["r"][:, None]).sum(1), 1.0, atol=1e-12)
    assert np.allclose(np.exp(X - f["c"][None, :]).sum(0), 1.0, atol=1e-12)
    assert f["loss_i"] >= 0 and f["loss_t"] >= 0
    assert np.all(f["r"] >= f["diag"]) and np.all(f["c"] >= f["diag"])


# ------------------------------------------------------------------ tiling and ring
@pytest.mark.parametrize("t", [1, 3, 16, 64])
def test_tiled_lse_equals_direct(t):
    b, d = 100, 8
    I = rand_feats(b, d, 51)
    T = rand_feats(b, d, 52)
    X = O.similarity(I, T, 30.0)
    assert np.allclose(O.tiled_lse_rows(X, t, t), O.lse_rows(X), rtol=1e-12, atol=1e-12)
    assert np.allclose(O.tiled_lse_rows(X, 7, t), O.lse_rows(X), rtol=1e-12, atol=1e-12)


def test_merge_order_independent():
    rng = np.random.default_rng(5)
    v = rng.normal(size=40) * 50
    a = O.NEG_INF
    for x in v:
        a = O.merge_lse(a, x)
    b = O.NEG_INF
    for x in v[::-1]:
        b = O.merge_lse(b, x)
    m = v.max()
    direct = m + math.log(math.fsum(math.exp(x - m) for x in v))
    assert a == pytest.approx(direct, rel=1e-13) and b == pytest.approx(direct, rel=1e-13)


def test_streamed_and_sampled_match_full():
    b, d = 300, 16
    I = rand_feats(b, d, 61)
    T = rand_feats(b, d, 62)
    f = O.loss_and_grads(I, T, 14.2857)
    st = O.streamed_forward(I, T, 14.2857, chunk=64)
    assert st["loss"] == pytest.approx(f["loss"], rel=1e-13)
    assert np.allclose(st["r"], f["r"], atol=1e-12) and np.allclose(st["c"], f["c"], atol=1e-12)
    rows = np.array([0, 5, 77, 299])
    dIs = O.sampled_row_grads(I, T, 14.2857, f["r"], f["c"], rows)
    dTs = O.sampled_row_grads(T, I, 14.2857, f["c"], f["r"], rows)
    assert np.allclose(dIs, f["dI"][rows], atol=1e-15) and np.allclose(dTs, f["dT"][rows], atol=1e-15)


@pytest.mark.parametrize("chunk", [1, 7, 64, 1000])
def test_streamed_row_lse_and_grads_match_full(chunk):
    """The large-b (cfg5) sampled helpers streamed over column chunks equal the materialised definition (whose
    pins are above: brute force, finite differences) for any chunking."""
    b, d = 200, 12
    I = rand_feats(b, d, 71)
    T = rand_feats(b, d, 72)
    f = O.loss_and_grads(I, T, 14.2857)
    rows = np.array([0, 3, 64, 128, 199])
    assert np.allclose(O.streamed_row_lse(I[rows], T, 14.2857, chunk=chunk), f["r"][rows], atol=1e-12)
    assert np.allclose(O.streamed_row_lse(T[rows], I, 14.2857, chunk=chunk), f["c"][rows], atol=1e-12)
    dIs = O.streamed_row_grads(I[rows], T, 14.2857, f["r"][rows], f["c"], rows, chunk=chunk)
    dTs = O.streamed_row_grads(T[rows], I, 14.2857, f["c"][rows], f["r"], rows, chunk=chunk)
    assert np.allclose(dIs, f["dI"][rows], atol=1e-15) and np.allclose(dTs, f["dT"][rows], atol=1e-15)


def test_ring_schedule_spec_example_and_coverage():
    # i=2, j=3 (1-based), n=4 -> k = (i+j-1) mod n = 0  == 0-based step 2
    assert O.ring_schedule(2, 4, 2) == 0
    for n in range(1, 17):
        seen = set()
        for step in range(n):
            held = [O.ring_schedule(r, n, step) for r in range(n)]
            assert sorted(held) == list(range(n))  # a permutation every step
            for r in range(n):
                seen.add((r, held[r]))
                if step + 1 < n:  # block held at step+1 is the one rank r+1 held at step (flows r+1 -> r)
                    assert O.ring_schedule(r, n, step + 1) == O.ring_schedule((r + 1) % n, n, step)
        assert len(seen) == n * n  # every (row shard, column shard) exactly once


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_ring_matches_direct(n):
    b, d = 64, 8
    I = rand_feats(b, d, 71)
    T = rand_feats(b, d, 72)
    f = O.loss_and_grads(I, T, 14.2857)
    rf = O.ring_forward(I, T, 14.2857, n)
    assert rf["loss"] == pytest.approx(f["loss"], rel=1e-13)
    assert np.allclose(rf["r"], f["r"], atol=1e-12) and np.allclose(rf["c"], f["c"], atol=1e-12)
    dI, dT = O.ring_backward(I, T, 14.2857, n, rf["r"], rf["c"])
    assert np.allclose(dI, f["dI"], atol=1e-15) and np.allclose(dT, f["dT"], atol=1e-15)


def test_ring_divisibility_error():
    I = rand_feats(7, 4, 1)
    with pytest.raises(ValueError):
        O.ring_forward(I, I, 1.0, 2)  # S:268 / S:437


def test_stability_large_magnitudes():
    b, d = 16, 4
    I = rand_feats(b, d, 81)
    T = rand_feats(b, d, 82)
    f = O.loss_and_grads(I, T, 5000.0)  # |x| up to 5000
    assert math.isfinite(f["loss"]) and np.isfinite(f["dI"]).all() and np.isfinite(f["dT"]).all()


def test_nan_propagates():
    X = np.array([[0.0, np.nan, 1.0]])
    assert np.isnan(O.tile_lse(X)[0])


def test_bf16_inputs_widen_exactly():
    I, T = make_features(16, 8, seed=0)
    assert I.dtype == torch.bfloat16
    a = O.to_f64(I)
    assert np.array_equal(a, I.float().numpy().astype(np.float64))


# ------------------------------------------------------------------ mutation sensitivity
def test_mutations_are_caught():
    b, d = 48, 8
    I = rand_feats(b, d, 91)
    T = rand_feats(b, d, 92)
    X = O.similarity(I, T, 14.2857)
    direct = O.lse_rows(X)

    def merge_paper_literal(l, v):  # Eq.4 taken literally: init 0 (not the identity)
        return l + np.log1p(np.exp(v - l))

    l = np.zeros(b)
    for j0 in range(0, b, 16):
        l = merge_paper_literal(l, O.tile_lse(X[:, j0:j0 + 16]))
    assert np.abs(l - direct).max() > 1e-6

    def merge_sign_flip(l, v):
        hi = np.maximum(l, v)
        return hi - np.log1p(np.exp(-np.abs(l - v)))

    l = np.full(b, O.NEG_INF)
    l = O.tile_lse(X[:, :16])
    for j0 in range(16, b, 16):
        l = merge_sign_flip(l, O.tile_lse(X[:, j0:j0 + 16]))
    assert np.abs(l - direct).max() > 1e-6

    # ring off-by-one: the held block (rank + step + 1) % n double-counts one block and skips another
    n, bs = 4, b // 4
    r = [np.full(bs, O.NEG_INF) for _ in range(n)]
    for step in range(n):
        for rank in range(n):
            k = (rank + step + (1 if step == n - 1 else 0)) % n
            Xk = O.similarity(I[rank * bs:(rank + 1) * bs], T[k * bs:(k + 1) * bs], 14.2857)
            r[rank] = O.merge_lse(r[rank], O.tile_lse(Xk))
    assert np.abs(np.concatenate(r) - direct).max() > 1e-6

    # missing max-shift overflows at large magnitude
    with np.errstate(over="ignore"):
        naive = np.log(np.exp(np.array([[1000.0, 1000.0]])).sum(1))
    assert not np.isfinite(naive[0]) and np.isfinite(O.tile_lse([[1000.0, 1000.0]])[0])

    # dropped symmetric term / transposed gradient operand are caught by finite differences
    dI, dT = O.backward(I[:5, :3], T[:5, :3], 2.0)
    fdI, fdT = brute.fd_grads(I[:5, :3].tolist(), T[:5, :3].tolist(), 2.0)
    assert not np.allclose(2 * dI, np.array(fdI), rtol=1e-3)  # losing the 1/2 of Q4 would fail
    assert not np.allclose(dT, np.array(fdI), rtol=1e-3)


def test_backward_abs_bounds_gradient():
    # |sum_j G_ij T_j| <= sum_j |G_ij| |T_j| (triangle inequality), with equality for nonnegative summands
    b, d = 30, 6
    I = rand_feats(b, d, 101)
    T = rand_feats(b, d, 102)
    dI, dT = O.backward(I, T, 5.0)
    aI, aT = O.backward_abs(I, T, 5.0)
    assert np.all(aI >= np.abs(dI) - 1e-15) and np.all(aT >= np.abs(dT) - 1e-15)
    Ip, Tp = np.abs(I), np.abs(T)
    cf = O.onehot_closed_form(8, 8, 8, 1.0)
    E = np.eye(8)
    aI1, _ = O.backward_abs(E, E, 1.0)
    # one-hot: off-class components of dI are s*g/b*m*q >= 0 and equal their magnitude bound
    off = ~np.eye(8, dtype=bool)
    assert np.allclose(aI1[off], np.abs(cf["dI"][off]), atol=1e-15)


def test_streamed_threads_bitwise_equal_serial():
    """The large-b parity tests run the streamed oracle with worker threads (wall time only): every output is
    bitwise the serial loop's (same per-chunk arithmetic, chunk-ordered combination)."""
    g = np.random.default_rng(3)
    I = g.standard_normal((1000, 24))
    T = g.standard_normal((1000, 24))
    a = oracle.streamed_forward(I, T, 3.0, chunk=96)
    b = oracle.streamed_forward(I, T, 3.0, chunk=96, workers=4)
    assert all(np.array_equal(a[k], b[k]) for k in ("r", "c", "diag")) and a["loss"] == b["loss"]
    assert oracle.streamed_grad_scale(I, T, 3.0, a["r"], a["c"], 0.7, chunk=96) == \
        oracle.streamed_grad_scale(I, T, 3.0, a["r"], a["c"], 0.7, chunk=96, workers=4)
