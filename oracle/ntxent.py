"""fp64 numpy oracle of the single-modality NT-Xent loss (SimCLR) -- TEST INFRASTRUCTURE ONLY.

SURVEY.md 8(f) f4: the second workload through the same kernels.  The paper names self-supervised
representation learning (SimCLR) as a contrastive application the method serves ("positive pairs
are created by augmenting the same image in different ways") but does not write the loss out, so this is
the standard definition (SimCLR's NT-Xent), written out with the similarity matrix fully materialised:

    views   Z = [A; B] (2b x d): A_i and B_i are the two views of example i
    X       = s Z Z^T, with the self-similarity X_ii excluded (masked to -inf)          (reading N2)
    r_k     = LSE_{k' != k} X_kk'                                                       (row LSE over 2b-1 views)
    pi(k)   = k + b mod 2b (the other view of the same example)                         (reading N1)
    L       = (1/2b) sum_k (r_k - X_{k,pi(k)})
    G_kk'   = dL/dX_kk' = (g/2b) (P_kk' - [k' == pi(k)]),  P_kk' = e^{X_kk' - r_k} (k' != k), G_kk = 0
    dZ      = s (G + G^T) Z        (X is s Z Z^T: both factors are Z)                   (reading N3)

No function here shares code with the CUDA path or imports it.
"""
from __future__ import annotations

import math

import numpy as np

from .infonce import _scale32, lse_rows, to_f64


def views(A, B) -> np.ndarray:
    A = to_f64(A)
    B = to_f64(B)
    if A.ndim != 2 or A.shape != B.shape:
        raise ValueError(f"shape error: A{A.shape} B{B.shape}")
    return np.concatenate([A, B], axis=0)


def similarity(A, B, s: float) -> np.ndarray:
    """X = s Z Z^T with the diagonal (self-similarity) set to -inf (reading N2)."""
    Z = views(A, B)
    X = _scale32(s) * (Z @ Z.T)
    np.fill_diagonal(X, -np.inf)
    return X


def forward(A, B, s: float) -> dict:
    """r over the 2b-1 other views of every view; pos_i = X_{i, i+b} = s <A_i, B_i>; L = mean_k (r_k - X_{k,pi(k)}).
    Returns r_a = r[:b] (A views), r_b = r[b:] (B views), pos [b], loss."""
    X = similarity(A, B, s)
    n = X.shape[0]
    b = n // 2
    r = lse_rows(X)
    pos = np.array([X[i, i + b] for i in range(b)])
    loss = math.fsum(np.concatenate([r[:b] - pos, r[b:] - pos])) / n
    return {"loss": loss, "r_a": r[:b].copy(), "r_b": r[b:].copy(), "pos": pos}


def backward(A, B, s: float, g: float = 1.0) -> tuple:
    """dA, dB of g*L: G = (g/2b)(P - Pi) with P the row softmax over the other views (G_kk = 0) and Pi the
    permutation matrix of the positives, then dZ = s (G + G^T) Z."""
    Z = views(A, B)
    X = similarity(A, B, s)
    n = Z.shape[0]
    b = n // 2
    r = lse_rows(X)
    P = np.exp(X - r[:, None])  # exp(-inf) = 0 on the diagonal
    G = (g / n) * P
    idx = np.arange(n)
    G[idx, (idx + b) % n] -= g / n
    dZ = _scale32(s) * ((G + G.T) @ Z)
    return dZ[:b].copy(), dZ[b:].copy()


def onehot_closed_form(b: int, K: int, d: int, s: float, g: float = 1.0) -> dict:
    """A_i = B_i = e_{i mod K}, K | b, K <= d, m = b/K.  Every view has 2m - 1 other views of its class (logit s,
    one of them its positive) and 2b - 2m views of other classes (logit 0): r = Lam = log((2m-1) e^s + 2b - 2m),
    L = Lam - s.  With p = e^{s - Lam}, q = e^{-Lam}, G is symmetric: (g/2b)(p - [positive]) within the class,
    (g/2b) q across classes, so dZ_k = 2 s sum_k' G_kk' z_k' = (s g / b) [((2m-1) p - 1) e_c + 2m q sum_{c' != c} e_c']."""
    if b % K or K > d:
        raise ValueError("need K | b and K <= d")
    s32 = _scale32(s)
    m = b // K
    lam = math.log((2 * m - 1) * math.exp(s32) + (2 * b - 2 * m))
    p = math.exp(s32 - lam)
    q = math.exp(-lam)
    dA = np.zeros((b, d))
    dA[:, :K] = s32 * g / b * 2 * m * q
    dA[np.arange(b), np.arange(b) % K] = s32 * g / b * ((2 * m - 1) * p - 1.0)
    return {"loss": lam - s32, "r_a": np.full(b, lam), "r_b": np.full(b, lam), "pos": np.full(b, s32),
            "dA": dA, "dB": dA.copy()}


def sampled_rows(A, B, s: float, r_a, r_b, rows, g: float = 1.0) -> tuple:
    """Exact fp64 gradient rows dA_i, dB_i for a sample of example indices i (large-b protocol), given the row
    LSEs r_a, r_b over all 2b views: dZ_k = (s g / 2b) sum_{k' != k} (P_kk' + P_k'k) z_k' - (s g / b) z_pi(k)."""
    Z = views(A, B)
    n = Z.shape[0]
    b = n // 2
    s32 = _scale32(s)
    r = np.concatenate([np.asarray(r_a, np.float64), np.asarray(r_b, np.float64)])
    out = []
    for half in (0, 1):
        ks = np.asarray(rows, dtype=np.int64) + half * b
        X = s32 * (Z[ks] @ Z.T)
        X[np.arange(len(ks)), ks] = -np.inf
        W = (g / n) * (np.exp(X - r[ks, None]) + np.exp(X - r[None, :]))
        W[np.arange(len(ks)), (ks + b) % n] -= 2.0 * g / n
        out.append(s32 * (W @ Z))
    return out[0], out[1]
