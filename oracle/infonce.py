"""fp64 numpy oracle of the symmetric InfoNCE loss (Inf-CL, arXiv 2410.17243) -- TEST INFRASTRUCTURE ONLY.

What the method reaches exactly (up to rounding order) is the plain definition of the loss and its
gradients, so the oracle is that definition written out with the similarity matrix fully materialised
(the "vanilla implementation").  The tiled pieces (tile_lse / merge_lse / tiled_lse_rows /
ring_*) follow the paper's Eq.3-Eq.5 and Alg.1/Alg.3 step by step, only so that tests can check that
tiling is exact; the GPU parity tests compare against ``forward``/``backward``.

Notation: b batch, d feature dim (paper's c), s logit scale (temperature omitted by the
paper, P:91 -> reading Q3), x_ij = s <I_i, T_j>, r_i = LSE_j x_ij (paper's l, image->text),
c_j = LSE_i x_ij (text->image), L = (L_I + L_T) / 2 (reading Q4).
"""
from __future__ import annotations

import math

import numpy as np

NEG_INF = -math.inf


def to_f64(x) -> np.ndarray:
    """Exact widening of the values the GPU received (bf16/fp32 torch tensor or array) to fp64."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu").to(torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def _scale32(s: float) -> float:
    """The logit scale as the GPU sees it: an fp32 runtime scalar (reading Q3), widened exactly."""
    return float(np.float32(s))


# --------------------------------------------------------------------------------------------------
# Eq.1 / Eq.3: the similarity matrix (or one tile of it)
# --------------------------------------------------------------------------------------------------
def similarity(I, T, s: float) -> np.ndarray:
    """X = s * I * T^T  ("x_ij = I_i . T_j", scale per reading Q3; Alg.2 l.8 P:268 for a tile)."""
    I = to_f64(I)
    T = to_f64(T)
    if I.ndim != 2 or T.ndim != 2 or I.shape[1] != T.shape[1]:
        raise ValueError(f"shape error: I{I.shape} T{T.shape}")
    return _scale32(s) * (I @ T.T)


# --------------------------------------------------------------------------------------------------
# Eq.5 and Eq.4: stable per-tile LSE and the serial merge
# --------------------------------------------------------------------------------------------------
def tile_lse(X) -> np.ndarray:
    """Row-wise l^{i,j} = m + log sum_k e^{X_:,k - m}, m = row max (Eq.5).

    NaN in -> NaN out.  A row of -inf stays -inf (empty tile).
    """
    X = np.asarray(X, dtype=np.float64)
    m = X.max(axis=1)
    mf = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(invalid="ignore"):
        ssum = np.exp(X - mf[:, None]).sum(axis=1)
        out = mf + np.log(ssum)
    return np.where(np.isneginf(m), NEG_INF, np.where(np.isnan(m), np.nan, out))


def merge_lse(a, v):
    """Eq.4 l <- l + log(1 + e^{l^{i,j} - l}) with the -inf identity (reading Q1) and the
    overflow-free symmetric form max(a,b) + log1p(e^{-|a-b|}) (reading Q2)."""
    a = np.asarray(a, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    hi = np.maximum(a, v)
    lo = np.minimum(a, v)
    with np.errstate(invalid="ignore"):
        out = hi + np.log1p(np.exp(lo - hi))
    out = np.where(np.isneginf(lo), hi, out)  # identity: (-inf) (+) v = v, also guards (-inf)-(-inf)
    return out


def lse_rows(X) -> np.ndarray:
    """Direct row LSE of a full matrix (Eq.5 applied to whole rows): r_i = LSE_j X_ij."""
    return tile_lse(X)


def lse_cols(X) -> np.ndarray:
    """Direct column LSE (the text->image direction, "symmetric"): c_j = LSE_i X_ij."""
    return tile_lse(np.asarray(X, dtype=np.float64).T)


def tiled_lse_rows(X, t_r: int, t_c: int) -> np.ndarray:
    """Alg.2 on a materialised X: for each row tile (parallel for, l.3) start from the
    identity (reading Q1), then for each column tile (l.6, bound n_c per reading Q6, ceil per Q11)
    compute the tile LSE (Eq.5, l.9-10) and merge it (Eq.4, l.11-12)."""
    X = np.asarray(X, dtype=np.float64)
    b_r, b_c = X.shape
    out = np.empty(b_r)
    for i0 in range(0, b_r, t_r):
        l = np.full(min(t_r, b_r - i0), NEG_INF)
        for j0 in range(0, b_c, t_c):
            l = merge_lse(l, tile_lse(X[i0:i0 + t_r, j0:j0 + t_c]))
        out[i0:i0 + t_r] = l
    return out


# --------------------------------------------------------------------------------------------------
# The plain definition: loss, LSEs, gradients (Eq.1, Eq.2, Eq.6-8, symmetric per Q4/Q5)
# --------------------------------------------------------------------------------------------------
def forward(I, T, s: float) -> dict:
    """Materialise X, then r (row LSE), c (column LSE), diag x_ii and
    L = (L_I + L_T)/2 with L_I = mean_i(r_i - x_ii) (Eq.2) and L_T = mean_j(c_j - x_jj)."""
    X = similarity(I, T, s)
    b = X.shape[0]
    if X.shape[1] != b:
        raise ValueError("I and T must have the same number of rows")
    r = lse_rows(X)
    c = lse_cols(X)
    diag = np.diag(X).copy()
    L_I = math.fsum(r - diag) / b
    L_T = math.fsum(c - diag) / b
    return {"loss": 0.5 * (L_I + L_T), "loss_i": L_I, "loss_t": L_T, "r": r, "c": c, "diag": diag}


def loss_only(I, T, s: float) -> float:
    return forward(I, T, s)["loss"]


def backward(I, T, s: float, g: float = 1.0, r=None, c=None, want_ds: bool = False, chunk: int = 4096):
    """Gradients of g * L.  Eq.7 gives dL_I/dI_i = -(1/b) T_i + (1/b) sum_j e^{x_ij - l_i} T_j
    with the scale omitted; restoring s and adding the symmetric text->image term (readings Q3-Q5):

        G_ij = g/(2b) * (e^{x_ij - r_i} + e^{x_ij - c_j}) - (g/b) * [i == j]
        dI   = s * G T          dT = s * G^T I          ds = sum_ij G_ij x_ij / s

    Computed in row chunks of X so memory is one chunk plus O(b d); r and c default to the exact LSEs.
    """
    I = to_f64(I)
    T = to_f64(T)
    s32 = _scale32(s)
    b, d = I.shape
    if r is None or c is None:
        f = forward(I, T, s)
        r = f["r"] if r is None else r
        c = f["c"] if c is None else c
    r = np.asarray(r, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    dI = np.zeros((b, d))
    dT = np.zeros((b, d))
    ds = 0.0
    for i0 in range(0, b, chunk):
        i1 = min(b, i0 + chunk)
        Xc = s32 * (I[i0:i1] @ T.T)
        G = (g / (2.0 * b)) * (np.exp(Xc - r[i0:i1, None]) + np.exp(Xc - c[None, :]))
        rows = np.arange(i0, i1)
        G[rows - i0, rows] -= g / b
        dI[i0:i1] = s32 * (G @ T)
        dT += s32 * (G.T @ I[i0:i1])
        if want_ds:
            ds += float((G * (I[i0:i1] @ T.T)).sum())
    if want_ds:
        return dI, dT, ds
    return dI, dT


def backward_abs(I, T, s: float, g: float = 1.0, r=None, c=None, chunk: int = 4096):
    """Magnitude of the gradient summands: (|s| |G| |T|, |s| |G|^T |I|) elementwise, with G as in ``backward``.
    Any evaluation that rounds G (or T, I) to a working precision with unit roundoff u has componentwise error
    <= ~u * this bound (standard GEMM rounding analysis); it is the conditioning term of the gradient gate."""
    I = to_f64(I)
    T = to_f64(T)
    s32 = _scale32(s)
    b, d = I.shape
    if r is None or c is None:
        f = forward(I, T, s)
        r, c = f["r"], f["c"]
    r = np.asarray(r, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    aI = np.zeros((b, d))
    aT = np.zeros((b, d))
    for i0 in range(0, b, chunk):
        i1 = min(b, i0 + chunk)
        Xc = s32 * (I[i0:i1] @ T.T)
        G = (g / (2.0 * b)) * (np.exp(Xc - r[i0:i1, None]) + np.exp(Xc - c[None, :]))
        rows = np.arange(i0, i1)
        G[rows - i0, rows] -= g / b
        G = np.abs(G)
        aI[i0:i1] = abs(s32) * (G @ np.abs(T))
        aT += abs(s32) * (G.T @ np.abs(I[i0:i1]))
    return aI, aT


def loss_and_grads(I, T, s: float, g: float = 1.0) -> dict:
    f = forward(I, T, s)
    dI, dT = backward(I, T, s, g, f["r"], f["c"])
    f.update(dI=dI, dT=dT)
    return f


# --------------------------------------------------------------------------------------------------
# Large-b protocol: exact fp64 streamed over row chunks, sampled gradients
# --------------------------------------------------------------------------------------------------
def _chunk_map(fn, starts, chunk_bytes: int, workers: int = 1) -> list:
    """[fn(i0) for i0 in starts]; with workers > 1 (the large-b parity tests' wall time) evaluated by up to that
    many threads (numpy's exp and matmul release the GIL).  Each chunk's arithmetic is exactly the serial loop's
    and the results come back in chunk order, so every caller combines them in the same order as a plain loop:
    threading changes wall time only.  Workers are capped by host memory (~12 GB of chunk temporaries).  The
    default (1) is the plain loop, which is what bench.py times as the CPU baseline."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    starts = list(starts)
    workers = max(1, min(workers, os.cpu_count() or 1, len(starts), int(12e9 // max(1, chunk_bytes))))
    if workers == 1:
        return [fn(i0) for i0 in starts]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, starts))


def streamed_forward(I, T, s: float, chunk: int = 1024, row_limit: int | None = None, workers: int = 1) -> dict:
    """Same definition as ``forward`` but X is streamed in row chunks: r per chunk, c by merging the
    chunk's column LSEs (Eq.4 merge, reading Q1/Q2).  O(chunk * b) memory; exact up to rounding.
    ``row_limit`` restricts the rows (a bounded sample of the workload for CPU timing): r and diag are
    then for those rows only and c is the partial LSE over them."""
    I = to_f64(I)
    T = to_f64(T)
    s32 = _scale32(s)
    b = I.shape[0]
    nrows = b if row_limit is None else min(b, row_limit)
    r = np.empty(nrows)
    diag = np.empty(nrows)
    c = np.full(T.shape[0], NEG_INF)

    def one(i0):  # one row chunk of X: its row LSEs, its column LSEs (merged below in chunk order), its diagonal
        i1 = min(nrows, i0 + chunk)
        Xc = s32 * (I[i0:i1] @ T.T)
        return tile_lse(Xc), tile_lse(Xc.T), Xc[np.arange(i1 - i0), np.arange(i0, i1)]

    for i0, (rc, cc, dc) in zip(range(0, nrows, chunk),
                                _chunk_map(one, range(0, nrows, chunk), 4 * chunk * T.shape[0] * 8, workers)):
        i1 = min(nrows, i0 + chunk)
        r[i0:i1] = rc
        c = merge_lse(c, cc)
        diag[i0:i1] = dc
    out = {"r": r, "c": c, "diag": diag}
    if row_limit is None:
        out["loss"] = 0.5 * (math.fsum(r - diag) + math.fsum(c - diag)) / b
    return out


def streamed_grad_scale(I, T, s: float, r, c, g: float = 1.0, chunk: int = 2048, workers: int = 1) -> float:
    """g dL/ds = sum_ij G_ij <I_i, T_j> with G as in ``backward`` (x_ij = s <I_i, T_j> is linear in s, so
    dL/ds = sum_ij (dL/dx_ij) x_ij / s), streamed over row chunks of X without forming dI, dT:
    one GEMM per chunk.  r, c are the LSEs (exact ones from ``streamed_forward`` for an exact result)."""
    I = to_f64(I)
    T = to_f64(T)
    s32 = _scale32(s)
    b = I.shape[0]
    r = np.asarray(r, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    def one(i0):  # one row chunk: sum_ij G_ij P_ij over its rows
        i1 = min(b, i0 + chunk)
        P = I[i0:i1] @ T.T
        Xc = s32 * P
        G = (g / (2.0 * b)) * (np.exp(Xc - r[i0:i1, None]) + np.exp(Xc - c[None, :]))
        rows = np.arange(i0, i1)
        G[rows - i0, rows] -= g / b
        return float((G * P).sum())

    acc = _chunk_map(one, range(0, b, chunk), 6 * chunk * T.shape[0] * 8, workers)
    return math.fsum(acc)


def sampled_row_grads(A, B, s: float, lse_a, lse_b, rows, g: float = 1.0) -> np.ndarray:
    """Exact fp64 gradient rows dA_i = s * sum_j G_ij B_j for a sample of rows i of the stationary side.
    G_ij = g/(2b)(e^{x_ij - lse_a_i} + e^{x_ij - lse_b_j}) - (g/b)[i==j].  With (A,B,lse_a,lse_b) =
    (I,T,r,c) this is dI; with (T,I,c,r) it is dT (dT_j = s sum_i G_ij I_i, same formula transposed)."""
    A = to_f64(A)
    B = to_f64(B)
    s32 = _scale32(s)
    b = A.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    X = s32 * (A[rows] @ B.T)
    G = (g / (2.0 * b)) * (np.exp(X - np.asarray(lse_a)[rows, None]) + np.exp(X - np.asarray(lse_b)[None, :]))
    G[np.arange(len(rows)), rows] -= g / b
    return s32 * (G @ B)


def streamed_row_lse(A_rows, B, s: float, chunk: int = 131072) -> np.ndarray:
    """Exact fp64 LSE over ALL rows of B of x_ij = s <A_rows_i, B_j> for a sample of rows (A_rows [k][d]),
    streamed over row chunks of B with the Eq.4 merge (reading Q1/Q2): O(k * chunk) memory, so usable at the
    paper's 4M batch where B in fp64 alone is 26 GB.  B may be a bf16 torch tensor (widened chunk by chunk)."""
    A_rows = to_f64(A_rows)
    s32 = _scale32(s)
    out = np.full(A_rows.shape[0], NEG_INF)
    for j0 in range(0, B.shape[0], chunk):
        X = s32 * (A_rows @ to_f64(B[j0:j0 + chunk]).T)
        out = merge_lse(out, tile_lse(X))
    return out


def streamed_row_grads(A_rows, B, s: float, lse_rows, lse_b, rows, g: float = 1.0, chunk: int = 131072) -> np.ndarray:
    """``sampled_row_grads`` streamed over row chunks of B: dA_i = s sum_j G_ij B_j for global rows ``rows``
    (A_rows = A[rows]), G_ij = g/(2b)(e^{x_ij - lse_rows_i} + e^{x_ij - lse_b_j}) - (g/b)[j == rows_i]."""
    A_rows = to_f64(A_rows)
    s32 = _scale32(s)
    b = B.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    lse_rows = np.asarray(lse_rows, dtype=np.float64)
    lse_b = np.asarray(lse_b, dtype=np.float64)
    out = np.zeros_like(A_rows)
    for j0 in range(0, b, chunk):
        Bc = to_f64(B[j0:j0 + chunk])
        X = s32 * (A_rows @ Bc.T)
        G = (g / (2.0 * b)) * (np.exp(X - lse_rows[:, None]) + np.exp(X - lse_b[None, j0:j0 + Bc.shape[0]]))
        hit = (rows >= j0) & (rows < j0 + Bc.shape[0])
        G[np.nonzero(hit)[0], rows[hit] - j0] -= g / b
        out += s32 * (G @ Bc)
    return out


# --------------------------------------------------------------------------------------------------
# Cross-GPU ring (Alg.1, Alg.3) simulated in one process on materialised shards
# --------------------------------------------------------------------------------------------------
def ring_schedule(rank: int, world: int, step: int) -> int:
    """Index of the text block held by ``rank`` at 0-based ``step``: k = (i + j - 1) mod n with
    1-based j (Alg.3 l.7) == (rank + step) mod n; data flows from rank+1 to rank (reading Q13)."""
    if not (0 <= rank < world) or not (0 <= step < world):
        raise ValueError("rank/step out of range")
    return (rank + step) % world


def ring_forward(I, T, s: float, world: int) -> dict:
    """Alg.1: each worker holds row shard I^i; for n rounds it computes the local LSE of
    (I^i, held T) (Alg.2 via tile_lse on the shard product), merges it into l^i (Eq.4) and passes T on.
    The held block's column LSE partial travels with it (symmetric direction)."""
    I = to_f64(I)
    T = to_f64(T)
    b = I.shape[0]
    if b % world:
        raise ValueError(f"configuration error: b={b} not divisible by n={world}")
    bs = b // world
    r = [np.full(bs, NEG_INF) for _ in range(world)]
    c = [np.full(bs, NEG_INF) for _ in range(world)]  # indexed by block owner
    diag = [None] * world
    for step in range(world):
        for rank in range(world):
            k = ring_schedule(rank, world, step)
            X = similarity(I[rank * bs:(rank + 1) * bs], T[k * bs:(k + 1) * bs], s)
            r[rank] = merge_lse(r[rank], tile_lse(X))
            c[k] = merge_lse(c[k], tile_lse(X.T))
            if k == rank:
                diag[rank] = np.diag(X).copy()
    r = np.concatenate(r)
    c = np.concatenate(c)
    diag = np.concatenate(diag)
    loss = 0.5 * (math.fsum(r - diag) + math.fsum(c - diag)) / b
    return {"r": r, "c": c, "diag": diag, "loss": loss}


def ring_backward(I, T, s: float, world: int, r, c, g: float = 1.0):
    """Alg.3: dI^i accumulates locally; a dT cache rotates with the text block and, after n
    hops, ends at its owner.  Per-step work is Alg.4's recompute (Q8/Q9 readings)."""
    I = to_f64(I)
    T = to_f64(T)
    s32 = _scale32(s)
    b, d = I.shape
    bs = b // world
    dI = np.zeros((b, d))
    dT = np.zeros((b, d))
    for step in range(world):
        for rank in range(world):
            k = ring_schedule(rank, world, step)
            R = slice(rank * bs, (rank + 1) * bs)
            C = slice(k * bs, (k + 1) * bs)
            X = s32 * (I[R] @ T[C].T)
            G = (g / (2.0 * b)) * (np.exp(X - r[R][:, None]) + np.exp(X - c[C][None, :]))
            if k == rank:
                G[np.arange(bs), np.arange(bs)] -= g / b
            dI[R] += s32 * (G @ T[C])
            dT[C] += s32 * (G.T @ I[R])
    return dI, dT


# --------------------------------------------------------------------------------------------------
# Closed forms used as pins (and as full-size structured parity cases)
# --------------------------------------------------------------------------------------------------
def onehot_closed_form(b: int, K: int, d: int, s: float, g: float = 1.0) -> dict:
    """I_i = T_i = e_{i mod K}, K | b, K <= d, m = b/K.  Each row has m logits equal to s and b-m equal
    to 0, so r_i = c_i = Lam = log(m e^s + b - m) and L = Lam - s.  With p = e^{s - Lam}, q = e^{-Lam}:
    G_ij = g/b * (p if same class else q) - (g/b)[i==j], dI_i = s * sum_j G_ij e_{j mod K}."""
    if b % K or K > d:
        raise ValueError("need K | b and K <= d")
    s32 = _scale32(s)
    m = b // K
    lam = math.log(m * math.exp(s32) + (b - m)) if s32 < 700 else s32 + math.log(m + (b - m) * math.exp(-s32))
    p = math.exp(s32 - lam)
    q = math.exp(-lam)
    # dI_i = s*g/b * [ (m p - 1) e_{k(i)} + m q sum_{k' != k(i)} e_{k'} ]
    k = np.arange(b) % K
    dI = np.zeros((b, d))
    dI[:, :K] = s32 * g / b * m * q
    dI[np.arange(b), k] = s32 * g / b * (m * p - 1.0)
    return {"loss": lam - s32, "r": np.full(b, lam), "c": np.full(b, lam), "diag": np.full(b, s32),
            "dI": dI, "dT": dI.copy()}


def codebook_closed_form(ci, ct, ai, at, s: float, g: float = 1.0, rows=None) -> dict:
    """Rows drawn from K codewords: I_i = ci[ai[i]], T_j = ct[at[j]].  With the K x K Gram matrix
    H = s ci ct^T and code counts n_t[k] = #{j: at[j]=k}, n_i[k] = #{i: ai[i]=k}:
    r_i = LSE_k (H[ai_i, k] + log n_t[k]),  c_j = LSE_k (H[k, at_j] + log n_i[k]),  x_ii = H[ai_i, at_i].
    Gradients: dI_i = s * sum_j G_ij T_j grouped by code (exact, O(K^2 d + b d)).  ``rows`` selects the
    gradient rows returned (all if None)."""
    ci = to_f64(ci)
    ct = to_f64(ct)
    s32 = _scale32(s)
    ai = np.asarray(ai)
    at = np.asarray(at)
    b = ai.shape[0]
    K = ci.shape[0]
    H = s32 * (ci @ ct.T)
    n_t = np.bincount(at, minlength=K).astype(np.float64)
    n_i = np.bincount(ai, minlength=K).astype(np.float64)
    with np.errstate(divide="ignore"):
        log_nt = np.log(n_t)
        log_ni = np.log(n_i)
    rk = tile_lse(H + log_nt[None, :])  # per image code
    ck = tile_lse(H.T + log_ni[None, :])  # per text code
    r = rk[ai]
    c = ck[at]
    diag = H[ai, at]
    loss = 0.5 * (math.fsum(r - diag) + math.fsum(c - diag)) / b
    out = {"loss": loss, "r": r, "c": c, "diag": diag}
    rows = np.arange(b) if rows is None else np.asarray(rows)
    # dI_i = s g/(2b) sum_k n_t[k] (e^{H[a,k]-r_i} + e^{H[a,k]-ck[k]}) ct[k] - s g/b T_i
    Wi = n_t[None, :] * (np.exp(H - rk[:, None]) + np.exp(H - ck[None, :]))  # K_img x K_txt
    dIk = (s32 * g / (2.0 * b)) * (Wi @ ct)  # per image code
    dI = dIk[ai[rows]] - (s32 * g / b) * ct[at[rows]]
    Wt = n_i[:, None] * (np.exp(H - rk[:, None]) + np.exp(H - ck[None, :]))  # K_img x K_txt
    dTk = (s32 * g / (2.0 * b)) * (Wt.T @ ci)  # per text code
    dT = dTk[at[rows]] - (s32 * g / b) * ci[ai[rows]]
    out.update(dI=dI, dT=dT, rows=rows)
    return out
