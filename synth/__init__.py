"""Seeded synthetic feature generators shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no similarity, no LSE, no gradient): it only draws
L2-normalised feature rows shaped like CLIP image/text embeddings and rounds them to the storage dtype.
Recipe:

* Row ``g`` of a global batch draws ``N(0, 1)^d`` from a counter-based Philox stream keyed by
  ``(seed, stream_id, g // BLOCK)`` so a row's content never depends on the world size ``n``.
* ``independent``: image and text rows come from independent streams ("random pairs").
* ``paired``: ``T_g = normalise(I_g + sigma * eps_g)`` (mean cosine ~0.71 at sigma=1): trained positives.
* ``identical``: every image and text row is the same unit vector (closed form L = log b).
* ``onehot``: ``I_g = T_g = e_{g mod K}`` (closed form, usable at any b).
* ``codebook``: rows are drawn from K random unit codewords (closed form via the K x K Gram matrix).
* Rows are normalised in fp32, then rounded to bf16 by round-to-nearest-even (``torch.Tensor.to``).
"""
from __future__ import annotations

import numpy as np
import torch

BLOCK = 4096
_STREAM_IMAGE = 1
_STREAM_TEXT = 2
_STREAM_NOISE = 3
_STREAM_CODES = 4


def _normal_rows(seed: int, stream: int, row0: int, rows: int, d: int) -> np.ndarray:
    """fp32 N(0,1) rows [row0, row0+rows) of a (seed, stream) counter-based stream, independent of chunking."""
    out = np.empty((rows, d), dtype=np.float32)
    g = row0
    while g < row0 + rows:
        blk = g // BLOCK
        start = blk * BLOCK
        take = min(row0 + rows, start + BLOCK) - g
        bitgen = np.random.Philox(key=np.array([seed & 0xFFFFFFFFFFFFFFFF, (stream << 40) | blk], dtype=np.uint64))
        rng = np.random.Generator(bitgen)
        # draw the whole block prefix up to the last row we need so row content is position-stable
        need = g - start + take
        blkvals = rng.standard_normal((need, d), dtype=np.float32)
        out[g - row0:g - row0 + take] = blkvals[g - start:]
        g += take
    return out


def _normalise(x: np.ndarray) -> np.ndarray:
    n = np.sqrt((x.astype(np.float32) ** 2).sum(axis=1, keepdims=True, dtype=np.float32))
    n[n == 0] = 1.0
    return (x / n).astype(np.float32)


def _to_dtype(x: np.ndarray, dtype: torch.dtype) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(dtype) if dtype != torch.float32 else t


def make_features(b: int, d: int, seed: int = 0, dist: str = "independent", dtype: torch.dtype = torch.bfloat16,
                  row0: int = 0, rows: int | None = None, sigma: float = 1.0, K: int = 32):
    """Return (I, T) CPU tensors of global rows [row0, row0+rows) of a batch of size b, feature dim d.

    The global batch size b only matters for the structured distributions; rows are position-stable.
    """
    rows = b - row0 if rows is None else rows
    if dist == "independent":
        I = _normalise(_normal_rows(seed, _STREAM_IMAGE, row0, rows, d))
        T = _normalise(_normal_rows(seed, _STREAM_TEXT, row0, rows, d))
    elif dist == "paired":
        I = _normalise(_normal_rows(seed, _STREAM_IMAGE, row0, rows, d))
        eps = _normalise(_normal_rows(seed, _STREAM_NOISE, row0, rows, d))
        T = _normalise(I + np.float32(sigma) * eps)
    elif dist == "identical":
        u = _normalise(_normal_rows(seed, _STREAM_IMAGE, 0, 1, d))
        I = np.repeat(u, rows, axis=0)
        T = I.copy()
    elif dist == "onehot":
        if K > d:
            raise ValueError("onehot needs K <= d")
        idx = (np.arange(row0, row0 + rows) % K)
        I = np.zeros((rows, d), dtype=np.float32)
        I[np.arange(rows), idx] = 1.0
        T = I.copy()
    elif dist == "codebook":
        codes_i = _normalise(_normal_rows(seed, _STREAM_CODES, 0, K, d))
        codes_t = _normalise(_normal_rows(seed + 1, _STREAM_CODES, 0, K, d))
        ai, at = codebook_assignment(b, K, seed)
        I = codes_i[ai[row0:row0 + rows]]
        T = codes_t[at[row0:row0 + rows]]
    else:
        raise ValueError(f"unknown dist {dist!r}")
    return _to_dtype(I, dtype), _to_dtype(T, dtype)


def codebook_assignment(b: int, K: int, seed: int):
    """Code index per global row for images and texts (deterministic, position-stable)."""
    g = np.arange(b, dtype=np.int64)
    ai = (g * 2654435761 + seed) % K
    at = (g * 40503 + 7 * seed + 3) % K
    return ai, at


def codebook_vectors(d: int, K: int, seed: int, dtype: torch.dtype = torch.bfloat16):
    """The K image and K text codewords after storage rounding (what the GPU actually sees)."""
    ci = _to_dtype(_normalise(_normal_rows(seed, _STREAM_CODES, 0, K, d)), dtype)
    ct = _to_dtype(_normalise(_normal_rows(seed + 1, _STREAM_CODES, 0, K, d)), dtype)
    return ci, ct


def shard(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Rows [rank*b_s, (rank+1)*b_s) of a global batch (paper P:209)."""
    b = x.shape[0]
    if b % world:
        raise ValueError(f"b={b} not divisible by world={world}")
    bs = b // world
    return x[rank * bs:(rank + 1) * bs]


def make_features_device(b: int, d: int, seed: int, device, dtype=torch.bfloat16, dist: str = "independent",
                         sigma: float = 1.0):
    """Fast on-device generator for benchmark- and paper-sized batches (same distributions, different stream):
    torch's CUDA Philox, fp32 normalisation, RNE rounding.  dist "independent" or "paired"
    (T = normalise(I + sigma * normalise(eps)), as make_features)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    I = torch.nn.functional.normalize(torch.randn(b, d, device=device, generator=gen, dtype=torch.float32), dim=1)
    if dist == "independent":
        T = torch.randn(b, d, device=device, generator=gen, dtype=torch.float32)
    elif dist == "paired":
        T = torch.randn(b, d, device=device, generator=gen, dtype=torch.float32)
        T = I + sigma * torch.nn.functional.normalize(T, dim=1)
    else:
        raise ValueError(f"unknown dist {dist!r}")
    T = torch.nn.functional.normalize(T, dim=1).to(dtype)
    return I.to(dtype), T


def make_onehot_device(b: int, d: int, K: int, device, dtype=torch.bfloat16):
    """The ``onehot`` distribution built directly on a device (same values as make_features(..., dist="onehot"))."""
    I = torch.zeros(b, d, device=device, dtype=dtype)
    idx = torch.arange(b, device=device) % K
    I[torch.arange(b, device=device), idx] = 1
    return I, I.clone()
