"""Full-size parity (SURVEY.md 8(c) "large-b protocol"), in the launch configuration bench.py times.

* cfg2 (b=65536, d=512, bf16, 1 GPU) on random paired inputs: every r_i, c_j and the loss against the exact fp64
  oracle streamed over row chunks, and 256 stratified gradient rows of dI and dT against the exact fp64 rows
  (oracle.sampled_row_grads with the oracle's own r, c).
* cfg3 (b=262144, d=768) at n=1, and cfg4's / cfg5's per-rank workloads (b = 1M / 4M, d=768, through the 8-rank
  virtual ring: b_s = 131072 / 524288) on structured inputs with closed forms (one-hot classes, codebook), exact
  at any b.
* cfg3 on random paired inputs at n = 1 and through the 8-rank virtual ring (b_s = 32768), and cfg4 (b = 1M)
  through the 8-rank virtual ring, by the sampled
  protocol: exact r, c at 256 stratified rows / columns, loss from the GPU's r, c and the exact diagonal, and 256
  exact gradient rows of dI and dT.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import make_features, make_onehot_device, codebook_assignment, codebook_vectors
from paper_2410_17243_b200 import loss as K

pytestmark = pytest.mark.gpu

S = 14.2857


def rel_norm(got, ref):
    return np.linalg.norm(np.asarray(got, np.float64) - ref) / np.linalg.norm(ref)


def stratified_rows(b, n=256, seed=0):
    """Rows spread over 128-row tiles and positions within a tile (first/last rows of tiles included)."""
    rng = np.random.default_rng(seed)
    rows = set([0, 1, 63, 64, 127, 128, b - 1, b - 128, b - 129])
    while len(rows) < n:
        rows.add(int(rng.integers(0, b)))
    return np.array(sorted(rows))


def test_cfg2_full_size_random_paired():
    b, d = 65536, 512
    I, T = make_features(b, d, seed=1, dist="paired")
    Id, Td = I.cuda(), T.cuda()
    loss, r, c, dg = K.infcl_forward(Id, Td, b, S)
    dI, dT = K.infcl_backward(Id, Td, b, S, r, c, dg, torch.tensor(1.0, device="cuda"))
    torch.cuda.synchronize()
    ref = oracle.streamed_forward(I, T, S, chunk=512, workers=8)
    assert abs(loss.item() - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    assert np.abs(r.cpu().numpy() - ref["r"]).max() <= 2e-3
    assert np.abs(c.cpu().numpy() - ref["c"]).max() <= 2e-3
    assert np.abs(dg.cpu().numpy() - ref["diag"]).max() <= 2e-3
    rows = stratified_rows(b)
    rdI = oracle.sampled_row_grads(I, T, S, ref["r"], ref["c"], rows)
    rdT = oracle.sampled_row_grads(T, I, S, ref["c"], ref["r"], rows)
    assert rel_norm(dI.cpu().numpy()[rows], rdI) <= 2e-3
    assert rel_norm(dT.cpu().numpy()[rows], rdT) <= 2e-3
    # O(bd) identity over ALL rows: sum <dI_i, I_i> = sum <dT_j, T_j> (= s dL/ds)
    a = (dI.double() * Id.double()).sum().item()
    bb = (dT.double() * Td.double()).sum().item()
    assert abs(a - bb) <= 1e-3 * max(abs(a), abs(bb), 1e-12)


@pytest.mark.parametrize("b,d,world", [(262144, 768, 1), (1048576, 768, 8), (4194304, 768, 8)])
def test_large_onehot_closed_form(b, d, world):
    """One-hot classes: r = c = log(m e^s + b - m), L = that - s, closed-form gradients (oracle.onehot_closed_form).
    world=8 runs cfg4's / cfg5's exact per-rank shards (b_s = 131072 / 524288) through the virtual 8-rank ring
    schedule (cfg5: the paper's 4M headline batch, ~60 GB and ~80 s on one B200)."""
    K_ = 512
    s = 1.0  # well-conditioned gradient (DESIGN.md Tolerances)
    Id, Td = make_onehot_device(b, d, K_, "cuda")
    if world == 1:
        loss, r, c, dg = K.infcl_forward(Id, Td, b, s)
        dI, dT = K.infcl_backward(Id, Td, b, s, r, c, dg, torch.tensor(1.0, device="cuda"))
    else:
        loss, r, c, dg = K.infcl_forward_virtual(Id, Td, s, world)
        dI, dT = K.infcl_backward_virtual(Id, Td, s, world, r, c, dg, torch.tensor(1.0, device="cuda"))
    torch.cuda.synchronize()
    m = b // K_
    lam = float(np.log(m * np.exp(np.float32(s)) + (b - m)))
    assert abs(loss.item() - (lam - float(np.float32(s)))) <= 1e-4 * abs(lam - s)
    assert (r - lam).abs().max().item() <= 2e-3 and (c - lam).abs().max().item() <= 2e-3
    rows = stratified_rows(b, 64)
    # closed form per row (oracle.onehot_closed_form, evaluated for the sampled rows only): dI_i = s/b [ (m p - 1) e_k + m q sum_{k' != k} e_k' ],  p = e^{s - lam}, q = e^{-lam}
    p = np.exp(np.float32(s) - lam)
    q = np.exp(-lam)
    s32 = float(np.float32(s))
    want = np.zeros((len(rows), d))
    want[:, :K_] = s32 / b * m * q
    want[np.arange(len(rows)), rows % K_] = s32 / b * (m * p - 1.0)
    assert rel_norm(dI.cpu().numpy()[rows], want) <= 2e-3
    assert rel_norm(dT.cpu().numpy()[rows], want) <= 2e-3


def test_cfg3_codebook_closed_form():
    """Codebook inputs (K random unit codewords per side): exact r, c, loss and gradient rows at b = 262144."""
    b, d, K_, seed = 262144, 768, 256, 5
    I, T = make_features(b, d, seed=seed, dist="codebook", K=K_)
    ci, ct = codebook_vectors(d, K_, seed)
    ai, at = codebook_assignment(b, K_, seed)
    Id, Td = I.cuda(), T.cuda()
    del I, T
    loss, r, c, dg = K.infcl_forward(Id, Td, b, S)
    dI, dT = K.infcl_backward(Id, Td, b, S, r, c, dg, torch.tensor(1.0, device="cuda"))
    torch.cuda.synchronize()
    rows = stratified_rows(b, 128)
    cf = oracle.codebook_closed_form(ci, ct, ai, at, S, rows=rows)
    assert abs(loss.item() - cf["loss"]) <= 1e-4 * abs(cf["loss"])
    assert np.abs(r.cpu().numpy() - cf["r"]).max() <= 2e-3
    assert np.abs(c.cpu().numpy() - cf["c"]).max() <= 2e-3
    assert rel_norm(dI.cpu().numpy()[rows], cf["dI"]) <= 2e-3
    assert rel_norm(dT.cpu().numpy()[rows], cf["dT"]) <= 2e-3


def e2e_boundaries(b):
    """Row / column boundaries of infcl_loss_grad_host's pipelined schedule (api.cu: forward I chunks at
    sixteenths {1, 4, 10}, the hybrid backward's fused / two-pass split at 8, dT-pass chunks at {6, 11, 15},
    128-row aligned; T split at 3/8, 256 aligned)."""
    at16 = [min(b, (b * e // 16 + 127) // 128 * 128) for e in (1, 4, 6, 8, 10, 11, 15)]
    return at16 + [min(b, (b * 3 // 8 + 255) // 256 * 256)]


@pytest.mark.parametrize("b,d", [(32768, 128), (40000, 64), (65536, 512)])
def test_e2e_host_entry_chunked(b, d):
    """Host end-to-end entry at sizes where it pipelines PCIe copies against row chunks of the forward and of
    the dT pass (b = 40000 leaves ragged chunks; b = 65536, d = 512 is cfg2, the shape bench.py's e2e times):
    the loss against the streamed fp64 oracle and stratified gradient rows plus
    the rows on both sides of every chunk / piece boundary against the exact fp64 rows."""
    I, T = make_features(b, d, seed=11, dist="paired")
    loss, dI, dT = K.infcl_loss_grad_host(I.pin_memory(), T.pin_memory(), S)
    ref = oracle.streamed_forward(I, T, S, chunk=512, workers=8)
    assert abs(loss.item() - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    rows = stratified_rows(b, 96)
    rows = np.unique(np.concatenate([rows, [x for c in e2e_boundaries(b) for x in (c - 1, c)]]))
    rows = rows[(rows >= 0) & (rows < b)]
    rdI = oracle.sampled_row_grads(I, T, S, ref["r"], ref["c"], rows)
    rdT = oracle.sampled_row_grads(T, I, S, ref["c"], ref["r"], rows)
    assert rel_norm(dI.numpy()[rows], rdI) <= 2e-3
    assert rel_norm(dT.numpy()[rows], rdT) <= 2e-3


@pytest.mark.parametrize("b,d", [(256 * 74 + 300, 64), (256 * 74 * 2 + 4000, 64), (256 * 74 + 300, 512)])
def test_wide_forward_waves_and_tail(b, d):
    """Row counts that give the wide forward (256 rows per pair) one / two full waves of 74 pairs plus a ragged
    tail split across pairs (Sched tail ranges, row-partial tail slots): every r_j, c_j and the loss exact
    against the streamed fp64 oracle, plus the backward's sampled gradient rows.  d = 512 runs the resident-A
    variant (segment changes reload the stationary rows inside the ring transactions); d = 64 streams A."""
    I, T = make_features(b, d, seed=23, dist="paired")
    Id, Td = I.cuda(), T.cuda()
    loss, r, c, dg = K.infcl_forward(Id, Td, b, S)
    dI, dT = K.infcl_backward(Id, Td, b, S, r, c, dg, torch.tensor(1.0, device="cuda"))
    torch.cuda.synchronize()
    ref = oracle.streamed_forward(I, T, S, chunk=512, workers=8)
    assert abs(loss.item() - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    assert np.abs(r.cpu().numpy() - ref["r"]).max() <= 2e-3
    assert np.abs(c.cpu().numpy() - ref["c"]).max() <= 2e-3
    assert np.abs(dg.cpu().numpy() - ref["diag"]).max() <= 2e-3
    rows = stratified_rows(b, 64)
    rows = np.unique(np.concatenate([rows, [256 * 74 - 1, 256 * 74, b - 300, b - 1]]))
    rows = rows[rows < b]
    assert rel_norm(dI.cpu().numpy()[rows], oracle.sampled_row_grads(I, T, S, ref["r"], ref["c"], rows)) <= 2e-3
    assert rel_norm(dT.cpu().numpy()[rows], oracle.sampled_row_grads(T, I, S, ref["c"], ref["r"], rows)) <= 2e-3


@pytest.mark.parametrize("b,world", [(262144, 1), (262144, 8), (1048576, 8)])
def test_cfg3_random_sampled_protocol(b, world):
    """cfg3 (b = 262144, d = 768) on RANDOM paired inputs by the large-b protocol: exact fp64 r_i
    for 256 stratified rows and c_j for 256 stratified columns (O(b d) each), the loss recomputed from the GPU's
    r, c and the exact diagonal, and 256 gradient rows of dI and dT from exact P (oracle r at those rows) and the
    GPU's c (resp. r).  world = 8 runs cfg3's / cfg4's n = 8 per-rank shapes (b_s = 32768 / 131072) through the
    virtual ring."""
    d = 768
    I, T = make_features(b, d, seed=4, dist="paired")
    Id, Td = I.cuda(), T.cuda()
    g = torch.tensor(1.0, device="cuda")
    if world == 1:
        loss, r, c, dg = K.infcl_forward(Id, Td, b, S)
        dI, dT = K.infcl_backward(Id, Td, b, S, r, c, dg, g)
    else:
        loss, r, c, dg = K.infcl_forward_virtual(Id, Td, S, world)
        dI, dT = K.infcl_backward_virtual(Id, Td, S, world, r, c, dg, g)
    torch.cuda.synchronize()
    r, c, dg = r.cpu().numpy(), c.cpu().numpy(), dg.cpu().numpy()
    rows = stratified_rows(b, 256, seed=1)
    cols = stratified_rows(b, 256, seed=2)
    I64, T64 = oracle.to_f64(I), oracle.to_f64(T)
    s32 = float(np.float32(S))
    r_ex = oracle.tile_lse(s32 * (I64[rows] @ T64.T))
    c_ex = oracle.tile_lse(s32 * (T64[cols] @ I64.T))
    assert np.abs(r[rows] - r_ex).max() <= 2e-3
    assert np.abs(c[cols] - c_ex).max() <= 2e-3
    diag_ex = s32 * np.einsum("ij,ij->i", I64, T64)
    assert np.abs(dg - diag_ex).max() <= 2e-3
    L = 0.5 * (np.sum(r.astype(np.float64) - diag_ex) + np.sum(c.astype(np.float64) - diag_ex)) / b
    assert abs(loss.item() - L) <= 1e-4 * abs(L)
    r_rows = np.array(r, dtype=np.float64)
    r_rows[rows] = r_ex
    rdI = oracle.sampled_row_grads(I, T, S, r_rows, c, rows)
    assert rel_norm(dI.cpu().numpy()[rows], rdI) <= 2e-3
    c_rows = np.array(c, dtype=np.float64)
    c_rows[cols] = c_ex
    rdT = oracle.sampled_row_grads(T, I, S, c_rows, r, cols)
    assert rel_norm(dT.cpu().numpy()[cols], rdT) <= 2e-3


def test_cfg5_random_sampled_protocol():
    """cfg5 -- the paper's 4M headline batch (Table 2; b = 4194304, d = 768) -- on RANDOM paired inputs at
    s = 14.2857, at its exact per-rank shape (b_s = 524288) through the virtual 8-rank ring (Alg.1 / Alg.3,
    P:539-558), by the large-b protocol: exact fp64 r_i at 256 stratified rows and c_j at 256
    columns (streamed over all 4M columns), the diagonal, the loss recomputed from the GPU's r, c and the exact
    diagonal, 256 exact gradient rows of dI and dT (oracle.streamed_row_grads), and the O(b d) identity
    sum <dI, I> = sum <dT, T>.  Inputs are generated on the device (synth.make_features_device, paired) and
    widened on the host chunk by chunk."""
    from synth import make_features_device
    b, d, world = 4194304, 768, 8
    Id, Td = make_features_device(b, d, seed=5, device="cuda", dist="paired")
    g = torch.tensor(1.0, device="cuda")
    loss, r, c, dg = K.infcl_forward_virtual(Id, Td, S, world)
    dI, dT = K.infcl_backward_virtual(Id, Td, S, world, r, c, dg, g)
    torch.cuda.synchronize()
    ident_i = sum((dI[j:j + 262144].double() * Id[j:j + 262144].double()).sum().item() for j in range(0, b, 262144))
    ident_t = sum((dT[j:j + 262144].double() * Td[j:j + 262144].double()).sum().item() for j in range(0, b, 262144))
    rows = stratified_rows(b, 256, seed=11)
    cols = stratified_rows(b, 256, seed=12)
    ridx = torch.from_numpy(rows).cuda()
    cidx = torch.from_numpy(cols).cuda()
    dI_rows, dT_cols = dI[ridx].cpu().numpy(), dT[cidx].cpu().numpy()
    del dI, dT
    r, c, dg = r.cpu().numpy(), c.cpu().numpy(), dg.cpu().numpy()
    I, T = Id.cpu(), Td.cpu()
    del Id, Td
    assert abs(ident_i - ident_t) <= 1e-3 * max(abs(ident_i), abs(ident_t))
    s32 = float(np.float32(S))
    r_ex = oracle.streamed_row_lse(I[rows], T, S)
    c_ex = oracle.streamed_row_lse(T[cols], I, S)
    assert np.abs(r[rows] - r_ex).max() <= 2e-3
    assert np.abs(c[cols] - c_ex).max() <= 2e-3
    diag_ex = np.concatenate([s32 * np.einsum("ij,ij->i", oracle.to_f64(I[j0:j0 + 262144]),
                                              oracle.to_f64(T[j0:j0 + 262144])) for j0 in range(0, b, 262144)])
    assert np.abs(dg - diag_ex).max() <= 2e-3
    L = 0.5 * (np.sum(r.astype(np.float64) - diag_ex) + np.sum(c.astype(np.float64) - diag_ex)) / b
    assert abs(loss.item() - L) <= 1e-4 * abs(L)
    c_all = c.astype(np.float64)
    c_all[cols] = c_ex
    r_all = r.astype(np.float64)
    r_all[rows] = r_ex
    want_i = oracle.streamed_row_grads(I[rows], T, S, r_ex, c_all, rows)
    want_t = oracle.streamed_row_grads(T[cols], I, S, c_ex, r_all, cols)
    assert rel_norm(dI_rows, want_i) <= 2e-3
    assert rel_norm(dT_cols, want_t) <= 2e-3
