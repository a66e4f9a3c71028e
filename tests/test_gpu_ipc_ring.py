"""Multi-process ring on ONE GPU through the IPC transport (include/infcl.h, INFCL_TRANSPORT_IPC).

world processes (gloo process group for the handle exchange, all ranks on cuda:0) each run infcl_forward /
infcl_backward on their own shard; the blocks, column states and LSE vectors travel by copy-engine writes into
the neighbour's receive region, synchronised by stream memory operations -- the same host schedule and
counters as on a multi-GPU box, with real inter-process concurrency.  Rank results are gathered and compared
with the fp64 oracle on the whole batch (north-star gates).  Two iterations check that the fill / release /
all-reduce counters carry across calls.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, b, d, s, dtype_name, outdir, fused=False):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    if fused:  # the fused backward ring (travelling dT partials) at these small shards too
        os.environ["INFCL_GC_MIN_ROWS"] = "0"
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_17243_b200 import loss as K
        from synth import make_features, shard
        torch.cuda.set_device(0)
        dt = torch.float32 if dtype_name == "fp32" else torch.bfloat16
        I, T = make_features(b, d, seed=5, dist="paired", dtype=dt)
        Ii, Ti = shard(I, rank, world).cuda(), shard(T, rank, world).cuda()
        comm = K.RingComm(transport="ipc", max_b=b, max_d=d, dtype=dt)
        g = torch.tensor(1.0, device="cuda")
        for it in range(2):
            loss, r, c, dg = K.infcl_forward(Ii, Ti, b, s, rank, world, comm)
            dI, dT = K.infcl_backward(Ii, Ti, b, s, r, c, dg, g, rank, world, comm)
            torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), loss=loss.item(), r=r.cpu().numpy(), c=c.cpu().numpy(),
                 dI=dI.cpu().numpy(), dT=dT.cpu().numpy())
        dist.barrier()
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("b,d,world,dtype_name,fused", [(2 * 2048, 512, 2, "bf16", False), (3 * 700, 64, 3, "bf16", False),
                                                        (4 * 1500, 128, 4, "bf16", False), (2 * 320, 64, 2, "fp32", False),
                                                        (8 * 520, 64, 8, "bf16", False), (2 * 2048, 512, 2, "bf16", True),
                                                        (3 * 700, 64, 3, "bf16", True), (8 * 520, 64, 8, "bf16", True),
                                                        (4 * 1500, 768, 4, "bf16", True)])
def test_ipc_ring_multiprocess(tmp_path, b, d, world, dtype_name, fused):
    """fused: the single-pass backward ring whose dT partials travel (forced at these small shards; the default
    uses it from 16K rows per rank); otherwise the two-pass backward ring."""
    import oracle
    from synth import make_features
    s = 14.2857
    mp.start_processes(_worker, args=(world, _free_port(), b, d, s, dtype_name, str(tmp_path), fused), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"rank{q}.npz") for q in range(world)]
    I, T = make_features(b, d, seed=5, dist="paired", dtype=torch.float32 if dtype_name == "fp32" else torch.bfloat16)
    ref = oracle.forward(I, T, s)
    rdI, rdT = oracle.backward(I, T, s, 1.0, ref["r"], ref["c"])
    for p in parts:  # the all-reduced loss is identical on every rank
        assert float(p["loss"]) == float(parts[0]["loss"])
    assert abs(float(parts[0]["loss"]) - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    r = np.concatenate([p["r"] for p in parts])
    c = np.concatenate([p["c"] for p in parts])
    assert np.abs(r - ref["r"]).max() <= 2e-3
    assert np.abs(c - ref["c"]).max() <= 2e-3
    dI = np.concatenate([p["dI"] for p in parts])
    dT = np.concatenate([p["dT"] for p in parts])
    for got, want in ((dI, rdI), (dT, rdT)):
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-3


def _worker_onehot(rank, world, port, b, d, K_, s, outdir):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_17243_b200 import loss as K
        from synth import make_onehot_device
        torch.cuda.set_device(0)
        bs = b // world
        Id, Td = make_onehot_device(b, d, K_, "cuda")
        Ii, Ti = Id[rank * bs:(rank + 1) * bs].contiguous(), Td[rank * bs:(rank + 1) * bs].contiguous()
        del Id, Td
        comm = K.RingComm(transport="ipc", max_b=b, max_d=d)
        loss, r, c, dg = K.infcl_forward(Ii, Ti, b, s, rank, world, comm)
        dI, dT = K.infcl_backward(Ii, Ti, b, s, r, c, dg, torch.tensor(1.0, device="cuda"), rank, world, comm)
        torch.cuda.synchronize()
        rows = np.array([0, 1, 127, 128, 4095, bs // 2, bs - 129, bs - 1])
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), loss=loss.item(), rmax=(r - r.mean()).abs().max().item(),
                 r0=r[0].item(), c0=c[0].item(), cmax=(c - c.mean()).abs().max().item(), rows=rows + rank * bs,
                 dI=dI[rows].cpu().numpy(), dT=dT[rows].cpu().numpy())
        dist.barrier()
        comm.close()
    finally:
        dist.destroy_process_group()


def test_ipc_ring_cfg3_onehot_closed_form(tmp_path):
    """cfg3's batch (b = 262144, d = 768) as a 2-process IPC ring on one GPU (b_s = 131072: 201-MB blocks in
    the receive slots), checked against the one-hot closed form (oracle.onehot_closed_form; exact at any b)."""
    b, d, K_, s, world = 262144, 768, 512, 1.0, 2
    mp.start_processes(_worker_onehot, args=(world, _free_port(), b, d, K_, s, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"rank{q}.npz") for q in range(world)]
    m = b // K_
    s32 = float(np.float32(s))
    lam = float(np.log(m * np.exp(np.float32(s)) + (b - m)))
    p, q = np.exp(s32 - lam), np.exp(-lam)
    for part in parts:
        assert abs(float(part["loss"]) - (lam - s32)) <= 1e-4 * abs(lam - s32)
        assert abs(float(part["r0"]) - lam) <= 2e-3 and abs(float(part["c0"]) - lam) <= 2e-3
        assert float(part["rmax"]) <= 2e-3 and float(part["cmax"]) <= 2e-3
        rows = part["rows"]
        want = np.zeros((len(rows), d))
        want[:, :K_] = s32 / b * m * q
        want[np.arange(len(rows)), rows % K_] = s32 / b * (m * p - 1.0)
        for got in (part["dI"], part["dT"]):
            assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-3


def _worker_ntxent(rank, world, port, b, d, s, outdir):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_17243_b200 import loss as K
        from synth import make_features, shard
        torch.cuda.set_device(0)
        A, B = make_features(b, d, seed=6, dist="paired")
        Ai, Bi = shard(A, rank, world).cuda(), shard(B, rank, world).cuda()
        comm = K.RingComm(transport="ipc", max_b=b, max_d=d)
        g = torch.tensor(0.5, device="cuda")
        for it in range(2):
            loss, la, lb, pos = K.ntxent_forward(Ai, Bi, b, s, rank, world, comm)
            dA, dB = K.ntxent_backward(Ai, Bi, b, s, la, lb, pos, g, rank, world, comm)
            torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), loss=loss.item(), la=la.cpu().numpy(), lb=lb.cpu().numpy(),
                 dA=dA.cpu().numpy(), dB=dB.cpu().numpy())
        dist.barrier()
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("b,d,world", [(2 * 1024, 256, 2), (3 * 520, 64, 3)])
def test_ipc_ring_ntxent(tmp_path, b, d, world):
    """NT-Xent as a world-process ring: the (B, B) and (A, A) self-similarity rings and the
    (A, B) ring per forward, four backward rings; gathered results against oracle.ntxent at north-star gates."""
    from oracle import ntxent as N
    from synth import make_features
    s = 14.2857
    mp.start_processes(_worker_ntxent, args=(world, _free_port(), b, d, s, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"rank{q}.npz") for q in range(world)]
    A, B = make_features(b, d, seed=6, dist="paired")
    ref = N.forward(A, B, s)
    rdA, rdB = N.backward(A, B, s, 0.5)
    for p in parts:
        assert float(p["loss"]) == float(parts[0]["loss"])
    assert abs(float(parts[0]["loss"]) - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    assert np.abs(np.concatenate([p["la"] for p in parts]) - ref["r_a"]).max() <= 2e-3
    assert np.abs(np.concatenate([p["lb"] for p in parts]) - ref["r_b"]).max() <= 2e-3
    for key, want in (("dA", rdA), ("dB", rdB)):
        got = np.concatenate([p[key] for p in parts])
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-3
