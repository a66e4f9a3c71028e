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


def _worker(rank, world, port, b, d, s, dtype_name, outdir):
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


@pytest.mark.parametrize("b,d,world,dtype_name", [(2 * 2048, 512, 2, "bf16"), (3 * 700, 64, 3, "bf16"),
                                                  (4 * 1500, 128, 4, "bf16"), (2 * 320, 64, 2, "fp32")])
def test_ipc_ring_multiprocess(tmp_path, b, d, world, dtype_name):
    import oracle
    from synth import make_features
    s = 14.2857
    mp.start_processes(_worker, args=(world, _free_port(), b, d, s, dtype_name, str(tmp_path)), nprocs=world,
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
