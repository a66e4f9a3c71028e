"""world_size-2 (and 4) multi-process tests of the N>1 host logic on CPU with the gloo backend.

* the ring protocol the C driver runs (send to r-1 / receive from r+1, n-1 block hops, the column state
  travelling with its block plus one return hop home), driven by the library's own schedule function
  infcl_ring_block, with per-step tile math from the oracle -- results must equal the oracle's direct forward;
* the NCCL unique-id bootstrap used by RingComm (rank 0 creates, torch.distributed broadcasts);
* bench.py's max-over-ranks timing reduction.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _ring_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        import oracle
        from oracle import infonce as O
        from paper_2410_17243_b200 import _lib as L
        from synth import make_features, shard
        lib = L.lib()
        b, d, s = 64 * world, 16, 14.2857
        I, T = make_features(b, d, seed=11)
        Ii, Ti = shard(I, rank, world), shard(T, rank, world)
        bs = b // world
        held = Ti.clone()
        held_c = torch.full((bs,), -float("inf"), dtype=torch.float64)
        r = np.full(bs, -np.inf)
        diag = None
        for step in range(world):
            k = lib.infcl_ring_block(rank, world, step)
            assert torch.equal(held, shard(T, k, world))  # we hold exactly the block the schedule names
            X = O.similarity(Ii, held, s)
            r = O.merge_lse(r, O.tile_lse(X))
            held_c = torch.from_numpy(O.merge_lse(held_c.numpy(), O.tile_lse(X.T)))
            if k == rank:
                diag = np.diag(X).copy()
            send_to, recv_from = (rank - 1) % world, (rank + 1) % world
            nxt_c = torch.empty_like(held_c)
            ops = [dist.P2POp(dist.isend, held_c, send_to), dist.P2POp(dist.irecv, nxt_c, recv_from)]
            if step + 1 < world:
                nxt = torch.empty_like(held)
                ops += [dist.P2POp(dist.isend, held, send_to), dist.P2POp(dist.irecv, nxt, recv_from)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            held_c = nxt_c
            if step + 1 < world:
                held = nxt
        c = held_c.numpy()  # after the return hop our own block's column state is home
        part = torch.tensor([float(np.sum(r - diag) + np.sum(c - diag))], dtype=torch.float64)
        dist.all_reduce(part)
        loss = part.item() / (2 * b)
        ref = oracle.forward(I, T, s)
        sl = slice(rank * bs, (rank + 1) * bs)
        ok = (abs(loss - ref["loss"]) < 1e-12 and np.allclose(r, ref["r"][sl], atol=1e-12)
              and np.allclose(c, ref["c"][sl], atol=1e-12))
        q.put((rank, bool(ok), loss, ref["loss"]))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, repr(e), None))
    finally:
        dist.destroy_process_group()


def _run(target, world, timeout=180):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=timeout) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_ring_protocol_gloo(world):
    res = _run(_ring_worker, world)
    assert all(ok for _, ok, _, _ in res), res


def _uid_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        import ctypes
        from paper_2410_17243_b200 import _lib as L
        uid = torch.zeros(128, dtype=torch.uint8)
        status = 0
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            status = L.lib().infcl_get_unique_id(ctypes.cast(buf, ctypes.c_void_p))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        dist.broadcast(uid, src=0)
        q.put((rank, status, bytes(uid.tolist())))
    finally:
        dist.destroy_process_group()


def test_unique_id_bootstrap_gloo():
    res = _run(_uid_worker, 2, timeout=120)
    if res[0][1] == 5:
        pytest.skip("libnccl.so.2 not loadable on this host")
    assert res[0][1] == 0
    assert res[0][2] == res[1][2] and any(res[0][2])


def _bench_reduce_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        import bench
        q.put((rank, bench.max_over_ranks(float(rank + 1) * 1.5)))
    finally:
        dist.destroy_process_group()


def test_bench_max_over_ranks_gloo():
    res = _run(_bench_reduce_worker, 2, timeout=120)
    assert res == [(0, 3.0), (1, 3.0)]


def _comm_sum_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        from types import SimpleNamespace
        from paper_2410_17243_b200.loss import comm_sum
        sub = [dist.new_group([0, 1]), dist.new_group([2, 3])]  # every rank creates every group
        mine = sub[rank // 2]
        x = torch.tensor(float(rank + 1), dtype=torch.float64)
        local = comm_sum(x.clone(), None)  # local loss in a multi-rank job: no reduction
        one = comm_sum(x.clone(), SimpleNamespace(world=1, group=None))
        ring = comm_sum(x.clone(), SimpleNamespace(world=2, group=mine))  # ring on a subgroup: that group only
        q.put((rank, float(local), float(one), float(ring)))
    finally:
        dist.destroy_process_group()


def test_grad_scale_reduction_scope_gloo():
    """g dL/ds partials are summed over the loss's own ring group only -- not over the default group
    when the loss is local (comm None / world 1), and over a subgroup when the ring spans one."""
    res = _run(_comm_sum_worker, 4, timeout=120)
    assert res == [(0, 1.0, 1.0, 3.0), (1, 2.0, 2.0, 3.0), (2, 3.0, 3.0, 7.0), (3, 4.0, 4.0, 7.0)]
