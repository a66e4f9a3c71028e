"""Thin torch binding over the C ABI: device memory, streams and process groups only.

Every step of the loss runs in libinfcl.so; this module allocates caller-owned buffers (so
``torch.cuda.max_memory_allocated`` sees all of them), marshals pointers and the current stream, and wraps
the pair forward/backward as an ``autograd.Function``.  The names mirror include/infcl.h.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib as L

_DT = {torch.bfloat16: L.INFCL_BF16, torch.float32: L.INFCL_FP32}


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype not in _DT:
        raise TypeError(f"features must be bf16 or fp32, got {t.dtype}")
    return _DT[t.dtype]


def _check_features(I: torch.Tensor, T: torch.Tensor):
    if not (I.is_cuda and T.is_cuda):
        raise ValueError("infcl: features must be CUDA tensors (there is no CPU path)")
    if I.shape != T.shape or I.dim() != 2 or I.dtype != T.dtype:
        raise ValueError(f"infcl: shape/dtype mismatch I{tuple(I.shape)} {I.dtype} T{tuple(T.shape)} {T.dtype}")
    return I.contiguous(), T.contiguous()


def workspace_bytes(b: int, d: int, world: int = 1, dtype=torch.bfloat16, comm=None) -> int:
    return int(L.lib().infcl_comm_workspace_bytes(comm.handle if comm is not None else None, b, d, world,
                                                  _DT[dtype]))


def alloc_workspace(b: int, d: int, world: int, dtype, device, copies: int = 1, comm=None) -> torch.Tensor:
    n = workspace_bytes(b, d, world, dtype, comm) * copies
    return torch.empty(max(n, 256), dtype=torch.uint8, device=device)


class RingComm:
    """Ring communicator of the library for this process group (include/infcl.h), bootstrapped through
    torch.distributed.  transport="nccl": the library's own NCCL communicator (unique id broadcast);
    transport="ipc": copy-engine writes into the neighbours' receive regions over CUDA IPC peer mappings
    (handles all-gathered), sized for shards of up to max_b / world rows of max_d features."""

    def __init__(self, group=None, device=None, transport: str = "nccl", max_b: int | None = None,
                 max_d: int | None = None, dtype=torch.bfloat16):
        import torch.distributed as dist
        self.group = group  # the process group the ring (and every cross-rank reduction of this comm) spans
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.transport = transport
        dev = torch.cuda.current_device() if device is None else device
        self.handle = ctypes.c_void_p()
        if transport == "ipc":
            if max_b is None or max_d is None:
                raise ValueError("RingComm(transport='ipc') needs max_b and max_d to size the receive region")
            L.call("infcl_comm_init_ipc", ctypes.byref(self.handle), self.rank, self.world, dev, int(max_b),
                   int(max_d), _DT[dtype])
            buf = (ctypes.c_uint8 * 64)()
            L.call("infcl_comm_ipc_handle", self.handle, ctypes.cast(buf, ctypes.c_void_p))
            mine = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                mine = mine.cuda()
            allh = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(allh, mine, group=group)
            raw = b"".join(bytes(h.cpu().tolist()) for h in allh)
            hbuf = (ctypes.c_uint8 * len(raw)).from_buffer_copy(raw)
            st = L.lib().infcl_comm_ipc_connect(self.handle, ctypes.cast(hbuf, ctypes.c_void_p))
            detail = L.lib().infcl_last_error().decode(errors="replace") if st else ""

            def agree(status):  # collective outcome (MIN over ranks); also a barrier
                ok = torch.tensor([1 if status == 0 else 0], dtype=torch.int32)
                if dist.get_backend(group) == "nccl":
                    ok = ok.cuda()
                dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
                return int(ok.item()) == 1

            # every rank mapped every region before anyone writes into one
            if agree(st):
                st = L.lib().infcl_comm_ipc_selftest(self.handle, 10000)  # the ring's copy/write/wait paths
                detail = L.lib().infcl_last_error().decode(errors="replace") if st else ""
                if agree(st):
                    return
            self.close()
            raise L.InfclError(st or 4, "IPC ring setup", detail or "a peer rank failed to connect or self-test")
        if transport != "nccl":
            raise ValueError(f"unknown transport {transport!r}")
        uid = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            L.call("infcl_get_unique_id", ctypes.cast(buf, ctypes.c_void_p))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            uid = uid.cuda()
        dist.broadcast(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = bytes(uid.cpu().tolist())
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(raw)
        L.call("infcl_comm_init", ctypes.byref(self.handle), self.rank, self.world, ctypes.cast(idbuf, ctypes.c_void_p),
               dev)

    def region_bytes(self) -> int:
        """Device bytes the library owns for this communicator (the IPC receive region; 0 for NCCL)."""
        return int(L.lib().infcl_comm_ipc_region_bytes(self.handle)) if self.transport == "ipc" else 0

    def close(self):
        if self.handle:
            L.lib().infcl_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def infcl_forward(I_local, T_local, b: int, logit_scale: float, rank: int = 0, world: int = 1, comm=None,
                  workspace=None):
    """Returns (loss scalar tensor, row_lse r, col_lse c, diag x_ii) for this rank's rows (include/infcl.h)."""
    I_local, T_local = _check_features(I_local, T_local)
    bs, d = I_local.shape
    dev = I_local.device
    r = torch.empty(bs, device=dev, dtype=torch.float32)
    c = torch.empty_like(r)
    dg = torch.empty_like(r)
    loss = torch.empty((), device=dev, dtype=torch.float32)
    ws = workspace if workspace is not None else alloc_workspace(b, d, world, I_local.dtype, dev, comm=comm)
    L.call("infcl_forward", comm.handle if comm is not None else None, I_local.data_ptr(), T_local.data_ptr(),
           _dtype_code(I_local), b, d, float(logit_scale), rank, world, r.data_ptr(), c.data_ptr(), dg.data_ptr(),
           loss.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    return loss, r, c, dg


def infcl_backward(I_local, T_local, b: int, logit_scale: float, row_lse, col_lse, diag, grad_loss, rank: int = 0,
                   world: int = 1, comm=None, workspace=None):
    """Returns (dI, dT) fp32 for this rank's rows; grad_loss is a device scalar tensor."""
    I_local, T_local = _check_features(I_local, T_local)
    bs, d = I_local.shape
    dev = I_local.device
    dI = torch.empty(bs, d, device=dev, dtype=torch.float32)
    dT = torch.empty_like(dI)
    g = grad_loss.detach().to(device=dev, dtype=torch.float32).reshape(()).contiguous()
    ws = workspace if workspace is not None else alloc_workspace(b, d, world, I_local.dtype, dev, comm=comm)
    L.call("infcl_backward", comm.handle if comm is not None else None, I_local.data_ptr(), T_local.data_ptr(),
           _dtype_code(I_local), b, d, float(logit_scale), rank, world, row_lse.data_ptr(), col_lse.data_ptr(),
           diag.data_ptr(), g.data_ptr(), dI.data_ptr(), dT.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    return dI, dT


def ntxent_forward(A_local, B_local, b: int, logit_scale: float, rank: int = 0, world: int = 1, comm=None,
                   workspace=None):
    """NT-Xent (SimCLR) over the 2b views [A; B] (include/infcl.h infcl_ntxent_forward): returns (loss, lse_a,
    lse_b, pos) for this rank's examples; b = global number of examples."""
    A_local, B_local = _check_features(A_local, B_local)
    bs, d = A_local.shape
    dev = A_local.device
    la = torch.empty(bs, device=dev, dtype=torch.float32)
    lb = torch.empty_like(la)
    pos = torch.empty_like(la)
    loss = torch.empty((), device=dev, dtype=torch.float32)
    ws = workspace if workspace is not None else alloc_workspace(b, d, world, A_local.dtype, dev, comm=comm)
    L.call("infcl_ntxent_forward", comm.handle if comm is not None else None, A_local.data_ptr(), B_local.data_ptr(),
           _dtype_code(A_local), b, d, float(logit_scale), rank, world, la.data_ptr(), lb.data_ptr(), pos.data_ptr(),
           loss.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    return loss, la, lb, pos


def ntxent_backward(A_local, B_local, b: int, logit_scale: float, lse_a, lse_b, pos, grad_loss, rank: int = 0,
                    world: int = 1, comm=None, workspace=None):
    """Returns (dA, dB) fp32 = g dL/dA, g dL/dB of the NT-Xent loss for this rank's examples."""
    A_local, B_local = _check_features(A_local, B_local)
    bs, d = A_local.shape
    dev = A_local.device
    dA = torch.empty(bs, d, device=dev, dtype=torch.float32)
    dB = torch.empty_like(dA)
    g = grad_loss.detach().to(device=dev, dtype=torch.float32).reshape(()).contiguous()
    ws = workspace if workspace is not None else alloc_workspace(b, d, world, A_local.dtype, dev, comm=comm)
    L.call("infcl_ntxent_backward", comm.handle if comm is not None else None, A_local.data_ptr(), B_local.data_ptr(),
           _dtype_code(A_local), b, d, float(logit_scale), rank, world, lse_a.data_ptr(), lse_b.data_ptr(),
           pos.data_ptr(), g.data_ptr(), dA.data_ptr(), dB.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    return dA, dB


class _NTXentFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, A_local, B_local, b, logit_scale, rank, world, comm):
        loss, la, lb, pos = ntxent_forward(A_local, B_local, b, logit_scale, rank, world, comm)
        ctx.save_for_backward(A_local, B_local, la, lb, pos)
        ctx.meta = (b, logit_scale, rank, world, comm)
        return loss

    @staticmethod
    def backward(ctx, grad_out):
        A_local, B_local, la, lb, pos = ctx.saved_tensors
        b, s, rank, world, comm = ctx.meta
        dA, dB = ntxent_backward(A_local, B_local, b, s, la, lb, pos, grad_out, rank, world, comm)
        return dA.to(A_local.dtype), dB.to(B_local.dtype), None, None, None, None, None


def ntxent_loss(A_local: torch.Tensor, B_local: torch.Tensor, logit_scale: float, comm: "RingComm | None" = None):
    """Differentiable NT-Xent (SimCLR) loss over the global batch of view pairs (this rank's shards)."""
    world = comm.world if comm is not None else 1
    rank = comm.rank if comm is not None else 0
    return _NTXentFunction.apply(A_local, B_local, A_local.shape[0] * world, float(logit_scale), rank, world, comm)


def comm_sum(t: torch.Tensor, comm=None) -> torch.Tensor:
    """Sum a per-rank partial over the ranks of ``comm``'s ring, in place: a no-op for a local loss (comm None or
    world 1) -- never over an unrelated default process group (a DDP job computing a local loss must not add
    other ranks' partials) -- and over the comm's own group otherwise."""
    if comm is None or comm.world <= 1:
        return t
    import torch.distributed as dist
    dist.all_reduce(t, group=comm.group)
    return t


def infcl_grad_scale(I_local, dI_local, logit_scale: float, comm=None):
    """g * dL/ds (learnable temperature): sum_i <dI_i, I_i> / s over the global batch (include/infcl.h).
    The per-rank partial is summed over ``comm``'s ranks (the ring the loss was computed on), if any."""
    I_local = I_local.contiguous()
    dI_local = dI_local.contiguous()
    out = torch.empty((), device=I_local.device, dtype=torch.float64)
    L.call("infcl_grad_scale_partial", I_local.data_ptr(), dI_local.data_ptr(), _dtype_code(I_local),
           I_local.shape[0], I_local.shape[1], float(logit_scale), out.data_ptr(), _stream())
    return comm_sum(out, comm)


def infcl_forward_virtual(I, T, logit_scale: float, world: int):
    """Whole batch on one device, ring schedule over `world` logical ranks (test of the ring engine)."""
    I, T = _check_features(I, T)
    b, d = I.shape
    dev = I.device
    r = torch.empty(b, device=dev, dtype=torch.float32)
    c = torch.empty_like(r)
    dg = torch.empty_like(r)
    loss = torch.empty((), device=dev, dtype=torch.float32)
    ws = alloc_workspace(b, d, world, I.dtype, dev, copies=world)
    L.call("infcl_forward_virtual", I.data_ptr(), T.data_ptr(), _dtype_code(I), b, d, float(logit_scale), world,
           r.data_ptr(), c.data_ptr(), dg.data_ptr(), loss.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    return loss, r, c, dg


def infcl_backward_virtual(I, T, logit_scale: float, world: int, r, c, dg, grad_loss):
    I, T = _check_features(I, T)
    b, d = I.shape
    dev = I.device
    dI = torch.empty(b, d, device=dev, dtype=torch.float32)
    dT = torch.empty_like(dI)
    g = grad_loss.detach().to(device=dev, dtype=torch.float32).reshape(()).contiguous()
    ws = alloc_workspace(b, d, world, I.dtype, dev, copies=world)
    L.call("infcl_backward_virtual", I.data_ptr(), T.data_ptr(), _dtype_code(I), b, d, float(logit_scale), world,
           r.data_ptr(), c.data_ptr(), dg.data_ptr(), g.data_ptr(), dI.data_ptr(), dT.data_ptr(), ws.data_ptr(),
           ws.numel(), _stream())
    return dI, dT


def infcl_loss_grad_host(I_host: torch.Tensor, T_host: torch.Tensor, logit_scale: float, grad_loss: float = 1.0,
                         scratch: torch.Tensor | None = None, out=None):
    """End-to-end call with HOST tensors (copies inside the library call); returns (loss, dI, dT) on host.
    ``out`` = (loss, dI, dT) preallocated host tensors (pinned for full PCIe bandwidth) to reuse across calls."""
    b, d = I_host.shape
    dt = _dtype_code(I_host)
    n = int(L.lib().infcl_e2e_scratch_bytes(b, d, dt))
    if scratch is None or scratch.numel() < n:
        scratch = torch.empty(n, dtype=torch.uint8, device="cuda")
    if out is None:
        pin = I_host.is_pinned()
        dI = torch.empty(b, d, dtype=torch.float32, pin_memory=pin)
        dT = torch.empty_like(dI)
        loss = torch.empty((), dtype=torch.float32, pin_memory=pin)
    else:
        loss, dI, dT = out
    L.call("infcl_loss_grad_host", I_host.data_ptr(), T_host.data_ptr(), dt, b, d, float(logit_scale),
           float(grad_loss), loss.data_ptr(), dI.data_ptr(), dT.data_ptr(), scratch.data_ptr(), scratch.numel(),
           _stream())
    return loss, dI, dT


class _InfCLFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, I_local, T_local, scale_t, b, logit_scale, rank, world, comm):
        loss, r, c, dg = infcl_forward(I_local, T_local, b, logit_scale, rank, world, comm)
        ctx.save_for_backward(I_local, T_local, r, c, dg)
        ctx.meta = (b, logit_scale, rank, world, comm, scale_t is not None and scale_t.requires_grad)
        return loss

    @staticmethod
    def backward(ctx, grad_out):
        I_local, T_local, r, c, dg = ctx.saved_tensors
        b, s, rank, world, comm, want_ds = ctx.meta
        dI, dT = infcl_backward(I_local, T_local, b, s, r, c, dg, grad_out, rank, world, comm)
        ds = None
        if want_ds:  # g * dL/ds = sum_i <dI_i, I_i> / s over the global batch (include/infcl.h)
            ds = infcl_grad_scale(I_local, dI, s, comm).to(torch.float32)
        return dI.to(I_local.dtype), dT.to(T_local.dtype), ds, None, None, None, None, None


def infcl_loss(I_local: torch.Tensor, T_local: torch.Tensor, logit_scale, comm: RingComm | None = None):
    """Symmetric InfoNCE loss L = (L_I + L_T)/2 over the global batch (this rank's shards), differentiable in
    I_local, T_local and -- when ``logit_scale`` is a tensor that requires grad (CLIP's learnable temperature,
    the scale itself, not its log) -- in the logit scale."""
    world = comm.world if comm is not None else 1
    rank = comm.rank if comm is not None else 0
    b = I_local.shape[0] * world
    scale_t = logit_scale if isinstance(logit_scale, torch.Tensor) else None
    s = float(logit_scale.detach()) if scale_t is not None else float(logit_scale)
    return _InfCLFunction.apply(I_local, T_local, scale_t, b, s, rank, world, comm)
