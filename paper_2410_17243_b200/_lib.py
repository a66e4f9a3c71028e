"""ctypes binding of include/infcl.h: argument marshalling only (every step of the path runs in libinfcl.so).

The library is loaded from this package directory (built in-tree by ``build.py``); a missing library is a
hard error -- there is no fallback implementation.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# INFCL_LIB: an A/B build variant of the same sources (scripts/build_variant.py); never a different implementation
LIB_PATH = os.environ.get("INFCL_LIB") or os.path.join(_HERE, "libinfcl.so")

INFCL_BF16 = 0
INFCL_FP32 = 1
INFCL_TRANSPORT_NCCL = 0
INFCL_TRANSPORT_IPC = 1

STATUS = {0: "INFCL_OK", 1: "INFCL_ERR_INVALID_ARG", 2: "INFCL_ERR_SHAPE", 3: "INFCL_ERR_CONFIG",
          4: "INFCL_ERR_CUDA", 5: "INFCL_ERR_NCCL", 6: "INFCL_ERR_WORKSPACE", 7: "INFCL_ERR_UNSUPPORTED"}

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i = ctypes.c_int
_f = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes); the exact list of symbols include/infcl.h declares
SIGNATURES = {
    "infcl_status_string": (ctypes.c_char_p, [_i]),
    "infcl_last_error": (ctypes.c_char_p, []),
    "infcl_version": (_i, []),
    "infcl_get_unique_id": (_i, [_p]),
    "infcl_comm_init": (_i, [ctypes.POINTER(_p), _i, _i, _p, _i]),
    "infcl_comm_destroy": (_i, [_p]),
    "infcl_workspace_bytes": (_sz, [_i64, _i, _i, _i]),
    "infcl_comm_workspace_bytes": (_sz, [_p, _i64, _i, _i, _i]),
    "infcl_comm_init_ipc": (_i, [ctypes.POINTER(_p), _i, _i, _i, _i64, _i, _i]),
    "infcl_comm_ipc_handle": (_i, [_p, _p]),
    "infcl_comm_ipc_connect": (_i, [_p, _p]),
    "infcl_comm_ipc_selftest": (_i, [_p, _i]),
    "infcl_comm_ipc_region_bytes": (_sz, [_p]),
    "infcl_comm_transport": (_i, [_p]),
    "infcl_forward": (_i, [_p, _p, _p, _i, _i64, _i, _f, _i, _i, _p, _p, _p, _p, _p, _sz, _p]),
    "infcl_backward": (_i, [_p, _p, _p, _i, _i64, _i, _f, _i, _i, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "infcl_forward_virtual": (_i, [_p, _p, _i, _i64, _i, _f, _i, _p, _p, _p, _p, _p, _sz, _p]),
    "infcl_backward_virtual": (_i, [_p, _p, _i, _i64, _i, _f, _i, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "infcl_grad_scale_partial": (_i, [_p, _p, _i, _i64, _i, _f, _p, _p]),
    "infcl_ntxent_forward": (_i, [_p, _p, _p, _i, _i64, _i, _f, _i, _i, _p, _p, _p, _p, _p, _sz, _p]),
    "infcl_ntxent_backward": (_i, [_p, _p, _p, _i, _i64, _i, _f, _i, _i, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "infcl_e2e_scratch_bytes": (_sz, [_i64, _i, _i]),
    "infcl_loss_grad_host": (_i, [_p, _p, _i, _i64, _i, _f, _f, _p, _p, _p, _p, _sz, _p]),
    "infcl_ring_block": (_i, [_i, _i, _i]),
    "infcl_ring_schedule": (_i, [_i, _i, _i, ctypes.POINTER(ctypes.c_int32), _i]),
    "infcl_launch_count": (ctypes.c_uint64, []),
    "infcl_reset_launch_count": (None, []),
    "infcl_profile_enable": (None, [_i]),
    "infcl_profile_read": (_i, [_i, ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_double)]),
}

# libinfcl_diag.so (include/infcl_diag.h): hardware probes and microbenchmarks, never on the product path
DIAG_PATH = os.path.join(_HERE, "libinfcl_diag.so")
DIAG_SIGNATURES = {
    "infcl_diag_last_error": (ctypes.c_char_p, []),
    "infcl_probe_umma": (_i, [_p, _p, _i, _i, _i, _i, _i, _i, _p, _i, _p]),
    "infcl_probe_umma_ts": (_i, [_p, _p, _i, _i, _p, _p]),
    "infcl_probe_mma_rate": (_i, [_i, _i, _i, _i, _i, _p, _p]),
    "infcl_diag_max_clusters": (_i, [_i]),
    "infcl_diag_tma_rate": (_i, [_p, _i, _i, _i, _i, _i, _p]),
    "infcl_diag_tma_rate2": (_i, [_p, _i, _i, _i, _i, _i, _i, _p]),
    "infcl_diag_tma_rate3": (_i, [_p, _i, _i, _i, _i, _i, _i, _p]),
    "infcl_diag_walk": (_i, [_i, _i, _i, _i, _p]),
    "infcl_diag_walk2": (_i, [_i, _i, _i, _i, _i, _p]),
    "infcl_diag_copy": (_i, [_p, _p, _sz, _i, _p]),
    "infcl_diag_reduce_rate": (_i, [_p, _i64, _i, _i, _i, _i, _p]),
}

_lib = None


class InfclError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {detail}")
        self.status = status


def lib():
    """Load libinfcl.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2410_17243_b200.build` "
                              "(or __graft_entry__.build()) -- there is no fallback implementation")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_diag = None


def diag():
    """Load libinfcl_diag.so (probes; separate from the product library)."""
    global _diag
    if _diag is None:
        if not os.path.exists(DIAG_PATH):
            raise ImportError(f"{DIAG_PATH} missing: run `python -m paper_2410_17243_b200.build`")
        D = ctypes.CDLL(DIAG_PATH)
        for name, (res, args) in DIAG_SIGNATURES.items():
            fn = getattr(D, name)
            fn.restype = res
            fn.argtypes = args
        _diag = D
    return _diag


def diag_call(name: str, *args):
    st = getattr(diag(), name)(*args)
    if st != 0:
        raise InfclError(st, name, diag().infcl_diag_last_error().decode(errors="replace"))


def check(status: int, where: str):
    if status != 0:
        raise InfclError(status, where, lib().infcl_last_error().decode(errors="replace"))


def call(name: str, *args):
    """Call an infcl_* entry point returning infcl_status and raise InfclError on failure."""
    st = getattr(lib(), name)(*args)
    check(st, name)
