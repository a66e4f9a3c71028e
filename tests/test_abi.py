"""CPU checks of the C ABI: the library loads without a GPU and exports every symbol include/infcl.h declares;
host-only entry points behave; device entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

from paper_2410_17243_b200 import _lib as L

INCLUDE = os.path.join(os.path.dirname(__file__), "..", "include")
HEADER = os.path.join(INCLUDE, "infcl.h")
DIAG_HEADER = os.path.join(INCLUDE, "infcl_diag.h")


def declared_symbols(path=HEADER):
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(infcl_[a-z0-9_]+)\s*\(", src)))


def exported_symbols(so):
    """Defined dynamic symbols of a shared library (nm -D), i.e. everything a dlsym can reach."""
    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    return sorted({ln.split()[-1] for ln in out.splitlines() if ln.strip() and ln.split()[-2] in "TtDdBbRrWwVv"})


def test_header_symbols_exported():
    names = declared_symbols()
    assert len(names) >= 15
    lib = L.lib()
    for n in names:
        assert hasattr(lib, n), n
        assert n in L.SIGNATURES, f"binding lacks {n}"
    assert set(L.SIGNATURES) == set(names)


def test_product_exports_exactly_the_header():
    """libinfcl.so exports the symbols include/infcl.h declares and nothing else (no undeclared entry points,
    no C++ internals, no probes: those live in libinfcl_diag.so)."""
    assert exported_symbols(L.LIB_PATH) == declared_symbols()


def test_diag_library_exports_exactly_its_header():
    names = declared_symbols(DIAG_HEADER)
    assert exported_symbols(L.DIAG_PATH) == names
    assert set(L.DIAG_SIGNATURES) == set(names)
    assert not set(names) & set(declared_symbols())  # disjoint from the product ABI
    D = L.diag()
    for n in names:
        assert hasattr(D, n), n


def test_host_functions():
    lib = L.lib()
    assert lib.infcl_version() >= 100
    assert lib.infcl_ring_block(2, 4, 2) == 0
    assert lib.infcl_ring_block(0, 4, 4) == -1
    for n in (1, 2, 3, 8, 16):
        for step in range(n):
            assert sorted(lib.infcl_ring_block(r, n, step) for r in range(n)) == list(range(n))
    assert lib.infcl_status_string(3) == b"INFCL_ERR_CONFIG"
    assert lib.infcl_workspace_bytes(7, 32, 2, 0) == 0  # b % world
    assert lib.infcl_workspace_bytes(1024, 512, 1, 0) > 0


def test_validation_errors_without_gpu():
    lib = L.lib()
    buf = ctypes.create_string_buffer(4096)
    p = ctypes.cast(buf, ctypes.c_void_p)
    # b not divisible by world -> CONFIG, detected before touching any device
    st = lib.infcl_forward(None, p, p, 0, 7, 32, 1.0, 0, 2, p, p, p, p, p, 4096, None)
    assert st == 3 and b"divisible" in lib.infcl_last_error()
    assert lib.infcl_forward(None, p, p, 0, 64, 30, 1.0, 0, 1, p, p, p, p, p, 4096, None) == 2  # d % 8
    assert lib.infcl_forward(None, p, p, 0, 64, 32, float("inf"), 0, 1, p, p, p, p, p, 4096, None) == 1
    assert lib.infcl_forward(None, None, p, 0, 64, 32, 1.0, 0, 1, p, p, p, p, p, 4096, None) == 1
    # a valid call on a GPU-less host must fail (UNSUPPORTED or WORKSPACE), never silently succeed
    assert lib.infcl_forward(None, p, p, 0, 64, 32, 1.0, 0, 1, p, p, p, p, p, 1 << 40, None) != 0


def test_product_path_does_not_import_oracle():
    import paper_2410_17243_b200
    pkg = os.path.dirname(paper_2410_17243_b200.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_binding_rejects_host_tensors_and_shape_mismatch():
    """The Python binding is marshalling only: host tensors never reach a CPU fallback (there is none)."""
    import pytest
    import torch
    from paper_2410_17243_b200 import loss as K
    I = torch.zeros(64, 32, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        K.infcl_forward(I, I, 64, 1.0)
    with pytest.raises((ValueError, TypeError)):
        K._check_features(torch.zeros(64, 32), torch.zeros(64, 16))
    with pytest.raises(TypeError):
        K._dtype_code(torch.zeros(4, 8, dtype=torch.float16))


def test_workspace_and_e2e_scratch_sizes():
    """Workspace grows linearly in b (O(b d) per GPU, SURVEY 8(d) memory) and is 0 for invalid shapes."""
    lib = L.lib()
    w1 = lib.infcl_workspace_bytes(65536, 512, 1, 0)
    w2 = lib.infcl_workspace_bytes(131072, 512, 1, 0)
    assert 1.9 < w2 / w1 < 2.1
    # a ring rank also holds two travelling blocks (2 b_s d bf16) and their LSE vectors
    assert lib.infcl_workspace_bytes(65536, 512, 8, 0) >= 2 * (65536 // 8) * 512 * 2
    assert lib.infcl_workspace_bytes(0, 512, 1, 0) == 0
    s1 = lib.infcl_e2e_scratch_bytes(65536, 512, 0)
    # e2e scratch holds the bf16 inputs, fp32 gradients, LSE vectors and the workspace
    assert s1 >= 2 * 65536 * 512 * 2 + 2 * 65536 * 512 * 4 + w1


def test_ipc_transport_host_checks_without_gpu():
    """IPC ring communicator: argument checks before any device work; NULL-comm queries; the comm-aware
    workspace equals the NCCL-layout size for a NULL comm (world 1 / NCCL)."""
    lib = L.lib()
    out = ctypes.c_void_p()
    assert lib.infcl_comm_init_ipc(None, 0, 2, 0, 1024, 64, 0) == 1                   # null out
    assert lib.infcl_comm_init_ipc(ctypes.byref(out), 0, 1, 0, 1024, 64, 0) == 3      # world < 2
    assert lib.infcl_comm_init_ipc(ctypes.byref(out), 2, 2, 0, 1024, 64, 0) == 3      # rank out of range
    assert lib.infcl_comm_init_ipc(ctypes.byref(out), 0, 2, 0, 1023, 64, 0) == 2      # b % world
    assert lib.infcl_comm_init_ipc(ctypes.byref(out), 0, 2, 0, 1024, 64, 0) != 0      # no GPU here: fails loudly
    assert not out.value
    assert lib.infcl_comm_transport(None) == -1
    assert lib.infcl_comm_ipc_region_bytes(None) == 0
    assert lib.infcl_comm_ipc_handle(None, None) == 1
    assert lib.infcl_comm_ipc_connect(None, None) == 1
    assert lib.infcl_comm_ipc_selftest(None, 10) == 1
    for b, d, w in ((65536, 512, 1), (65536, 512, 8), (4096, 768, 2)):
        assert lib.infcl_comm_workspace_bytes(None, b, d, w, 0) == lib.infcl_workspace_bytes(b, d, w, 0)
