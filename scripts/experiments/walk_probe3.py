"""Loop-structure probe 3: cost of commits vs waits (csrc/probe.cu probe_walk2_kernel)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
tiles, KB = 2000, 8
for ns in (4, 6):
    for mode in (128, 0, 256, 16, 16 | 256, 32 | 128, 16 | 32 | 64, 16 | 32 | 64 | 256):
        rc = L.infcl_diag_walk2(tiles, KB, ns, mode, 74, ctypes.c_void_p(out.data_ptr()))
        n_mma = tiles * KB * 4
        print(f"ns={ns} mode={mode:3d} (nowait={(mode>>7)&1} commit2={(mode>>8)&1} producer={(mode>>4)&1} epi={(mode>>5)&1}) rc={rc} "
              f"total={out[1].item()/n_mma:6.1f} cyc/mma", flush=True)
