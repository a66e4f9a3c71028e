"""S-GEMM loop-structure probe (csrc/probe.cu probe_walk_kernel): cycles per MMA for feature combinations."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(2, dtype=torch.int64, device="cuda")
tiles, KB, ns = 2000, 8, 4
for mode in (0, 1, 2, 3, 4, 7, 8, 15):
    rc = L.infcl_diag_walk(tiles, KB, ns, mode, ctypes.c_void_p(out.data_ptr()))
    n_mma = tiles * KB * 4
    print(f"mode={mode:2d} (walkA={mode&1} walkB={(mode>>1)&1} rotD={(mode>>2)&1} ring={(mode>>3)&1}) rc={rc} "
          f"issue={out[0].item()/n_mma:6.1f} total={out[1].item()/n_mma:6.1f} cyc/mma", flush=True)
