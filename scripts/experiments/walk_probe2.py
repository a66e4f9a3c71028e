"""Loop-structure probe with real warp roles (csrc/probe.cu probe_walk2_kernel): cycles per MMA."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
tiles, KB, ns = 2000, 8, 4
for ncl in (1, 74):
    for mode in (0, 16, 32, 32 | 64, 16 | 32, 16 | 32 | 64):
        rc = L.infcl_diag_walk2(tiles, KB, ns, mode, ncl, ctypes.c_void_p(out.data_ptr()))
        n_mma = tiles * KB * 4
        print(f"clusters={ncl:3d} mode={mode:3d} (producer={(mode>>4)&1} epi={(mode>>5)&1} tmem_ld={(mode>>6)&1}) rc={rc} "
              f"issue={out[0].item()/n_mma:6.1f} total={out[1].item()/n_mma:6.1f} cyc/mma", flush=True)
