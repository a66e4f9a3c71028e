"""Loop-structure probe 5: one commit per stage vs one commit per two stages (M=128 pair MMAs, real roles)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
KB, ns, tiles = 8, 4, 2000
for rep in range(2):
    for mode in (16 | 32 | 64, 16 | 32 | 64 | 1024, 0, 1024):
        rc = L.infcl_diag_walk2(tiles, KB, ns, mode, 74, ctypes.c_void_p(out.data_ptr()))
        cyc = out[1].item() / (tiles * KB * 4)
        print(f"mode={mode:5d} (producer={(mode>>4)&1} epi={(mode>>5)&1} commit-per-2={(mode>>10)&1}) rc={rc} {cyc:6.1f} cyc/mma  eff {64/cyc:5.1%}", flush=True)
