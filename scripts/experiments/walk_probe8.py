"""Loop-structure probe 8: is the 64-cycle pair MMA loop throttled by how far the issuer may run ahead of MMA
completion?  mode 128 = no ring waits at all; ns = ring stages (32 KB each) the issuer may run ahead."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for name, shape in (("SS M128N256", 0), ("TS M128N256", 4096)):
    for KB, ns, mode in ((8, 4, 128), (8, 4, 0), (4, 2, 0), (4, 3, 0), (4, 4, 0), (4, 6, 0), (4, 6, 1024), (4, 6, 16), (4, 6, 1040)):
        tiles = 4000
        rc = L.infcl_diag_walk2(tiles, KB, ns, mode | shape, 74, ctypes.c_void_p(out.data_ptr()))
        cyc = out[1].item() / (tiles * KB * 4)
        print(f"{name:12s} KB={KB} ns={ns} mode={mode:5d} (nowait={(mode>>7)&1} producer={(mode>>4)&1} "
              f"paircommit={(mode>>10)&1}) rc={rc} {cyc:6.1f} cyc/mma efficiency {64 / cyc:5.1%}", flush=True)
