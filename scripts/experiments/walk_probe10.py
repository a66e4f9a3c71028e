"""MMA issue style in the walk probe's M=128 N=256 pair S loop (74 clusters): 8-MMA asm block with in-asm descriptor
adds (kernel style), 8 single-MMA asm statements with C++ descriptors (L, 131072), one elected lane issuing plain
asm MMAs (E, 262144); with the ring waits / commits (mode 0), pair commits (1024), none (128 | 65536)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for style, sb in (("asm8", 0), ("L", 131072), ("E", 262144)):
    for mode in (0, 1024, 128 | 65536, 16 | 1024):
        rc = L.infcl_diag_walk2(2000, 8, 4, mode | sb, 74, ctypes.c_void_p(out.data_ptr()))
        cyc = out[1].item() / (2000 * 8 * 4)
        print(f"style={style:4s} mode={mode:6d} rc={rc} {cyc:6.1f} cyc/mma {64 / cyc:5.1%}", flush=True)
