"""Loop-structure probe 6: the S GEMM's M=128 N=256 pair loop vs the transposed S^T shape (M=256 N=128, operands
swapped: same bytes per stage) vs M=256 N=256, with the real warp roles (producer ring, epilogue handshake)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
KB = 8
for name, shape, ns, tiles in (("M128N256", 0, 4, 2000), ("M256N128 (S^T)", 2048, 4, 2000), ("M256N256", 512, 3, 1000)):
    for mode in (0, 16, 16 | 32 | 64, 16 | 32 | 64 | 1024):
        rc = L.infcl_diag_walk2(tiles, KB, ns, mode | shape, 74, ctypes.c_void_p(out.data_ptr()))
        n_mma = tiles * KB * 4
        ideal = 128 if shape == 512 else 64
        cyc = out[1].item() / n_mma
        print(f"{name:15s} ns={ns} mode={mode:5d} (producer={(mode>>4)&1} epi={(mode>>5)&1} paircommit={(mode>>10)&1}) "
              f"rc={rc} {cyc:6.1f} cyc/mma  efficiency {ideal / cyc:5.1%}", flush=True)
