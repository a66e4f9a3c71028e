"""Loop-structure probe 7: the dI GEMM's TS form (A = G in TMEM, B = 32-KB ring stage, M=128 N=256 pair, 64-cycle
MMAs) vs the SS M=128 N=256 loop, real smem footprints and ring handshakes (probe_walk2_kernel)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
KB = 8
for name, shape in (("SS M128N256", 0), ("TS M128N256", 4096)):
    for mode in (0, 16, 16 | 1024):
        rc = L.infcl_diag_walk2(2000, KB, 4, mode | shape, 74, ctypes.c_void_p(out.data_ptr()))
        cyc = out[1].item() / (2000 * KB * 4)
        print(f"{name:12s} mode={mode:5d} (producer={(mode>>4)&1} paircommit={(mode>>10)&1}) rc={rc} {cyc:6.1f} cyc/mma "
              f"efficiency {64 / cyc:5.1%}", flush=True)
