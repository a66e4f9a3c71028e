"""Loop-structure probe 4: M=128 pair vs M=256 pair ("wide") S-GEMM loops with the real warp roles."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
KB = 8
for wide, ns, tiles in ((0, 4, 2000), (512, 2, 1000), (512, 3, 1000)):
    for mode in (0, 16, 16 | 32 | 64):
        rc = L.infcl_diag_walk2(tiles, KB, ns, mode | wide, 74, ctypes.c_void_p(out.data_ptr()))
        n_mma = tiles * KB * 4
        ideal = 128 if wide else 64
        cyc = out[1].item() / n_mma
        print(f"wide={wide>0} ns={ns} mode={mode:3d} (producer={(mode>>4)&1} epi={(mode>>5)&1}) rc={rc} "
              f"{cyc:6.1f} cyc/mma  efficiency {ideal / cyc:5.1%}", flush=True)
