"""Which part of the pair kernel's loop structure costs the 64-cycle pair MMAs their rate?  The real S-GEMM
instruction stream (M=128 N=256, 8-MMA asm blocks, 192-KB footprint) with one structural element added at a time:
1 accumulate=0 at each tile start, 2 D rotating over 4 buffers per tile, 4 D alternating between two regions every
stage (the backward's S / dA interleave), 8 a commit to a real barrier per stage and a wait 3 stages back."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for var in (0, 1, 2, 3, 4, 8, 12, 15):
    it = 65536
    code = (74 << 8) | 128 | (var << 1)
    L.diag_call("infcl_probe_mma_rate", 128, 256, code, 2, it, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    c = out.cpu().tolist()
    print(f"variant {var:2d} (acc0={var & 1} rotD={(var >> 1) & 1} altD={(var >> 2) & 1} commit+wait={(var >> 3) & 1}) "
          f"{c[1] / it:6.1f} cyc/mma  rate {64 / (c[1] / it):5.3f}", flush=True)
