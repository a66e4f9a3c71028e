"""Is the ~96-cycle cost of a 64-cycle pair MMA (walk probes) set by the operand footprint?  The pair kernel's real
S-GEMM instruction stream (8-MMA asm blocks, M=128 N=256) over 1, 2 or 4 ring stages of operands, no barriers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for ncl in (1, 74):
    for wrap in (1, 2, 4):
        for ld in (0, 2):
            it = 65536
            code = (ncl << 8) | 128 | (ld << 5) | ((wrap if wrap < 4 else 0) << 1)
            L.diag_call("infcl_probe_mma_rate", 128, 256, code, 2, it, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            c = out.cpu().tolist()
            print(f"M128N256 stream stages={wrap} clusters={ncl:3d} tmem_ld={ld} {c[1]/it:6.1f} cyc/mma  rate {64/(c[1]/it):5.3f}", flush=True)
