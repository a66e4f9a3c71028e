"""Loop-structure elements of the walk probes added to the real S-GEMM stream one at a time (see mma_rate8.py):
variant bit 4 is now a tcgen05.fence::after_thread_sync per stage."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for var in (0, 4, 8, 12, 15, 11):
    it = 65536
    code = (74 << 8) | 128 | (var << 1)
    L.diag_call("infcl_probe_mma_rate", 128, 256, code, 2, it, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    c = out.cpu().tolist()
    print(f"variant {var:2d} (acc0={var & 1} rotD={(var >> 1) & 1} fence={(var >> 2) & 1} commit+wait={(var >> 3) & 1}) "
          f"{c[1] / it:6.1f} cyc/mma  rate {64 / (c[1] / it):5.3f}", flush=True)
