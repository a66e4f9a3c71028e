"""Do warps parked in barrier.cluster.wait slow down the MMA-issuing warp?  The real S-GEMM stream (M=128 N=256 pair,
192-KB footprint) with the CTA's idle warps waiting on an mbarrier (try_wait) vs in the cluster barrier."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for M, N, stream in ((128, 256, 128), (256, 256, 0), (256, 128, 0)):
    for cb in (0, 1):
        it = 65536
        L.diag_call("infcl_probe_mma_rate", M, N, (74 << 8) | stream, 2, it | (cb << 29), out.data_ptr(),
                    torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        c = out.cpu().tolist()
        ideal = M * N / 512
        print(f"M{M}N{N} stream={stream > 0} idle warps in {'cluster barrier' if cb else 'mbarrier try_wait'}: "
              f"{c[1] / it:6.1f} cyc/mma  rate {ideal / (c[1] / it):5.3f}", flush=True)
