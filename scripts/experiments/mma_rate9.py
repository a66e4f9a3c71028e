"""Does the operand DATA change the pair-MMA rate?  The real S-GEMM stream (M=128 N=256, 192-KB footprint) with the
operand smem filled with bf16 1.0 (0x3f80) vs the walk probes' 0x3c00 (bf16 2^-7; fp16 1.0), and random bits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for fill in (0, 1):
    for M, N, stream in ((128, 256, 128), (128, 256, 0), (256, 256, 0)):
        it = 65536
        code = (74 << 8) | stream
        L.diag_call("infcl_probe_mma_rate", M, N, code, 2, it | (fill << 30), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        c = out.cpu().tolist()
        ideal = M * N / 512
        print(f"fill={'0x3c00' if fill else '0x3f80'} M{M}N{N} stream={stream > 0} {c[1] / it:6.1f} cyc/mma  rate {ideal / (c[1] / it):5.3f}", flush=True)
