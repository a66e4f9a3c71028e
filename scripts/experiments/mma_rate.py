"""Measure raw tcgen05.mma throughput for the shapes the pair kernel issues."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for (M, N, amn, ncta, name) in [(128, 256, 0, 2, "S GEMM pair M128 N256 Kmaj"), (256, 128, 1, 2, "dA GEMM pair M256 N128 A-MNmaj"),
                                (256, 128, 0, 2, "pair M256 N128 Kmaj"), (256, 256, 0, 2, "pair M256 N256 Kmaj"),
                                (128, 256, 0, 1, "1cta M128 N256"), (128, 128, 0, 1, "1cta M128 N128"),
                                (128, 64, 0, 2, "pair M128 N64"), (256, 64, 1, 2, "pair M256 N64 MN")]:
    it = 4096
    L.diag_call("infcl_probe_mma_rate", M, N, amn, ncta, it, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    c = out.cpu().tolist()
    flops_per_sm = 2 * M * N * 16 / ncta
    print(f"{name:32s} issue={c[0]/it:7.1f} cyc/mma  total={c[1]/it:7.1f} cyc/mma  -> {flops_per_sm/(c[1]/it):7.0f} flop/clk/SM")
