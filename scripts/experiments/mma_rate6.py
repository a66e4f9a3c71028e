"""MMA issue rate of the CTA-pair shapes the fused backward could use (probe_rate_kernel, libinfcl_diag.so).

Question: is the producers' M=128 N=256 pair S GEMM (64-cycle MMAs) slow because each SM's shared memory serves its
own A rows plus the whole B (both halves, read by both tensor cores) -- (M/2 + N) * K * 2 B per MMA -- or because of
a fixed per-instruction cost of short MMAs?  The two models differ for M=256 N=128 (K-major A): 128 B/clk of operand
reads (full rate under the smem model) vs the same 64-cycle instruction (slow under the overhead model).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2410_17243_b200 import _lib as L  # noqa: E402

out = torch.zeros(4, dtype=torch.int64, device="cuda")
shapes = [(128, 256, 0, "M128N256 K-major A (S now)"), (256, 128, 0, "M256N128 K-major A (S^T)"),
          (256, 128, 1, "M256N128 MN-major A (dA)"), (256, 256, 0, "M256N256 K-major A"),
          (256, 256, 1, "M256N256 MN-major A")]
for (M, N, amn, name) in shapes:
    ideal = M * N / 512.0  # cycles per K=16 MMA of a CTA pair at 8192 dense bf16 FLOP/clk/SM
    for ncl in (1, 74):
        for G in (0, 8):
            for ld in (0, 2):
                it = 65536
                code = (ncl << 8) | (ld << 5) | (G << 1) | amn
                L.diag_call("infcl_probe_mma_rate", M, N, code, 2, it, out.data_ptr(),
                            torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                c = out.cpu().tolist()
                cyc = c[1] / it
                print(f"{name:28s} clusters={ncl:3d} commit/{G if G else '-'} tmem_ld={ld} "
                      f"{cyc:7.1f} cyc/mma  ideal {ideal:5.1f}  rate {ideal / cyc:5.3f}", flush=True)
