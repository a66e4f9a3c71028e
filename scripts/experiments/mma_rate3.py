import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for rep in range(2):
  for (M, N, amn, name) in [(128, 256, 0, "S pair M128N256"), (256, 128, 1, "dA pair M256N128 MN"), (256, 256, 0, "pair M256N256")]:
    for G in (0, 8):
        code = amn if G == 0 else (G << 1) | amn
        it = 8192
        L.diag_call("infcl_probe_mma_rate", M, N, code, 2, it, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        c = out.cpu().tolist()
        print(f"{name:22s} stage-group={G:2d} total={c[1]/it:7.1f} cyc/mma -> {2*M*N*16/2/(c[1]/it):6.0f} flop/clk/SM", flush=True)
