import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for (M, N, amn, name) in [(128, 256, 0, "S pair M128N256"), (256, 128, 1, "dA pair M256N128 MN")]:
    for ld in (0, 1, 2):
        code = (8 << 1) | amn | (ld << 5)
        it = 8192
        L.diag_call("infcl_probe_mma_rate", M, N, code, 2, it, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        c = out.cpu().tolist()
        print(f"{name:22s} tmem-ld-mode={ld} total={c[1]/it:7.1f} cyc/mma", flush=True)
