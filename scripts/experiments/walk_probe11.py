"""Two MMA-issuing warps (alternate ring stages, different SM sub-partitions) vs one, in the walk probe's M=128 N=256
pair loop with ring waits and per-stage commits (mode 0), pair commits (1024), no waits/commits (128 | 65536)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for two in (0, 524288):
    for mode in (0, 1024, 128 | 65536):
        rc = L.infcl_diag_walk2(2000, 8, 4, mode | two, 74, ctypes.c_void_p(out.data_ptr()))
        cyc = out[1].item() / (2000 * 8 * 4)
        print(f"issuers={2 if two else 1} mode={mode:6d} rc={rc} {cyc:6.1f} cyc/mma {64 / cyc:5.1%}", flush=True)
