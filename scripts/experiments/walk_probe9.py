"""Bisect the walk probe's 64-cycle-MMA slowdown (probe_walk2_kernel, M=128 N=256 pair S loop, 74 clusters): remove
the per-stage tcgen05 fences (8192), the D rotation (16384), the accumulate-0 tile starts (32768), the per-stage
commits (65536, with no waits: 128)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for mode in (0, 128, 128 | 65536, 128 | 65536 | 8192, 128 | 65536 | 8192 | 16384, 128 | 65536 | 8192 | 16384 | 32768,
             8192, 16384, 32768, 8192 | 16384 | 32768):
    rc = L.infcl_diag_walk2(2000, 8, 4, mode, 74, ctypes.c_void_p(out.data_ptr()))
    cyc = out[1].item() / (2000 * 8 * 4)
    print(f"mode={mode:6d} nowait={(mode >> 7) & 1} nocommit={(mode >> 16) & 1} nofence={(mode >> 13) & 1} "
          f"fixedD={(mode >> 14) & 1} alwaysacc={(mode >> 15) & 1} rc={rc} {cyc:6.1f} cyc/mma {64 / cyc:5.1%}", flush=True)
