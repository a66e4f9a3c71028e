"""L2 fp32 reduction throughput from 148 SMs (single-pass backward feasibility).
Needed by a single-pass backward at cfg2: 512 KB of fp32 dT partial per CTA-pair tile = ~7.3 TB/s at 1.4 PF."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
D = L.diag()
win = 256 * 512  # one column tile (256 columns x d = 512) of fp32: 512 KB
dst = torch.zeros(148 * 4 * win, device="cuda")
st = torch.cuda.current_stream()
for mode, name in [(0, "bulk same offset"), (1, "bulk staggered"), (2, "bulk disjoint"), (3, "red.v4 staggered")]:
    for chunk in (32768, 65536, 131072):
        n = 148
        iters = 200
        dwin = 4 * win * (148 if mode == 2 else 1)
        if D.infcl_diag_reduce_rate(dst.data_ptr(), dwin, chunk, 4, n, mode, st.cuda_stream):
            raise SystemExit("launch failed")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = D.infcl_diag_reduce_rate(dst.data_ptr(), dwin, chunk, iters, n, mode, st.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"mode {mode} {name:18s} chunk {chunk>>10:4d} KB: {n*iters*chunk/ms/1e6:8.1f} GB/s  ({ms:.2f} ms) rc={rc}",
              flush=True)
