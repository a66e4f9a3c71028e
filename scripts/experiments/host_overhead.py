"""Host enqueue cost per call (no synchronisation inside the loop) vs the device time per call, at small and
cfg2 batch: if the host cost approaches the device time, small ring steps are launch-bound."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
for b in (8192, 65536):
    d = 512
    I, T = make_features_device(b, d, seed=0, device="cuda")
    ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
    g = torch.ones((), device="cuda")
    loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    torch.cuda.synchronize()
    n = 40
    t0 = time.perf_counter()
    for _ in range(n):
        K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    t1 = time.perf_counter()
    for _ in range(n):
        K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        K.infcl_forward(I, T, b, 14.2857, workspace=ws)
        K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"b": b, "host_us_per_fwd_call": (t1 - t0) / n * 1e6, "host_us_per_bwd_call": (t2 - t1) / n * 1e6,
                      "device_us_per_step_back_to_back": e0.elapsed_time(e1) / n * 1e3}), flush=True)
