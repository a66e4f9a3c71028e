"""Paper-scale batches on ONE B200 (the paper's headline 4M batch ran on 8 A800): one timed fwd+bwd step at
b = 2M and 4M, d = 768, with peak device memory.  A warm-up on a small batch loads the kernels first."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device

d = int(os.environ.get("D", 768))
warm = make_features_device(65536, d, seed=1, device="cuda")
K.infcl_forward(warm[0], warm[1], 65536, 14.2857)
del warm
for b in [int(x) for x in os.environ.get("BS", "2097152,4194304").split(",")]:
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    I, T = make_features_device(b, d, seed=0, device="cuda")
    ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
    g = torch.ones((), device="cuda")
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    e1.record()
    dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
    e2.record()
    torch.cuda.synchronize()
    f, bw = e0.elapsed_time(e1), e1.elapsed_time(e2)
    peak = torch.cuda.max_memory_allocated() / 1e9
    print(json.dumps({"b": b, "d": d, "fwd_ms": f, "bwd_ms": bw, "samples_per_s": b / ((f + bw) / 1e3),
                      "step_tflops_8b2d": 8.0 * b * b * d / ((f + bw) / 1e3) / 1e12, "peak_gb": peak,
                      "loss": loss.item(), "finite_grads": bool(torch.isfinite(dI).all() and torch.isfinite(dT).all())}),
          flush=True)
    del I, T, ws, dI, dT, r, c, dg
