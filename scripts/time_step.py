"""Time forward / backward of the bench workload with CUDA events (env-driven diagnostics welcome)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b = int(os.environ.get("B", 65536)); d = int(os.environ.get("D", 512))
I, T = make_features_device(b, d, seed=0, device="cuda")
ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
g = torch.ones((), device="cuda")
def run():
    loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    e1 = torch.cuda.Event(enable_timing=True); e1.record()
    dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
    return loss, e1
for _ in range(2): run()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
e0.record(); loss, e1 = run(); e2.record(); torch.cuda.synchronize()
print(json.dumps({"tag": os.environ.get("TAG", ""), "b": b, "d": d, "fwd_ms": e0.elapsed_time(e1), "bwd_ms": e1.elapsed_time(e2), "loss": loss.item()}))
