"""One forward + backward of the bench workload (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b = int(os.environ.get("B", 65536)); d = int(os.environ.get("D", 512))
I, T = make_features_device(b, d, seed=0, device="cuda")
ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
g = torch.ones((), device="cuda")
for _ in range(int(os.environ.get("REPS", 1))):
    loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
torch.cuda.synchronize()
print("loss", loss.item())
