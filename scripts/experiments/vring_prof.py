"""One virtual-ring forward+backward (all n ranks' steps on one GPU) for an ncu launch list: per-kernel
durations of the small-step (b_s = b/n) regime that strong scaling hits at n = 8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b, d, world = int(os.environ.get("B", 65536)), int(os.environ.get("D", 512)), int(os.environ.get("W", 8))
I, T = make_features_device(b, d, seed=0, device="cuda")
g = torch.ones((), device="cuda")
for rep in range(2):
    loss, r, c, dg = K.infcl_forward_virtual(I, T, 14.2857, world)
    dI, dT = K.infcl_backward_virtual(I, T, 14.2857, world, r, c, dg, g)
torch.cuda.synchronize()
print("loss", loss.item())
