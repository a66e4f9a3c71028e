"""Tiny shapes of the fused backward kernels for compute-sanitizer (memcheck / synccheck / initcheck): the two-role
kernel (d = 64, 512 and 768's two consumer parts), the fused ring through the virtual 2-rank ring, and -- with
INFCL_BWD3=1 in the environment -- the three-role kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["INFCL_GC_MIN_ROWS"] = "0"
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features
g = torch.tensor(1.0, device="cuda")
for b, d in ((300, 64), (1100, 512), (1040, 768)):
    I, T = make_features(b, d, seed=1, dist="paired")
    Id, Td = I.cuda(), T.cuda()
    loss, r, c, dg = K.infcl_forward(Id, Td, b, 14.2857)
    dI, dT = K.infcl_backward(Id, Td, b, 14.2857, r, c, dg, g)
    if b % 2 == 0:
        lv, rv, cv, dgv = K.infcl_forward_virtual(Id, Td, 14.2857, 2)
        dIv, dTv = K.infcl_backward_virtual(Id, Td, 14.2857, 2, rv, cv, dgv, g)
    torch.cuda.synchronize()
    print(b, d, loss.item(), float(dI.norm()), float(dT.norm()), flush=True)
