"""Tiny forward+backward for compute-sanitizer runs: both forward kernels (wide: streamed and
resident A), the backward,
the virtual ring and the host e2e entry on small shapes with ragged tails."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features
for b, d in ((300, 64), (520, 128), (600, 256), (1100, 512)):  # d >= 256: resident-A forward
    I, T = make_features(b, d, seed=1, dist="paired")
    Id, Td = I.cuda(), T.cuda()
    loss, r, c, dg = K.infcl_forward(Id, Td, b, 14.2857)
    dI, dT = K.infcl_backward(Id, Td, b, 14.2857, r, c, dg, torch.tensor(1.0, device="cuda"))
    os.environ["INFCL_FWD_NARROW"] = "1"
    loss2, *_ = K.infcl_forward(Id, Td, b, 14.2857)
    del os.environ["INFCL_FWD_NARROW"]
    lv, *_ = K.infcl_forward_virtual(Id, Td, 14.2857, 2) if b % 2 == 0 else (loss,)
    torch.cuda.synchronize()
    print(b, d, loss.item(), loss2.item(), float(lv), float(dI.norm()), float(dT.norm()))
