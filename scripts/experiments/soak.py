"""Soak: many back-to-back forward+backward steps; every step's outputs must be bitwise identical to the first
(determinism makes any rare race or stale read visible), and no watchdog trap / CUDA error may occur."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
res = {}
for b, d, steps in ((65536, 512, 600), (19244, 512, 1500), (8192 * 3 + 300, 768, 600)):
    I, T = make_features_device(b, d, seed=9, device="cuda")
    g = torch.ones((), device="cuda")
    ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
    loss0, r0, c0, dg0 = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    dI0, dT0 = K.infcl_backward(I, T, b, 14.2857, r0, c0, dg0, g, workspace=ws)
    ref = [x.clone() for x in (loss0, r0, c0, dI0, dT0)]
    bad = 0
    t0 = time.time()
    for s in range(steps):
        loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
        dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
        if s % 10 == 9:
            bad += sum(not torch.equal(x, y) for x, y in zip(ref, (loss, r, c, dI, dT)))
    torch.cuda.synchronize()
    res[f"{b}x{d}"] = {"steps": steps, "checked_steps": steps // 10, "mismatches": bad, "seconds": time.time() - t0,
                       "loss": float(loss)}
print(json.dumps(res))
