"""Bitwise run-to-run determinism of the outputs (same inputs, same launch configuration)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
out = {}
for b, d in ((65536, 512), (19244, 512), (8192, 768)):
    I, T = make_features_device(b, d, seed=3, device="cuda")
    g = torch.ones((), device="cuda")
    res = []
    for _ in range(3):
        loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857)
        dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g)
        torch.cuda.synchronize()
        res.append((loss.clone(), r.clone(), c.clone(), dI.clone(), dT.clone()))
    same = [all(torch.equal(res[0][i], res[k][i]) for k in (1, 2)) for i in range(5)]
    out[f"{b}x{d}"] = dict(zip(["loss", "r", "c", "dI", "dT"], same))
    out[f"{b}x{d}_max_abs_diff_dI"] = float((res[0][3] - res[1][3]).abs().max())
print(json.dumps(out))
