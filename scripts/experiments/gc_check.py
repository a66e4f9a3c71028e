"""Fused single-pass backward check: run the backward for a list of shapes and save dI, dT (and loss) to
/tmp/gc_<tag>.pt; with CMP=1 compare the fused run against the two-pass run (INFCL_FUSED_BWD=0) and against
the fp64 oracle for the small shapes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
SHAPES = [(256, 64), (1000, 128), (4096, 512), (20000, 256), (65536, 512), (19244, 512), (70000, 64)]
tag = os.environ.get("TAG", "fused")
if os.environ.get("CMP"):
    import numpy as np
    import oracle
    from synth import make_features
    a = torch.load("/tmp/gc_fused.pt"); b = torch.load("/tmp/gc_twopass.pt")
    for k in a:
        x, y = a[k], b[k]
        r = {n: float((x[n] - y[n]).norm() / y[n].norm()) for n in ("dI", "dT")}
        r["bitwise_eq"] = {n: bool(torch.equal(x[n], y[n])) for n in ("dI", "dT")}
        bb, d = map(int, k.split("x"))
        if bb <= 4096:
            I, T = make_features(bb, d, seed=1, dist="independent")
            ref = oracle.loss_and_grads(I, T, 14.2857)
            for n in ("dI", "dT"):
                r["oracle_" + n] = float(np.linalg.norm(x[n].numpy() - ref[n]) / np.linalg.norm(ref[n]))
        print(k, json.dumps(r))
    sys.exit(0)
from paper_2410_17243_b200 import loss as K
from synth import make_features, make_features_device
out = {}
for bb, d in SHAPES:
    if bb <= 4096:
        I, T = make_features(bb, d, seed=1, dist="independent"); I, T = I.cuda(), T.cuda()
    else:
        I, T = make_features_device(bb, d, seed=1, device="cuda")
    g = torch.ones((), device="cuda")
    loss, r, c, dg = K.infcl_forward(I, T, bb, 14.2857)
    dI, dT = K.infcl_backward(I, T, bb, 14.2857, r, c, dg, g)
    torch.cuda.synchronize()
    out[f"{bb}x{d}"] = {"dI": dI.cpu(), "dT": dT.cpu()}
    print(tag, bb, d, "ok", float(dI.norm()), float(dT.norm()), flush=True)
torch.save(out, f"/tmp/gc_{tag}.pt")  # large: not under gpurun_out
