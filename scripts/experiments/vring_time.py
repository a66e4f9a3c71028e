"""Per-step overhead of the ring schedule: the virtual ring runs all n ranks' steps on one GPU, so its time
vs the n=1 time for the same global batch shows the cost of small per-step launches (tails, merges)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b, d = int(os.environ.get("B", 65536)), int(os.environ.get("D", 512))
I, T = make_features_device(b, d, seed=0, device="cuda")
g = torch.ones((), device="cuda")
for world in (1, 2, 4, 8):
    ts = []
    for rep in range(4):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        if world == 1:
            loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857)
            e1.record()
            dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g)
        else:
            loss, r, c, dg = K.infcl_forward_virtual(I, T, 14.2857, world)
            e1.record()
            dI, dT = K.infcl_backward_virtual(I, T, 14.2857, world, r, c, dg, g)
        e2.record()
        torch.cuda.synchronize()
        if rep:
            ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    f = statistics.median(x[0] for x in ts)
    bw = statistics.median(x[1] for x in ts)
    print(json.dumps({"world": world, "b": b, "d": d, "fwd_ms": f, "bwd_ms": bw, "total_ms": f + bw,
                      "per_rank_ms_if_parallel": (f + bw) / world}), flush=True)
