"""A/B of the host end-to-end entry's forward schedule (historical: INFCL_E2E_OLD_SCHEDULE existed in the round-1 build only): cfg2 loss+grads from pinned
host buffers, interleaved rounds, median ms per call."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b, d = int(os.environ.get("B", 65536)), int(os.environ.get("D", 512))
I, T = make_features_device(b, d, seed=77, device="cuda")
Ih, Th = I.cpu().pin_memory(), T.cpu().pin_memory()
scratch = torch.empty(int(K.L.lib().infcl_e2e_scratch_bytes(b, d, 0)), dtype=torch.uint8, device="cuda")
out = (torch.empty((), dtype=torch.float32).pin_memory(), torch.empty(b, d, dtype=torch.float32).pin_memory(),
       torch.empty(b, d, dtype=torch.float32).pin_memory())
res = {"new": [], "old": []}
losses = {}
for rnd in range(6):
    for v in ("new", "old"):
        if v == "old":
            os.environ["INFCL_E2E_OLD_SCHEDULE"] = "1"
        else:
            os.environ.pop("INFCL_E2E_OLD_SCHEDULE", None)
        K.infcl_loss_grad_host(Ih, Th, 14.2857, 1.0, scratch, out)
        t0 = time.perf_counter()
        for _ in range(3):
            K.infcl_loss_grad_host(Ih, Th, 14.2857, 1.0, scratch, out)
        res[v].append((time.perf_counter() - t0) / 3 * 1e3)
        losses[v] = float(out[0])
print(json.dumps({v: {"median_ms": statistics.median(x), "all": [round(y, 3) for y in x]} for v, x in res.items()}
                 | {"loss": losses}))
