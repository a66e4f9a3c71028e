"""Energy and time per backward (NVML total-energy counter around N back-to-back backward calls at cfg2)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, pynvml
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b = int(os.environ.get("B", 65536)); d = int(os.environ.get("D", 512)); n = int(os.environ.get("N", 40))
I, T = make_features_device(b, d, seed=0, device="cuda")
ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
g = torch.ones((), device="cuda")
loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
for _ in range(3):
    K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
torch.cuda.synchronize()
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
clk = []
e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for i in range(n):
    K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
    if i % 8 == 4:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
ev1.record(); torch.cuda.synchronize()
e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
ms = ev0.elapsed_time(ev1) / n
print(json.dumps({"tag": os.environ.get("TAG", ""), "b": b, "d": d, "ms_per_bwd": ms, "J_per_bwd": (e1 - e0) / 1e3 / n,
                  "avg_W": (e1 - e0) / 1e3 / (ms * n / 1e3), "sm_mhz": clk}))
