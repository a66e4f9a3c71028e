"""Time forward / backward of the bench workload with CUDA events: median of REPS (default 7) after warm-up."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b = int(os.environ.get("B", 65536)); d = int(os.environ.get("D", 512)); reps = int(os.environ.get("REPS", 7))
I, T = make_features_device(b, d, seed=0, device="cuda")
ws = K.alloc_workspace(b, d, 1, torch.bfloat16, "cuda")
g = torch.ones((), device="cuda")
def run():
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
    e0.record()
    loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857, workspace=ws)
    e1.record()
    dI, dT = K.infcl_backward(I, T, b, 14.2857, r, c, dg, g, workspace=ws)
    e2.record()
    return loss, e0, e1, e2
for _ in range(2): run()
torch.cuda.synchronize()
import threading
clk, pw, reasons, stop = [], [], set(), threading.Event()
def sample():
    try:
        import pynvml
        pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            reasons.add(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
            stop.wait(0.02)
    except Exception as e:  # diagnostics only
        reasons.add(str(e))
th = threading.Thread(target=sample, daemon=True); th.start()
f, bw = [], []
for _ in range(reps):
    loss, e0, e1, e2 = run(); torch.cuda.synchronize()
    f.append(e0.elapsed_time(e1)); bw.append(e1.elapsed_time(e2))
stop.set(); th.join()
print(json.dumps({"tag": os.environ.get("TAG", ""), "b": b, "d": d, "fwd_ms": statistics.median(f), "bwd_ms": statistics.median(bw),
                  "fwd_min": min(f), "bwd_min": min(bw), "loss": loss.item(),
                  "sm_mhz": statistics.median(clk) if clk else None, "watts": max(pw) if pw else None, "reasons": sorted(str(x) for x in reasons),
                  "f": [round(x, 3) for x in f], "bw": [round(x, 3) for x in bw]}))
