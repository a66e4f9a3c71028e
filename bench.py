#!/usr/bin/env python
"""Benchmark of the Inf-CL loss hot path on B200: loss forward+backward samples/s and peak GB/GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--b B] [--d D]

N=1 runs BASELINE.json configs[1] (b=65536, d=512, bf16); N>1 (one rank per GPU; launched under torchrun, or
spawned by this script through torch.distributed.run when WORLD_SIZE is unset) runs the same global batch as a
ring over the N GPUs (strong scaling: the same workload at every N).  A "step" is one full pass of the hot path: infcl_forward (fused S-tile GEMM +
row/column LSE + diagonal, Alg.1/2) and infcl_backward (recompute + dI and dT, Alg.3/4) over the whole batch.
Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle (the only "reference" this paper-only
run has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "loss fwd+bwd samples/s and peak GB/GPU vs batch at 1/2/4/8 B200"
UNIT = "samples/s"
L2_FLUSH_BYTES = 512 << 20


def max_over_ranks(x: float) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 50 ms DURING the timed region (B200_PROFILING.md clocks line).  Started before the
    warm-up steps and awaited (first sample) before the timed loop: nvidia-smi's start-up takes the driver for up to
    ~100 ms, which, inside the timed loop, stalled kernel launches and left the GPU idle (a 1.5-6.7 ms/step swing
    between back-to-back runs).  Only samples that arrive inside the timed window are summarised."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def wait_first(self, timeout: float = 10.0):
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)

    def window(self, t0: float, t1: float):
        self.t0, self.t1 = t0, t1

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        lines = [ln for (t, ln) in self.lines if t0 is None or t0 <= t <= t1 + 0.05]
        if not lines:  # a window shorter than the sampling period: the samples around it
            lines = [ln for (t, ln) in self.lines if t0 is None or t0 - 0.1 <= t <= t1 + 0.1]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw)}


# ------------------------------------------------------------------------------------------------ oracle (CPU)
def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def oracle_sample(I_host, T_host, s: float, rows: int) -> float:
    """Time the fp64 oracle (as it stands) on rows [0, rows) of the workload: forward row LSE + column-LSE
    partial over all b columns, and the dI and dT gradient rows for those rows.  Returns seconds."""
    import oracle
    t0 = time.perf_counter()
    f = oracle.streamed_forward(I_host, T_host, s, chunk=min(rows, 512), row_limit=rows)
    b = I_host.shape[0]
    r = f["r"]
    rr = __import__("numpy").concatenate([r, __import__("numpy").zeros(b - rows)])
    sel = list(range(rows))
    oracle.sampled_row_grads(I_host, T_host, s, rr, f["c"], sel)
    oracle.sampled_row_grads(T_host, I_host, s, f["c"], rr, sel)
    return time.perf_counter() - t0


def calibrate_rows(I_host, T_host, s: float, seconds: float) -> int:
    probe = 64
    t = oracle_sample(I_host, T_host, s, probe)
    rows = int(max(64, min(I_host.shape[0], probe * seconds / max(t, 1e-3))))
    return rows - rows % 64 if rows > 64 else rows


def cpu_baseline(I_host, T_host, s: float, seconds: float) -> dict:
    rows = calibrate_rows(I_host, T_host, s, seconds)
    t = oracle_sample(I_host, T_host, s, rows)
    b, d = I_host.shape
    return {"value": rows / t, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
            "sample": f"fp64 numpy oracle on image rows [0,{rows}) of the b={b}, d={d} batch: row LSE + column-LSE "
                      f"partial over all {b} columns, dI and dT rows; {t:.1f} s; value = rows/s = projected b/t_full "
                      "(oracle time is linear in rows)"}


# ------------------------------------------------------------------------------------------------ workloads
def workload(args, world):
    b = args.b if args.b else 65536
    d = args.d if args.d else 512
    name = f"cfg2 CLIP-ViT-B/16 shape: b={b}, d={d}, bf16" if (b, d) == (65536, 512) else f"custom b={b}, d={d}"
    if (b, d) == (262144, 768):
        name = f"cfg3 CLIP-ViT-L/14 shape: b={b}, d={d}, bf16"
    return b, d, name


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import make_features
    world = args.gpus
    b, d, name = workload(args, world)
    I_host, T_host = make_features(b, d, seed=args.seed)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rows = calibrate_rows(I_host, T_host, args.scale, per_step)
    for _ in range(args.warmup):
        oracle_sample(I_host, T_host, args.scale, rows)
    ts = [oracle_sample(I_host, T_host, args.scale, rows) for _ in range(args.steps)]
    t = statistics.mean(ts)
    value = rows / t
    cb = {"value": value, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
          "sample": f"each step: fp64 oracle on image rows [0,{rows}) of b={b}, d={d} (fwd row LSE + column "
                    "partial over all columns, dI and dT rows); value = rows/s = projected b / t_full"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": name, "b": b, "d": d, "logit_scale": args.scale, "parallelism": "cpu-oracle"},
           "impl": "reference", "cpu_baseline": cb,
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------------ our arm
def run_ours(args):
    from paper_2410_17243_b200 import _lib as L
    from paper_2410_17243_b200 import loss as K
    from synth import make_features_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # INFCL_BENCH_SAME_GPU=1 (test only): every rank on cuda:0 with a gloo process group, to exercise the N>1
    # path (IPC transport, timing reduction, JSON line) on a one-GPU box; its numbers are not throughput
    same_gpu = os.environ.get("INFCL_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    comm = None
    b, d, name = workload(args, world)
    if b % world:
        raise SystemExit(f"b={b} not divisible by world={world}")
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            comm = K.RingComm(transport=args.transport, max_b=b, max_d=d)
        except L.InfclError as e:  # e.g. no peer access between these GPUs: the NCCL transport still works
            if args.transport != "ipc":
                raise
            print(f"bench: IPC ring transport unavailable ({e}); using NCCL", file=sys.stderr, flush=True)
            args.transport = "nccl"
            comm = K.RingComm(transport="nccl")
    bs = b // world
    s = args.scale
    dev = torch.device("cuda", local)
    I, T = make_features_device(bs, d, seed=args.seed * 1000 + rank, device=dev)
    ws = K.alloc_workspace(b, d, world, torch.bfloat16, dev, comm=comm)
    g = torch.ones((), device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    region = comm.region_bytes() if comm else 0

    def step():
        loss, r, c, dg = K.infcl_forward(I, T, b, s, rank, world, comm, ws)
        dI, dT = K.infcl_backward(I, T, b, s, r, c, dg, g, rank, world, comm, ws)
        return loss, dI, dT

    clk = ClockSampler(local).__enter__()  # before the warm-up: its start-up must not overlap the timed loop
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clk.wait_first()
    # peak memory of ONE call (the paper's loss memory M_loss, Eq.9): outputs of earlier steps released,
    # the L2-flush buffer (a benchmark artefact) excluded; counts the I, T shards, the workspace, r, c, diag,
    # dI, dT, and the library-owned IPC receive region
    if world > 1:
        dist.barrier()
    torch.cuda.reset_peak_memory_stats(dev)
    out1 = step()
    torch.cuda.synchronize()
    peak_call = torch.cuda.max_memory_allocated(dev) - flush.numel() + region
    del out1
    lib = L.lib()
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    lib.infcl_reset_launch_count()
    lib.infcl_profile_enable(1)
    try:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        gc.disable()  # no collector pause while the host enqueues the timed steps
        t_win0 = time.time()
        # ~10 ms of device-side sleep ahead of the first step (outside every step's events): the host enqueues the
        # timed steps meanwhile, so a host-side stall (another process polling the driver) cannot leave the GPU idle
        # inside a step; each step's events still bracket exactly its own kernels
        torch.cuda._sleep(int(2e7))
        for e0, e1, e2 in evs:
            flush.zero_()  # L2 flush between timed steps (outside the per-step events)
            e0.record(stream)
            loss, r, c, dg = K.infcl_forward(I, T, b, s, rank, world, comm, ws)
            e1.record(stream)
            dI, dT = K.infcl_backward(I, T, b, s, r, c, dg, g, rank, world, comm, ws)
            e2.record(stream)
        host_enqueue_ms = (time.time() - t_win0) * 1e3
        torch.cuda.synchronize()
        clk.window(t_win0, time.time())
        if world > 1:
            dist.barrier()
    finally:
        gc.enable()
        clk.__exit__(None, None, None)
    launches = int(lib.infcl_launch_count())
    import ctypes
    prof = {}
    for kind in (0, 1, 2):
        n = ctypes.c_int()
        ms = ctypes.c_double()
        L.call("infcl_profile_read", kind, ctypes.byref(n), ctypes.byref(ms))
        prof[kind] = (n.value, ms.value)
    lib.infcl_profile_enable(0)
    fwd_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in evs) / args.steps
    bwd_ms = sum(e1.elapsed_time(e2) for _, e1, e2 in evs) / args.steps
    local_step_ms = fwd_ms + bwd_ms
    ms_step = max_over_ranks(local_step_ms)
    fwd_ms = max_over_ranks(fwd_ms)
    bwd_ms = max_over_ranks(bwd_ms)
    peak_gb = max_over_ranks(peak_call / 1e9)
    value = b / (ms_step / 1e3)
    lval = float(loss.item())

    # roofline of the dominant kernel (the backward pair kernel: 1 fused launch or 2 passes per ring step).  Denominator
    # (B200_PROFILING.md): the BURST cuBLAS peak for a kernel in a short step, the SUSTAINED (power-capped) one
    # only once a step lasts a second or more (b >= 512K); both fractions are reported
    peaks = measured_peaks()
    burst = peaks.get("bf16_tflops") or 1590.0
    sustained = peaks.get("bf16_tflops_sustained") or 1400.0
    src = "MEASURED_PEAKS.json" if "bf16_tflops" in peaks else "fallback (B200_PROFILING.md)"
    long_step = ms_step >= 1000.0
    peak = sustained if long_step else burst
    peak_src = f"{src} {'bf16_tflops_sustained' if long_step else 'bf16_tflops (burst)'}: step of {ms_step:.1f} ms " \
               f"{'>=' if long_step else '<'} 1 s"
    kind = 1 if prof[1][1] >= prof[0][1] else 0
    n_l, tot_ms = prof[kind]
    avg_ms = max_over_ranks(tot_ms / max(n_l, 1))
    if kind == 1:
        # algorithmic backward per rank and step: 6 b_s^2 d per ring step (S recompute + dI + dT), world steps; the
        # fused single-pass kernel is 1 launch per ring step, the two-pass backward 2 (dI and dT pass)
        per_step = n_l / args.steps
        flop_per_launch = 6.0 * bs * bs * d * world / per_step
        if per_step <= world:
            kname = ("pair_kernel<BWD,GC> (fused single-pass backward: producer pairs S recompute + G + dI GEMM, "
                     "consumer pairs dT GEMM from the G ring)")
        else:
            kname = "pair_kernel<BWD> (S recompute + G + dA GEMM; one pass of the two-pass backward)"
    else:
        flop_per_launch = 2.0 * bs * bs * d
        kname = "pair_kernel<FWD> (S GEMM + row/col LSE + diag)"
    achieved = flop_per_launch / (avg_ms / 1e3) / 1e12
    tkey = f"{'bwd' if kind == 1 else 'fwd'}_{b}_{d}_{world}"
    if kind == 1 and n_l / args.steps <= world:
        tkey = f"bwdfused_{b}_{d}_{world}"
    traffic = ncu_traffic().get(tkey)
    step_tf = 8.0 * b * b * d / world / (ms_step / 1e3) / 1e12
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": kname, "avg_launch_ms": avg_ms, "launches": n_l,
            "algorithmic_flop_per_launch": flop_per_launch, "peak_source": peak_src,
            "frac_burst": achieved / burst, "frac_sustained": achieved / sustained,
            "step_tflops_8b2d": step_tf, "step_frac_burst": step_tf / burst}
    # time of the step outside the two pair kernels (small merge/finish kernels, launch gaps and, at N > 1, the
    # ring exchange not hidden behind a kernel): per rank, max over ranks
    kern_ms = (prof[0][1] + prof[1][1]) / args.steps
    non_kernel_ms = max_over_ranks(local_step_ms - kern_ms)

    # ring traffic per rank and step: forward n-1 blocks + n column-state hops; backward two
    # passes of n-1 (block + LSE) hops.  Time-averaged rate = bytes / step time (a lower bound on the link rate
    # while transferring; the exchange overlaps the kernels)
    ring = None
    if world > 1:
        # forward: n-1 blocks + n column-state hops; backward: fused ring (1 launch per ring step) n-1 (block + LSE)
        # hops + n hops of the fp32 dT partial, or the two-pass ring 2 (n-1) (block + LSE) hops
        fused_ring = prof[1][0] / args.steps <= world
        rb = (world - 1) * bs * d * 2 + world * bs * 8 + (
            (world - 1) * (bs * d * 2 + bs * 4) + world * bs * d * 4 if fused_ring
            else 2 * (world - 1) * (bs * d * 2 + bs * 4))
        hops, hop_ms = prof[2]
        hop_bytes = bs * d * 2
        per_hop = max_over_ranks(hop_ms / max(hops, 1))
        ring = {"transport": args.transport, "backward": "fused (dT partials travel)" if fused_ring else "two-pass",
                "bytes_per_rank_per_step": rb,
                "avg_gb_s": rb / (ms_step / 1e3) / 1e9, "link_peak_gb_s": 900.0,
                "avg_frac_of_link": rb / (ms_step / 1e3) / 1e9 / 900.0,
                # per-hop comm-stream events (infcl_profile_read kind 2) around each travelling-block transfer
                "hops_per_step": hops / args.steps, "hop_bytes": hop_bytes, "hop_ms": per_hop,
                "hop_gb_s": hop_bytes / (per_hop / 1e3) / 1e9 if per_hop > 0 else None,
                "hop_frac_of_link": hop_bytes / (per_hop / 1e3) / 1e9 / 900.0 if per_hop > 0 else None,
                "hop_frac_of_measured_p2p": hop_bytes / (per_hop / 1e3) / 1e9 / 770.0 if per_hop > 0 else None,
                # exposed comm: step time outside the pair kernels at this N minus the same quantity at N = 1
                # (measured by bench.py --gpus 1: profiles/) -- here the raw non-kernel time per step
                "non_kernel_ms": non_kernel_ms}

    # end-to-end through the public API with host buffers
    e2e = run_e2e(args, K, b, d, bs, s, rank, world, comm, dev)
    ntx = run_ntxent(args, K, b, d, s, dev, flush) if world == 1 and not args.no_ntxent else None

    out = None
    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(I.cpu(), T.cpu(), s, args.cpu_seconds)
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": {"workload": name, "b": b, "d": d, "logit_scale": s, "parallelism": f"ring{world}" + (f"-{args.transport}" if world > 1 else ""),
                          "l2": "512 MB buffer written between timed steps (outside per-step events)",
                          "inputs": "L2-normalised N(0,1) rows, bf16 RNE, generated on device"},
               "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "non_kernel_ms": non_kernel_ms, "host_enqueue_ms": host_enqueue_ms, "peak_gb_per_gpu": peak_gb,
               "peak_gb_accounting": "one call: I,T shards + workspace + r,c,diag + dI,dT (+ IPC region); "
                                     "outputs of earlier steps released; L2-flush buffer excluded",
               "loss": lval,
               "gpu_launches": launches, "clocks": clk.summary(), "roofline": roof, "cpu_baseline": cb, "e2e": e2e}
        if ring is not None:
            out["ring"] = ring
        if ntx is not None:
            out["second_workload"] = ntx
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return out


def run_ntxent(args, K, b, d, s, dev, flush):
    """The second workload: NT-Xent (SimCLR) over the same number of views as the headline
    workload (b/2 examples x 2 views, d), device-resident, CUDA events per step, L2 flushed between steps."""
    from synth import make_features_device
    bx = b // 2
    A, B = make_features_device(bx, d, seed=args.seed * 1000 + 7, device=dev)
    ws = K.alloc_workspace(bx, d, 1, torch.bfloat16, dev)
    g = torch.ones((), device=dev)

    def step():
        loss, la, lb, pos = K.ntxent_forward(A, B, bx, s, workspace=ws)
        return K.ntxent_backward(A, B, bx, s, la, lb, pos, g, workspace=ws)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    n = max(3, min(args.steps, 10))
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.mean(ts)
    # executed work: forward 3 b_x^2 blocks (2 b_x^2 d each), backward 4 block passes (4 b_x^2 d each)
    flop = (3 * 2 + 4 * 4) * float(bx) * bx * d
    return {"workload": f"NT-Xent (SimCLR) over {2 * bx} views: {bx} examples x 2, d={d}, bf16",
            "metric": "loss fwd+bwd views/s", "value": 2 * bx / (ms / 1e3), "ms_per_step": ms, "steps": n,
            "executed_tflops": flop / (ms / 1e3) / 1e12}


def run_e2e(args, K, b, d, bs, s, rank, world, comm, dev):
    """Same metric through the public API with HOST buffers: H2D of the step's inputs (pinned), fwd+bwd,
    D2H of loss and gradients, every step inside the timed region."""
    from synth import make_features_device
    Ih, Th = make_features_device(bs, d, seed=77 + rank, device=dev)
    Ih = Ih.cpu().pin_memory()
    Th = Th.cpu().pin_memory()
    steps = max(2, min(args.steps, 5))
    h2d = 2 * bs * d * 2 * world
    d2h = (4 + 2 * bs * d * 4) * world
    times = []
    if world == 1:
        scratch = torch.empty(int(K.L.lib().infcl_e2e_scratch_bytes(b, d, 0)), dtype=torch.uint8, device=dev)
        out = (torch.empty((), dtype=torch.float32).pin_memory(), torch.empty(b, d, dtype=torch.float32).pin_memory(),
               torch.empty(b, d, dtype=torch.float32).pin_memory())
        K.infcl_loss_grad_host(Ih, Th, s, 1.0, scratch, out)
        for _ in range(steps):
            t0 = time.perf_counter()
            K.infcl_loss_grad_host(Ih, Th, s, 1.0, scratch, out)
            times.append(time.perf_counter() - t0)
    else:
        ws = K.alloc_workspace(b, d, world, torch.bfloat16, dev, comm=comm)
        g = torch.ones((), device=dev)
        dIh = torch.empty(bs, d, dtype=torch.float32).pin_memory()
        dTh = torch.empty_like(dIh)
        lh = torch.empty((), dtype=torch.float32).pin_memory()
        for it in range(steps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            I = Ih.to(dev, non_blocking=True)
            T = Th.to(dev, non_blocking=True)
            loss, r, c, dg = K.infcl_forward(I, T, b, s, rank, world, comm, ws)
            dI, dT = K.infcl_backward(I, T, b, s, r, c, dg, g, rank, world, comm, ws)
            lh.copy_(loss, non_blocking=True)
            dIh.copy_(dI, non_blocking=True)
            dTh.copy_(dT, non_blocking=True)
            torch.cuda.synchronize()
            if it:
                times.append(max_over_ranks(time.perf_counter() - t0))
    t = statistics.mean(times)
    return {"value": b / t, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": t * 1e3, "api": "infcl_loss_grad_host" if world == 1 else "infcl_forward/backward + copies"}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--b", type=int, default=0)
    ap.add_argument("--d", type=int, default=0)
    ap.add_argument("--scale", type=float, default=14.2857)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ntxent", action="store_true", help="skip the second-workload (NT-Xent) line")
    ap.add_argument("--transport", choices=["ipc", "nccl"], default="ipc",
                    help="ring transport for N>1: copy-engine writes over CUDA IPC peer memory (default) or NCCL P2P")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this script under torch.distributed.run (rank 0 prints the JSON line)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + \
            (sys.argv[1:] if argv is None else list(argv))
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
