"""Does a ring transfer overlap the persistent pair kernel (which holds every SM)?  Times, on one GPU:
(a) the backward pass kernel alone, (b) a 1-GB device-to-device copy alone (cudaMemcpyAsync, the IPC
transport's copy), (c) each beside the pair kernel on a second stream, (d) the same bytes moved by an SM copy kernel (torch copy_, the way
an NCCL kernel moves data) beside the pair kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import loss as K
from synth import make_features_device
b, d = 32768, 512
I, T = make_features_device(b, d, seed=0, device="cuda")
g = torch.ones((), device="cuda")
loss, r, c, dg = K.infcl_forward(I, T, b, 14.2857)
src = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def bwd():
    with torch.cuda.stream(s1):
        K.infcl_backward(I, T, b, 14.2857, r, c, dg, g)


def rt_copy():  # plain cudaMemcpyAsync
    assert K.L.diag().infcl_diag_copy(dst.data_ptr(), src.data_ptr(), src.numel(), 0, s2.cuda_stream) == 0


def sm_copy():
    with torch.cuda.stream(s2):
        dst.copy_(src)


for _ in range(2):
    res = {"bwd": timed(bwd), "memcpy_1GB": timed(rt_copy),
           "sm_copy_1GB": timed(sm_copy), "bwd+memcpy": timed(lambda: (bwd(), rt_copy())), "bwd+sm_copy": timed(lambda: (bwd(), sm_copy()))}
print(json.dumps(res))
