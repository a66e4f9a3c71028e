"""Diagnose the TS (A in TMEM) layout: structured operands reveal which A element each TMEM output reads."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2410_17243_b200 import _lib as L
K = 64
def run(A, B, mode):
    out = torch.full((2, 128, 128), float("nan"), device="cuda")
    Bd = (B.t().contiguous() if mode & 1 else B).bfloat16().cuda()
    L.diag_call("infcl_probe_umma_ts", A.bfloat16().cuda().data_ptr(), Bd.data_ptr(), K, mode, out.data_ptr(),
                torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu()
res = {}
for mode in (1, 0):
    # B = [I_K | 0] (K x 256): D[m][n] = A_eff[m][n], n < K.  A[r][k] = code(r, k) exactly representable in bf16:
    # probe rows one at a time would be slow; use A[r][k] = 1 iff k == r % K, then A[r][k] = r % 8 + 1 for k < 8
    B = torch.zeros(K, 256); B[torch.arange(K), torch.arange(K)] = 1
    A1 = torch.zeros(128, K); A1[torch.arange(128), torch.arange(128) % K] = 1
    o = run(A1, B, mode)
    res[mode] = o
    print(f"mode {mode} (B {'K' if mode & 1 else 'MN'}-major), A one-hot k = r % 64, B = identity:")
    for c in range(2):
        desc = []
        for lane in range(0, 128, 4):
            nz = (o[c, lane] != 0).nonzero().flatten().tolist()
            desc.append(f"{lane}:{nz[:3]}")
        print(f"  cta{c}", " ".join(desc))
    # A random small ints, B identity -> compare
    g = torch.Generator().manual_seed(1)
    A2 = torch.randint(-8, 8, (128, K), generator=g).float()
    o2 = run(A2, B, mode)
    ok = True
    for c in range(2):
        rows = A2[64 * c:64 * c + 64]
        full = torch.zeros(64, 256); full[:, :K] = rows
        exp = torch.cat([full[:, :128], full[:, 128:]], 0)
        ok &= torch.equal(o2[c], exp)
    print(f"  random-A identity-B exact: {ok}")
torch.save(res, "gpurun_out/ts_diag.pt")
