"""TMA path probe 3: is the ~75 B/clk/SM streaming cap per-SM ingress or L2 egress?  (a) fewer SMs streaming;
(b) clusters of 2 with .multicast::cluster (each SM still receives 32 KB per stage, L2 sends half)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
L = ctypes.CDLL(os.path.join(ROOT, "paper_2410_17243_b200/libinfcl_diag.so"))
n, d = 65536, 512
X = torch.randn(n, d, device="cuda").to(torch.bfloat16)
out = torch.zeros(148, dtype=torch.int64, device="cuda")
for nb in (148, 74, 36):
    for mode in (0, 1):
        for ns in (4, 6):
            iters = 4000
            out.zero_()
            rc = L.infcl_diag_tma_rate3(ctypes.c_void_p(X.data_ptr()), n, d, mode, ns, iters, nb,
                                        ctypes.c_void_p(out.data_ptr()))
            cyc = out[:nb].float().mean().item()
            print(f"blocks={nb:3d} mode={'multicast' if mode else 'private  '} ns={ns} rc={rc} "
                  f"{iters*32768/cyc:6.1f} B/clk/SM received", flush=True)
