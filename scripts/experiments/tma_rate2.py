"""TMA path probe 2: 2D tensor boxes vs 1D bulk copies (pre-swizzled tile images), per-SM B/clk vs stages."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
n, d = 65536, 512
X = torch.randn(n, d, device="cuda").to(torch.bfloat16)
out = torch.zeros(148, dtype=torch.int64, device="cuda")
names = {0: "2x 2D box[64x128] SW128", 1: "2x 1D bulk 16 KB", 2: "1x 1D bulk 32 KB"}
for nb in (148,):
    for ns in (3, 4, 6):
        for mode in (0, 1, 2):
            iters = 4000
            rc = L.infcl_diag_tma_rate2(ctypes.c_void_p(X.data_ptr()), n, d, mode, ns, iters, nb, ctypes.c_void_p(out.data_ptr()))
            cyc = out[:nb].float().mean().item()
            print(f"blocks={nb} ns={ns} {names[mode]:26s} rc={rc} {iters*32768/cyc:6.1f} B/clk/SM", flush=True)
