"""Per-SM TMA streaming throughput for the box shapes the pair kernel could use."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "paper_2410_17243_b200/libinfcl_diag.so"))
n, d = 65536, 512
X = torch.randn(n, d, device="cuda").to(torch.bfloat16)
out = torch.zeros(148, dtype=torch.int64, device="cuda")
names = {0: "2x box[64x64rows] per 16KB", 1: "1x box[64x128rows] per 16KB", 2: "1x 3D box(64,64,2) per 16KB", 3: "2x box[64x128] per 32KB"}
for nb in (148, 74, 16):
    for mode in (0, 1, 2, 3):
        iters = 4000
        rc = L.infcl_diag_tma_rate(ctypes.c_void_p(X.data_ptr()), n, d, mode, iters, nb, ctypes.c_void_p(out.data_ptr()))
        cyc = out[:nb].float().mean().item()
        sb = 32768 if mode == 3 else 16384
        print(f"blocks={nb:3d} {names[mode]:30s} rc={rc} {iters*sb/cyc:6.1f} B/clk/SM  chip {iters*sb*nb/cyc*1.9e9/1e12:6.2f} TB/s @1.9GHz", flush=True)
