"""Hardware self-test of the UMMA building blocks (TMA SW128 -> tcgen05.mma -> TMEM layouts).

Checks D = A B^T against a plain fp32 torch matmul of the same bf16 values, for 1-CTA M=128 and the
CTA-pair shapes (M=128 "2x2" layout, M=256) with K-major and MN-major A.  These are the layouts the loss
kernels are written against.
"""
import pytest
import torch

from paper_2410_17243_b200 import _lib as L

pytestmark = pytest.mark.gpu


def run_probe(M, N, K, a_mn, ncta, ncols):
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K + a_mn * 11 + ncta)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    Ad = (A.t().contiguous() if a_mn else A).cuda()
    Bd = B.cuda()
    out = torch.full((ncta, 128, ncols), float("nan"), device="cuda")
    L.diag_call("infcl_probe_umma", Ad.data_ptr(), Bd.data_ptr(), M, N, K, a_mn, ncta, 0, out.data_ptr(), ncols,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    return out.cpu(), ref


def close(a, b):
    return torch.allclose(a, b, rtol=1e-3, atol=1e-2)


@pytest.mark.parametrize("N", [128, 256])
@pytest.mark.parametrize("a_mn", [0, 1])
def test_1cta_m128(N, a_mn):
    out, ref = run_probe(128, N, 128, a_mn, 1, N)
    assert close(out[0], ref), (out[0, :2, :8], ref[:2, :8])


@pytest.mark.parametrize("a_mn", [0, 1])
def test_pair_m256(a_mn):
    # D (256 x 128): CTA c holds rows [128c, 128c+128) in lanes 0..127, all N columns
    out, ref = run_probe(256, 128, 128, a_mn, 2, 128)
    assert close(out[0], ref[:128]) and close(out[1], ref[128:]), (out[0, :2, :8], ref[:2, :8])


def test_pair_m128_2x2_layout():
    # D (128 x 256): CTA c holds rows [64c, 64c+64); lanes 0..63 = those rows, columns [0, 128),
    # lanes 64..127 = the same rows, columns [128, 256)  (CUTLASS "2x2" tmem_frg for UMMA_2SM M=128)
    out, ref = run_probe(128, 256, 128, 0, 2, 128)
    for c in range(2):
        rows = ref[64 * c:64 * c + 64]
        exp = torch.cat([rows[:, :128], rows[:, 128:]], dim=0)
        if not close(out[c], exp):
            # diagnostic: find for each lane which (row, col-offset) it matches
            pytest.fail(f"cta {c}: layout mismatch; out[:, :4]={out[c, ::16, :4]} ref rows={ref[::16, :4]}")


@pytest.mark.parametrize("K", [64, 256])
@pytest.mark.parametrize("b_km", [0, 1])
def test_pair_m128_ts_duplicated_a(K, b_km):
    # TS form (A in TMEM, duplicated 2x2 layout; B MN-major from smem), D in the same 2x2 layout as the SS pair M=128
    g = torch.Generator().manual_seed(K)
    A = torch.randn(128, K, generator=g).to(torch.bfloat16)
    B = torch.randn(K, 256, generator=g).to(torch.bfloat16)
    out = torch.full((2, 128, 128), float("nan"), device="cuda")
    Bd = (B.t().contiguous() if b_km else B).cuda()
    L.diag_call("infcl_probe_umma_ts", A.cuda().data_ptr(), Bd.data_ptr(), K, b_km, out.data_ptr(),
                torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.float() @ B.float()
    out = out.cpu()
    for c in range(2):
        rows = ref[64 * c:64 * c + 64]
        exp = torch.cat([rows[:, :128], rows[:, 128:]], dim=0)
        assert close(out[c], exp), (c, out[c, ::16, :4], exp[::16, :4])
