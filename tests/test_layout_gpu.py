"""The descriptor's b_layout ("B, ldb, b_layout ([N,K] K-major from torch, or
[K,N] as in the reference)"): GG_B_KN launches on the reference's Wt layout."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int8])
@pytest.mark.parametrize("shape", [(300, 520, 100), (1024, 768, 768)])
def test_reference_weight_layout_matches_k_major(dtype, shape):
    """b_layout = GG_B_KN (the reference's Wt [K, N]): the launcher's transpose into the
    caller's scratch, then the K-major kernel -- outputs and d identical to a K-major launch
    on Wt.T, with K (100 bf16 = 200 B) not a multiple of 16 bytes in the first shape."""
    M, N, Kd = shape
    g = torch.Generator(device="cpu").manual_seed(M + N)
    if dtype == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), generator=g, dtype=torch.int8).cuda()
        wt = torch.randint(-128, 128, (Kd, N), generator=g, dtype=torch.int8).cuda()
        b = torch.randint(-64, 65, (N,), generator=g, dtype=torch.int32).cuda()
        prec = L.GG_P_I64
    else:
        x = torch.randn(M, Kd, generator=g).to(dtype).cuda()
        wt = (torch.randn(Kd, N, generator=g) / Kd**0.5).to(dtype).cuda()
        b = (0.02 * torch.randn(N, generator=g)).float().cuda()
        prec = L.GG_P_F64
    ws, bs = K.offline_checksum(wt, b, prec, layout=1)
    bsv = bs.item()
    y1, r1 = K.protected_gemm_wt(x, wt, b, w_sum=ws, bias_sum=bsv, lo=-1e30, hi=1e30)
    y2, r2 = K.protected_gemm(x, wt.t().contiguous(), b, w_sum=ws, bias_sum=bsv, lo=-1e30, hi=1e30,
                              f32_mode="tf32")
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.uint8), y2.view(torch.uint8))
    assert torch.equal(r1.d.view(torch.int64), r2.d.view(torch.int64))
    yu, _ = K.protected_gemm_wt(x, wt, b, protect=False)
    assert torch.equal(yu.view(torch.uint8), y1.view(torch.uint8))
