"""Small launches of every K1 path and the auxiliary kernels, for compute-sanitizer."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
for (M, N, Kd) in ((197, 768, 256), (1576, 768, 256), (3000, 1000, 300)):
    x = torch.randn(M, Kd, device=dev, generator=g).bfloat16()
    w = (torch.randn(N, Kd, device=dev, generator=g) / Kd ** 0.5).bfloat16()
    b = 0.02 * torch.randn(N, device=dev, generator=g)
    ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
    h = torch.randn(M, N, device=dev, generator=g).bfloat16()
    y, r = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30)
    y2, r2 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30, residual=h)
    y3, r3 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30, act=L.GG_ACT_GELU_TANH)
    thr = 4 * float(r.d.abs().max().item()) + 1e-6
    y4, r4 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-thr, hi=thr,
                              injections=[K.Injection(row=M // 2, col=N // 2, bit=14)])
    K.replay_tiles(x, w, b, y4, r4.flags.clone(), r4, w_sum=ws, bias_sum=bs.item(), lo=-thr, hi=thr)
    y5, r5 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-thr, hi=thr,
                              injections=[K.Injection(row=M // 3, col=N // 3, bit=14)])
    K.replay_located(x, w, b, y5, r5, w_sum=ws, bias_sum=bs.item(), lo=-thr, hi=thr)
    xi = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device=dev, generator=g)
    wi = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device=dev, generator=g)
    bi = torch.randint(-64, 65, (N,), dtype=torch.int32, device=dev, generator=g)
    wsi, bsi = K.offline_checksum(wi, bi, L.GG_P_I64)
    K.protected_gemm(xi, wi, bi, w_sum=wsi, bias_sum=int(bsi.item()), lo=0, hi=0, out_dtype=torch.int8,
                     requant_shift=9, act=L.GG_ACT_RELU)
    K.protected_gemm_wt(xi, wi.t().contiguous(), bi, w_sum=wsi, bias_sum=int(bsi.item()), lo=0, hi=0)
img = torch.randn(2, 3, 224, 224, device=dev, generator=g).bfloat16()
pt = torch.empty(2 * 196, 768, device=dev, dtype=torch.bfloat16)
K.patchify(img, 16, pt)
hh = torch.empty(2 * 197, 768, device=dev, dtype=torch.bfloat16); aa = torch.empty_like(hh)
K.embed_layernorm(pt, torch.randn(197, 768, device=dev).bfloat16(), torch.randn(768, device=dev).bfloat16(),
                  torch.ones(768, device=dev), torch.zeros(768, device=dev), 1e-6, h_out=hh, ln_out=aa)
torch.cuda.synchronize()
print("sanitize paths done")
