"""proj / fc2 (ViT-B b256 bf16): K1 storing y vs storing residual + y (fused residual update),
protected and unprotected, plus the layer norm with and without its residual add."""
import statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device='cuda')
def t(fn, n=20):
    out = []
    for _ in range(n):
        flush.zero_(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); out.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(out[3:])
M = 50432
for name, N, Kd in (("proj", 768, 768), ("fc2", 768, 3072)):
    x = torch.randn(M, Kd, device='cuda').bfloat16(); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).bfloat16()
    b = torch.zeros(N, device='cuda'); ws, bs = K.offline_checksum(w, b, L.GG_P_F64); aux = K.checksum_aux(ws, torch.bfloat16)
    h = torch.randn(M, N, device='cuda').bfloat16(); y = torch.empty_like(h); res = K.CheckResult.empty(M, False, 'cuda')
    kw = dict(w_sum=ws, w_aux=aux, bias_sum=bs.item(), lo=-1e30, hi=1e30, out=y, result=res)
    r = {"plain prot": t(lambda: K.protected_gemm(x, w, b, **kw)),
         "residual prot": t(lambda: K.protected_gemm(x, w, b, residual=h, **kw)),
         "plain unprot": t(lambda: K.protected_gemm(x, w, b, protect=False, out=y)),
         "residual unprot": t(lambda: K.protected_gemm(x, w, b, protect=False, out=y, residual=h))}
    print(name, {k: round(v, 1) for k, v in r.items()})
g = torch.ones(768, device='cuda'); be = torch.zeros(768, device='cuda')
h = torch.randn(M, 768, device='cuda').bfloat16(); y = torch.randn_like(h); a = torch.empty_like(h); h2 = torch.empty_like(h)
print("layernorm", {"add+ln": round(t(lambda: K.add_layernorm(h, y, g, be, 1e-6, ln_out=a, h_out=h2)), 1),
                    "ln only": round(t(lambda: K.add_layernorm(h, None, g, be, 1e-6, ln_out=a)), 1)})
