"""Protected-GEMM timing under the GG_DEBUG diagnostic switches (one shape)."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in sys.argv[1:4]]
x = torch.randn(M, Kd, device='cuda').to(torch.bfloat16); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).to(torch.bfloat16)
b = torch.zeros(N, device='cuda')
ws, bs = K.offline_checksum(w, b, L.GG_P_F64); aux = K.checksum_aux(ws, torch.bfloat16); bsv = bs.item()
y = torch.empty(M, N, dtype=torch.bfloat16, device='cuda'); res = K.CheckResult.empty(M, False, 'cuda')
def t(fn, iters=30):
    for _ in range(5): fn()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / iters * 1e3
tu = t(lambda: K.protected_gemm(x, w, b, protect=False, out=y))
tp = t(lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, out=y, result=res))
print(f"GG_DEBUG={os.environ.get('GG_DEBUG', '0')} {M}x{N}x{Kd}: unprot {tu:7.1f}us prot {tp:7.1f}us overhead {100*(tp/tu-1):6.1f}%", flush=True)
