"""proj (50432 x 768 x 768 bf16) protected vs unprotected under the diagnostics library's
$GG_DEBUG switches (one process per setting): which part of the protected kernel costs."""
import os, statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in os.environ.get("SHAPE", "50432,768,768").split(",")]
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device='cuda')
x = torch.randn(M, Kd, device='cuda').bfloat16(); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).bfloat16()
b = torch.zeros(N, device='cuda'); ws, bs = K.offline_checksum(w, b, L.GG_P_F64); bsv = bs.item()
aux = K.checksum_aux(ws, torch.bfloat16); y = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
res = K.CheckResult.empty(M, False, 'cuda')
t = {0: [], 1: []}
for it in range(40):
    for prot in ((0, 1) if it % 2 else (1, 0)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if prot: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, out=y, result=res)
        else: K.protected_gemm(x, w, b, protect=False, out=y)
        e1.record(); torch.cuda.synchronize()
        if it >= 6: t[prot].append(e0.elapsed_time(e1) * 1e3)
u, p = statistics.median(t[0]), statistics.median(t[1])
print(f"dbg={os.environ.get('GG_DEBUG', '0'):6s} {M}x{N}x{Kd} unprot {u:6.1f} prot {p:6.1f} overhead {100 * (p / u - 1):5.1f}%")
