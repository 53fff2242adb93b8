"""(Use the diagnostics build for GG_DEBUG switches: GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_diag.so)
Protected vs unprotected timing of one shape: each arm is a CUDA graph of G launches, and
the two graphs are replayed alternately R times (both arms see the same clock / power-cap
state; no host launch overhead).  GG_DEBUG selects the diagnostic switches (read once per
process).  Usage: dbg_perf.py M N K [R] [bf16|i8|f16|tf32]"""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in sys.argv[1:4]]
R = int(sys.argv[4]) if len(sys.argv) > 4 else 12
G = int(min(64, max(4, 3e-3 / (2 * M * N * Kd / 1.2e15))))  # ~3 ms of work per graph replay
dt = {'bf16': torch.bfloat16, 'i8': torch.int8, 'f16': torch.float16, 'tf32': torch.float32}[sys.argv[5] if len(sys.argv) > 5 else 'bf16']
if dt == torch.int8:
    x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device='cuda'); w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device='cuda')
    b = torch.zeros(N, dtype=torch.int32, device='cuda'); prec = L.GG_P_I64
else:
    x = torch.randn(M, Kd, device='cuda').to(dt); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).to(dt)
    b = torch.zeros(N, device='cuda'); prec = L.GG_P_F64
ws, bs = K.offline_checksum(w, b, prec); aux = K.checksum_aux(ws, dt); bsv = bs.item()
y = torch.empty(M, N, dtype=K.default_out_dtype(dt), device='cuda'); res = K.CheckResult.empty(M, dt == torch.int8, 'cuda')
lo, hi = (0, 0) if dt == torch.int8 else (-1e30, 1e30)
unprot = lambda: K.protected_gemm(x, w, b, protect=False, out=y)
prot = lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=lo, hi=hi, out=y, result=res)
graphs = []
for fn in (unprot, prot):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(G): fn()
    graphs.append(g)
for g in graphs: g.replay()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * R + 1)]
ev[0].record()
for i in range(R):
    graphs[0].replay(); ev[2 * i + 1].record()
    graphs[1].replay(); ev[2 * i + 2].record()
torch.cuda.synchronize()
tu = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(R)) / (R * G) * 1e3
tp = sum(ev[2 * i + 1].elapsed_time(ev[2 * i + 2]) for i in range(R)) / (R * G) * 1e3
print(f"GG_DEBUG={os.environ.get('GG_DEBUG', '0'):>2} {M}x{N}x{Kd} {dt}: unprot {tu:7.1f}us prot {tp:7.1f}us overhead {100*(tp/tu-1):6.1f}%  (G={G})", flush=True)
