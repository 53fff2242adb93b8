"""A/B of the fused-GELU epilogue: fc1 50432x3072x768 bf16, act none / gelu, protect 0 / 1,
median of CUDA-event-timed launches (run once per library via $GEMMGUARD_LIB)."""
import os, statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = 50432, 3072, 768
x = torch.randn(M, Kd, device='cuda').bfloat16(); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).bfloat16()
b = torch.zeros(N, device='cuda'); ws, bs = K.offline_checksum(w, b, L.GG_P_F64); bsv = bs.item()
aux = K.checksum_aux(ws, torch.bfloat16); y = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
res = K.CheckResult.empty(M, False, 'cuda')
def run(act, prot):
    if prot: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, act=act, out=y, result=res)
    else: K.protected_gemm(x, w, b, protect=False, act=act, out=y)
out = {}
for act in (L.GG_ACT_NONE, L.GG_ACT_GELU_TANH):
    for prot in (0, 1):
        for _ in range(5): run(act, prot)
        ts = []
        for _ in range(40):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(act, prot); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
        out[(act, prot)] = statistics.median(ts)
lib = os.environ.get('GEMMGUARD_LIB', 'default')
print(lib.split('/')[-1], ' '.join(f"act{a}/p{p}={v:.1f}us" for (a, p), v in out.items()),
      f"gelu cost unprot {out[(1,0)]-out[(0,0)]:.1f} prot {out[(1,1)]-out[(0,1)]:.1f}")
