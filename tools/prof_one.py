"""One unprotected + one protected launch of a GEMM shape for ncu (args: M N K dtype [act])."""
import sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
M, N, Kd = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (50432, 768, 3072))]
dt = {'bf16': torch.bfloat16, 'i8': torch.int8, 'f16': torch.float16, 'tf32': torch.float32}[sys.argv[4] if len(sys.argv) > 4 else 'bf16']
act = L.GG_ACT_GELU_TANH if (len(sys.argv) > 5 and sys.argv[5] == 'gelu') else L.GG_ACT_NONE
if dt == torch.int8:
    x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device='cuda'); w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device='cuda'); b = torch.zeros(N, dtype=torch.int32, device='cuda'); prec = L.GG_P_I64
else:
    x = torch.randn(M, Kd, device='cuda').to(dt); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).to(dt); b = torch.zeros(N, device='cuda'); prec = L.GG_P_F64
ws, bs = K.offline_checksum(w, b, prec); bsv = bs.item(); aux = K.checksum_aux(ws, dt, 'tf32')
for _ in range(2):
    K.protected_gemm(x, w, b, protect=False, act=act, f32_mode='tf32')
    K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, act=act, f32_mode='tf32')
torch.cuda.synchronize()
