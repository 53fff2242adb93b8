"""Back-to-back launches of one shape (no sync in between): every launch's d must be
bit-identical to the first and nothing may flag (races in the cross-CTA fold / claim /
summary protocols show up here).  Usage: stress_determinism.py M N K dtype [launches]"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402

M, N, Kd = (int(v) for v in sys.argv[1:4])
dt = {'bf16': torch.bfloat16, 'f16': torch.float16, 'tf32': torch.float32, 'i8': torch.int8}[sys.argv[4]]
n = int(sys.argv[5]) if len(sys.argv) > 5 else 100
g = torch.Generator(device='cuda').manual_seed(1)
if dt == torch.int8:
    x = torch.randint(-128, 128, (M, Kd), dtype=dt, device='cuda', generator=g)
    w = torch.randint(-128, 128, (N, Kd), dtype=dt, device='cuda', generator=g)
    b = torch.zeros(N, dtype=torch.int32, device='cuda'); prec, lo, hi = L.GG_P_I64, 0, 0
else:
    x = torch.randn(M, Kd, device='cuda', generator=g).to(dt)
    w = (torch.randn(N, Kd, device='cuda', generator=g) / Kd ** 0.5).to(dt)
    b = torch.zeros(N, device='cuda'); prec, lo, hi = L.GG_P_F64, -1e30, 1e30
ws, bs = K.offline_checksum(w, b, prec)
outs = [K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=lo, hi=hi) for _ in range(n)]
torch.cuda.synchronize()
d0 = outs[0][1].d.view(torch.int64)
bad = sum(1 for _, r in outs if not torch.equal(r.d.view(torch.int64), d0) or int(r.nflag.item()) != 0)
print(f'{M}x{N}x{Kd} {sys.argv[4]}: {n} launches, {bad} differing or flagged')
sys.exit(1 if bad else 0)
