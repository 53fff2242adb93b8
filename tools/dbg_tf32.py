import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
for dt in (torch.float32, torch.bfloat16, torch.int8):
  for (M, N, Kd) in [(1024, 1024, 1024), (300, 520, 256), (50432, 768, 768)]:
    g = torch.Generator().manual_seed(0)
    if dt == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), generator=g, dtype=torch.int8).cuda(); w = torch.randint(-128, 128, (N, Kd), generator=g, dtype=torch.int8).cuda(); b = torch.zeros(N, dtype=torch.int32).cuda(); prec = L.GG_P_I64
    else:
        x = torch.randn(M, Kd, generator=g).to(dt).cuda(); w = (torch.randn(N, Kd, generator=g) / Kd**.5).to(dt).cuda(); b = torch.zeros(N).cuda(); prec = L.GG_P_F64
    ws, bs = K.offline_checksum(w, b, prec)
    y1, r1 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30); d1 = r1.d.clone()
    y2, r2 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30); d2 = r2.d.clone()
    torch.cuda.synchronize()
    same = torch.equal(d1.view(torch.int64) if d1.dtype == torch.float64 else d1, d2.view(torch.int64) if d2.dtype == torch.float64 else d2)
    if dt == torch.int8:
        ref = (x.cpu().long() @ ws.cpu() + int(bs.item())) - y1.cpu().long().sum(1)
        err = (d1.cpu() - ref).abs().max().item()
    else:
        ref = (x.double() @ ws + bs.double()) - y1.double().sum(1)
        err = ((d1 - ref).abs().max() / ((x.double().abs() @ ws.abs()).max())).item()
    print(dt, M, N, Kd, 'deterministic', same, 'max err vs fp64', err, flush=True)
