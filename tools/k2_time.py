import sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
for (N, Kd) in ((3072, 768), (768, 3072)):
    w = torch.randn(N, Kd, device='cuda').to(torch.bfloat16); b = torch.randn(N, device='cuda')
    for _ in range(3): K.offline_checksum(w, b, L.GG_P_F64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): K.offline_checksum(w, b, L.GG_P_F64)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"K2 W[{N},{Kd}] bf16 -> f64: {us:.1f} us, {N*Kd*2/us/1e3:.1f} GB/s")
