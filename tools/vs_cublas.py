"""Our unprotected K1 (protect = 0, the overhead baseline) and the protected K1 against cuBLAS
(torch.matmul + bias) on the ViT-B/16 b256 GEMM shapes, bf16, L2 flushed between launches."""
import statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device='cuda')
for name, M, N, Kd in (("qkv", 50432, 2304, 768), ("proj", 50432, 768, 768), ("fc1", 50432, 3072, 768),
                       ("fc2", 50432, 768, 3072)):
    x = torch.randn(M, Kd, device='cuda').bfloat16(); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).bfloat16()
    b = torch.zeros(N, device='cuda'); bb = b.bfloat16(); y = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
    ws, bs = K.offline_checksum(w, b, L.GG_P_F64); aux = K.checksum_aux(ws, torch.bfloat16); bsv = bs.item()
    res = K.CheckResult.empty(M, False, 'cuda')
    fns = {"cublas": lambda: torch.addmm(bb, x, w.t(), out=y),
           "k1_unprotected": lambda: K.protected_gemm(x, w, b, protect=False, out=y),
           "k1_protected": lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30,
                                                    out=y, result=res)}
    t = {k: [] for k in fns}
    for it in range(24):
        for k in (list(fns) if it % 2 else list(fns)[::-1]):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fns[k](); e1.record(); torch.cuda.synchronize()
            if it >= 4: t[k].append(e0.elapsed_time(e1) * 1e3)
    f = 2 * M * N * Kd
    print(name, "  ".join(f"{k} {statistics.median(v):7.1f} us {f / statistics.median(v) / 1e6:6.0f} TF/s" for k, v in t.items()))
