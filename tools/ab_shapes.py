"""Isolated launch times of the ViT-B/16 b256 GEMM shapes (bf16), protected vs unprotected,
median of CUDA-event-timed launches, L2 flushed between launches; run per library via $GEMMGUARD_LIB."""
import os, statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K, _lib as L
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device='cuda')
shapes = [("qkv", 50432, 2304, 768, 0), ("proj", 50432, 768, 768, 0), ("fc1", 50432, 3072, 768, 0),
          ("fc1+gelu", 50432, 3072, 768, 1), ("fc2", 50432, 768, 3072, 0)]
rows = []
for name, M, N, Kd, act in shapes:
    x = torch.randn(M, Kd, device='cuda').bfloat16(); w = (torch.randn(N, Kd, device='cuda') / Kd**.5).bfloat16()
    b = torch.zeros(N, device='cuda'); ws, bs = K.offline_checksum(w, b, L.GG_P_F64); bsv = bs.item()
    aux = K.checksum_aux(ws, torch.bfloat16); y = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
    res = K.CheckResult.empty(M, False, 'cuda')
    pred = torch.zeros(M, dtype=torch.int64, device='cuda')
    def run(prot):
        if prot: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, act=act, out=y, result=res,
                                  pred_in=pred if prot == 2 else None)
        else: K.protected_gemm(x, w, b, protect=False, act=act, out=y)
    t = {0: [], 1: [], 2: []}
    for it in range(30):
        for prot in ((0, 1, 2) if it % 2 else (2, 1, 0)):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(prot); e1.record(); torch.cuda.synchronize()
            if it >= 4: t[prot].append(e0.elapsed_time(e1) * 1e3)
    u, p, q = statistics.median(t[0]), statistics.median(t[1]), statistics.median(t[2])
    rows.append(f"{name:9s} unprot {u:7.1f} us  prot {p:7.1f} us  overhead {100*(p/u-1):5.1f}%  | with pred_in {q:7.1f} us {100*(q/u-1):5.1f}%")
print(os.environ.get('GEMMGUARD_LIB', 'default').split('/')[-1]); print("\n".join(rows))
