"""cfg2 int8 shapes: int32 outputs (the reference's) vs the fused requantised int8 outputs
(descriptor requant_shift), protected and unprotected, CUDA graphs of 20 launches."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_configs import interleaved  # noqa: E402
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402

DEV = torch.device("cuda")
for Bi in (1, 64, 256):
    for (Kd, N) in ((768, 768), (768, 2304), (768, 3072), (3072, 768)):
        M = 197 * Bi
        g = torch.Generator(device=DEV).manual_seed(N + Kd)
        x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device=DEV, generator=g)
        w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device=DEV, generator=g)
        b = torch.randint(-64, 65, (N,), dtype=torch.int32, device=DEV, generator=g)
        ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
        aux = K.checksum_aux(ws, torch.int8)
        bsv = int(bs.item())
        y32 = torch.empty(M, N, dtype=torch.int32, device=DEV)
        y8 = torch.empty(M, N, dtype=torch.int8, device=DEV)
        res = K.CheckResult.empty(M, True, DEV)
        rq = dict(requant_shift=10, act=L.GG_ACT_RELU)
        t = interleaved([lambda: K.protected_gemm(x, w, b, protect=False, out=y32),
                         lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, out=y32, result=res),
                         lambda: K.protected_gemm(x, w, b, protect=False, out=y8, **rq),
                         lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, out=y8, result=res, **rq)],
                        20)
        ops = 2 * M * N * Kd
        print(json.dumps({"B": Bi, "M": M, "N": N, "K": Kd, "us_i32_unprot": round(t[0], 2), "us_i32_prot": round(t[1], 2),
                          "us_i8_unprot": round(t[2], 2), "us_i8_prot": round(t[3], 2),
                          "tops_i32_prot": round(ops / t[1] / 1e6, 1), "tops_i8_prot": round(ops / t[3] / 1e6, 1)}))
