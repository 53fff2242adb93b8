"""Small-M (cfg2 B=1, M = 197) protected vs unprotected launch time, CUDA graphs of
`reps` launches, alternating rounds.  Run under the diagnostics library with
GG_DEBUG=<bits> to switch parts of the protected kernel off (breakdown).

    GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_diag.so GG_DEBUG=4 \
        python tools/small_m.py
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_configs import interleaved  # noqa: E402
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402

DEV = torch.device("cuda")
M = int(os.environ.get("SMALL_M", 197))
out = {"dbg": os.environ.get("GG_DEBUG", "0"), "M": M, "lib": Path(L.load()._name).name}
for kind in ("int8", "bf16"):
    for (Kd, N) in ((768, 768), (768, 2304), (768, 3072), (3072, 768)):
        g = torch.Generator(device=DEV).manual_seed(N + Kd)
        if kind == "int8":
            x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device=DEV, generator=g)
            w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device=DEV, generator=g)
            b = torch.randint(-64, 65, (N,), dtype=torch.int32, device=DEV, generator=g)
            ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
            y = torch.empty(M, N, dtype=torch.int32, device=DEV)
            bsv = int(bs.item())
        else:
            x = torch.randn(M, Kd, device=DEV, generator=g).to(torch.bfloat16)
            w = (torch.randn(N, Kd, device=DEV, generator=g) / Kd ** 0.5).to(torch.bfloat16)
            b = torch.zeros(N, device=DEV)
            ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
            y = torch.empty(M, N, dtype=torch.bfloat16, device=DEV)
            bsv = float(bs.item())
        aux = K.checksum_aux(ws, x.dtype)
        res = K.CheckResult.empty(M, kind == "int8", DEV)
        tu, tp = interleaved([lambda: K.protected_gemm(x, w, b, protect=False, out=y),
                              lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30,
                                                       out=y, result=res)], 64, rounds=10)
        out[f"{kind} {N}x{Kd}"] = [round(tu, 2), round(tp, 2), round(100 * (tp / tu - 1), 1)]
print(json.dumps(out))
