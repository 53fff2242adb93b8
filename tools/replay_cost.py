"""Cost of one detected output fault: K4 band replay vs tile-granular replay (column
checksums place the fault's 256-column tile, K1 recomputes only it, the band's rows are
re-checked) on the ViT-B b256 shapes without a fused activation, bf16 and int8.

    python tools/replay_cost.py        -> one JSON line per (shape, dtype, mode)
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402

dev = torch.device("cuda")
SHAPES = {"qkv": (50432, 2304, 768), "proj": (50432, 768, 768), "fc2": (50432, 768, 3072)}


def ops(M, N, Kd, dtype):
    g = torch.Generator(device=dev).manual_seed(N + Kd)
    if dtype == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device=dev, generator=g)
        w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device=dev, generator=g)
        b = torch.randint(-64, 65, (N,), dtype=torch.int32, device=dev, generator=g)
        ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
        return x, w, b, ws, int(bs.item())
    x = torch.randn(M, Kd, device=dev, generator=g).to(dtype)
    w = (torch.randn(N, Kd, device=dev, generator=g) / Kd ** 0.5).to(dtype)
    b = 0.02 * torch.randn(N, device=dev, generator=g)
    ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
    return x, w, b, ws, float(bs.item())


for name, (M, N, Kd) in SHAPES.items():
    for dtype in (torch.bfloat16, torch.int8):
        x, w, b, ws, bs = ops(M, N, Kd, dtype)
        aux = K.checksum_aux(ws, dtype)
        y, r0 = K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bs, lo=-1e30, hi=1e30, ws_key="rc")
        torch.cuda.synchronize()
        thr = 0.0 if dtype == torch.int8 else 4 * float(r0.d.abs().max().item())
        clean = y.clone()
        inj = K.injections_to_device([K.Injection(row=25000, col=N // 2 + 3, bit=14 if dtype != torch.int8 else 30)],
                                     dev)
        t_gemm = []
        out = {}
        for mode in ("band", "tile") * 6:
            res = K.CheckResult.empty(M, dtype == torch.int8, dev)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bs, lo=-thr, hi=thr, injections=inj, out=y,
                             result=res, ws_key="rc")
            e1.record()
            torch.cuda.synchronize()
            assert bool(res.triggered.item())
            if mode == "band":
                K.replay_tiles(x, w, b, y, res.flags.clone(), res, w_sum=ws, w_aux=aux, bias_sum=bs, lo=-thr, hi=thr,
                               ws_key="rc")
            else:
                K.replay_located(x, w, b, y, res, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr, ws_key="rc", w_aux=aux)
            e2.record()
            torch.cuda.synchronize()
            assert torch.equal(y, clean) and not bool(res.triggered.item())
            t_gemm.append(e0.elapsed_time(e1) * 1e3)
            out.setdefault(mode, []).append(e1.elapsed_time(e2) * 1e3)
        g = statistics.median(t_gemm)
        for mode, ts in out.items():
            print(json.dumps({"shape": name, "M": M, "N": N, "K": Kd, "dtype": str(dtype).split(".")[-1],
                              "replay": mode, "us_per_error": round(statistics.median(ts), 1),
                              "protected_launch_us": round(g, 1),
                              "per_error_pct_of_launch": round(100 * statistics.median(ts) / g, 1)}), flush=True)
