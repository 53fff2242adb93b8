"""Tail of a tiny protected launch (M <= 256) from the GG_TRACE library: per CTA the
epilogue / reducer stamps and, for the last arriver, the split of its fold.

    GEMMGUARD_LIB=paper_2310_03841_b200/_variants/libgemmguard_b200_trace.so \
        python tools/trace_tiny.py M N K [bf16|int8]
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200 import _lib as L, kernels as K  # noqa: E402

M, N, Kd = [int(v) for v in sys.argv[1:4]]
kind = sys.argv[4] if len(sys.argv) > 4 else "bf16"
dev = torch.device("cuda")
if kind == "int8":
    x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device=dev)
    w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device=dev)
    b = torch.zeros(N, dtype=torch.int32, device=dev)
    ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
    y = torch.empty(M, N, dtype=torch.int32, device=dev)
    bsv = int(bs.item())
else:
    x = torch.randn(M, Kd, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, Kd, device=dev) / Kd ** 0.5).to(torch.bfloat16)
    b = torch.zeros(N, device=dev)
    ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
    y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    bsv = float(bs.item())
aux = K.checksum_aux(ws, x.dtype)
res = K.CheckResult.empty(M, kind == "int8", dev)
lib = L.load()
lib.gg_trace_buffer.argtypes = [ctypes.c_void_p]
TT, EV = 64, 28
buf = torch.zeros(148 * TT * EV + 4 * 64 * 4, dtype=torch.int64, device=dev)
for protect in (False, True):
    run = (lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e30, hi=1e30, out=y,
                                    result=res)) if protect else (lambda: K.protected_gemm(x, w, b, protect=False,
                                                                                           out=y))
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    buf.zero_()
    lib.gg_trace_buffer(ctypes.c_void_p(buf.data_ptr()))
    run()
    torch.cuda.synchronize()
    lib.gg_trace_buffer(ctypes.c_void_p(0))
    t = buf.cpu().numpy()[:148 * TT * EV].reshape(148, TT, EV)
    print(f"=== protect={protect}  (cycles from the CTA's mma/epilogue start)")
    for c in range(148):
        r = t[c, 0]
        if not (r[:13] > 0).any():
            continue
        base = r[4] if r[4] > 0 else r[0]
        f = lambda e: int(r[e] - base) if r[e] > 0 else None  # noqa: E731
        line = (f" CTA {c:3d}: mma start 0 end {f(5)} | epi tfull {f(0)} rel {f(1)} done {f(2)} slot {f(3)}"
                f" | chk done {f(6)} slot {f(7)} | red got {f(8)} done {f(9)}")
        if r[24] > 0:
            line += (f" || LAST: before atomic {f(24)} acq_rel add {int(r[25] - r[24])} to closing barrier"
                     f" {int(r[26] - r[25])} all-thread fold + summary {int(r[27] - r[26])}")

        print(line)
