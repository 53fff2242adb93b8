"""Protected vs unprotected throughput over a grid of shapes and operand types (power-capped,
interleaved CUDA graphs as tools/dbg_perf.py).  One JSON line per (dtype, M, N, K).

    python tools/sweep.py [--out profiles/r01_sweep.jsonl]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402

DTYPES = {"bf16": torch.bfloat16, "f16": torch.float16, "i8": torch.int8, "tf32": torch.float32}
MS = (1024, 8192, 50432)
NK = ((768, 768), (3072, 768), (768, 3072), (4096, 4096))


def graph_of(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    return g


def run(dt, M, N, Kd):
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd)
    if dt == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device="cuda", generator=g)
        w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device="cuda", generator=g)
        b = torch.zeros(N, dtype=torch.int32, device="cuda")
        prec, lo, hi = L.GG_P_I64, 0, 0
    else:
        x = torch.randn(M, Kd, device="cuda", generator=g).to(dt)
        w = (torch.randn(N, Kd, device="cuda", generator=g) / Kd**0.5).to(dt)
        b = torch.zeros(N, device="cuda")
        prec, lo, hi = L.GG_P_F64, -1e30, 1e30
    ws, bs = K.offline_checksum(w, b, prec)
    aux = K.checksum_aux(ws, dt)
    bsv = bs.item()
    y = torch.empty(M, N, dtype=K.default_out_dtype(dt), device="cuda")
    res = K.CheckResult.empty(M, dt == torch.int8, "cuda")
    fl = 2 * M * N * Kd
    reps = int(min(64, max(4, 3e-3 / (fl / 1.2e15 + 5e-6))))
    gu = graph_of(lambda: K.protected_gemm(x, w, b, protect=False, out=y), reps)
    gp = graph_of(lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=lo, hi=hi, out=y,
                                           result=res), reps)
    tu = tp = 0.0
    rounds = 6
    for _ in range(rounds):
        for gr, which in ((gu, 0), (gp, 1)):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gr.replay()
            e.record()
            torch.cuda.synchronize()
            if which:
                tp += a.elapsed_time(e)
            else:
                tu += a.elapsed_time(e)
    tu, tp = 1e3 * tu / (rounds * reps), 1e3 * tp / (rounds * reps)
    return {"dtype": [k for k, v in DTYPES.items() if v == dt][0], "M": M, "N": N, "K": Kd, "us_unprot": tu,
            "us_prot": tp, "tflops_unprot": fl / (tu * 1e-6) / 1e12, "tflops_prot": fl / (tp * 1e-6) / 1e12,
            "overhead_pct": 100 * (tp / tu - 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    for name, dt in DTYPES.items():
        for M in MS:
            for N, Kd in NK:
                r = run(dt, M, N, Kd)
                line = json.dumps(r)
                print(line, flush=True)
                if a.out:
                    with open(a.out, "a") as f:
                        f.write(line + "\n")
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
