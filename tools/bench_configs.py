"""Measurements for BASELINE.json configs 0, 1, 3, 4 and the missing peaks.

One JSON object per line on stdout (and appended to --out):
  peaks   int8 / fp16 / tf32 dense matmul throughput on this GPU (torch: cuBLAS), burst
  cfg1    fp32 (tf32 tensor cores) 1024^3 protected GEMM, per-layer epsilon from 64 clean draws,
          1000 single-bit output flips (exponent + mantissa bits), one trial per launch
  cfg2    int8 sweep M = 197*B, B in {1, 8, 64, 256}, (K, N) in {(768,768), (768,2304), (768,3072),
          (3072,768)}: protected vs unprotected (interleaved CUDA graphs), TOPS, overhead, roofline
  cfg4    batched injection campaign engine on ViT-L/16 GEMM shapes (fp16 and tf32): B images per
          launch, one output flip per image (distinct rows), per-image detection; trials/s, coverage
  cfg5    Swin-B GEMM set (int8 fc1/fc2, bf16 qkv/proj/merge), batch 32: per-injected-error overhead
          (t_inj+replay - t_clean) / t_clean, replay recomputing only the flagged bands

GEMM-level proxies (no attention / norm glue): stated in each line's "scope".
Usage: python tools/bench_configs.py [--only cfg1,cfg2,...] [--out profiles/r01_configs.jsonl]
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402

DEV = torch.device("cuda", 0)
PEAKS = {}


def emit(obj, out):
    line = json.dumps(obj)
    print(line, flush=True)
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")


def graph_of(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    return g


def interleaved(fns, reps, rounds=8, per_round=False):
    """Per-call time (us) of each fn: CUDA graphs of `reps` calls replayed alternately
    (per_round=True: the list of per-round times per fn instead of the mean)."""
    gs = [graph_of(f, reps) for f in fns]
    for g in gs:
        g.replay()
    torch.cuda.synchronize()
    rows = [[] for _ in gs]
    for _ in range(rounds):
        for i, g in enumerate(gs):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            rows[i].append(1e3 * a.elapsed_time(b) / reps)
    return rows if per_round else [sum(r) / rounds for r in rows]


def best_of(fn, n=10):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e-3


# ---------------------------------------------------------------- peaks
def run_peaks(out):
    n = 8192
    a8 = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=DEV)
    b8 = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=DEV).t()
    t = best_of(lambda: torch._int_mm(a8, b8))
    PEAKS["int8"] = 2 * n**3 / t / 1e12
    h = torch.randn(n, n, device=DEV, dtype=torch.float16)
    t = best_of(lambda: h @ h)
    PEAKS["fp16"] = 2 * n**3 / t / 1e12
    f = torch.randn(n, n, device=DEV)
    torch.backends.cuda.matmul.allow_tf32 = True
    t = best_of(lambda: f @ f)
    torch.backends.cuda.matmul.allow_tf32 = False
    PEAKS["tf32"] = 2 * n**3 / t / 1e12
    emit({"config": "peaks", "how": "torch 8192^3 best of 10 (cuBLAS; _int_mm for int8), burst",
          "int8_tops": PEAKS["int8"], "fp16_tflops": PEAKS["fp16"], "tf32_tflops": PEAKS["tf32"]}, out)


def z_of(c):
    return statistics.NormalDist().inv_cdf((1 + c) / 2)


def calibrate(run, draws, conf):
    """Per-layer epsilon: mu +/- z*sigma over the d of `draws` clean launches (all rows)."""
    ds = [run(i).d.double().clone() for i in range(draws)]
    d = torch.cat(ds)
    mu, sd = float(d.mean()), float(d.std())
    z = z_of(conf)
    return mu, mu - z * sd, mu + z * sd


# ---------------------------------------------------------------- cfg1
def run_cfg1(out):
    M = N = Kd = 1024
    g = torch.Generator(device=DEV).manual_seed(0)
    w = torch.randn(N, Kd, device=DEV, generator=g) / math.sqrt(Kd)
    b = 0.02 * torch.randn(N, device=DEV, generator=g)
    ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
    aux = K.checksum_aux(ws, torch.float32)
    bsv = float(bs.item())
    xs = [torch.randn(M, Kd, device=DEV, generator=g) for _ in range(64)]
    res = K.CheckResult.empty(M, False, DEV)

    def clean(i):
        K.protected_gemm(xs[i], w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e300, hi=1e300, result=res)
        return res
    mu, lo, hi = calibrate(clean, 64, 0.9999)
    x = torch.randn(M, Kd, device=DEV, generator=g)
    rng = np.random.default_rng(0)
    n_trials = 1000
    rows = rng.integers(0, M, n_trials)
    cols = rng.integers(0, N, n_trials)
    bits = rng.integers(0, 31, n_trials)  # mantissa 0-22 + exponent 23-30 (sign excluded: default modes)
    injs = [K.injections_to_device([K.Injection(row=int(r), col=int(c), bit=int(bt))], DEV)
            for r, c, bt in zip(rows, cols, bits)]
    results = [K.CheckResult.empty(M, False, DEV) for _ in range(n_trials)]
    y = torch.empty(M, N, device=DEV)
    y_clean, _ = K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, mu=mu, lo=lo, hi=hi)
    torch.cuda.synchronize()

    def trial(i):
        K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, mu=mu, lo=lo, hi=hi, injections=injs[i],
                         out=y, result=results[i])
    for i in range(5):
        trial(i)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n_trials):
        trial(i)
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e)
    # detection: the injected row is flagged; the flip's |delta| against epsilon
    yc = y_clean.cpu().numpy()
    detected = flagged_other = 0
    detectable = detectable_hit = 0
    half = (hi - lo) / 2
    for i in range(n_trials):
        f = results[i].flags.cpu().numpy()
        r, c, bt = int(rows[i]), int(cols[i]), int(bits[i])
        hit = bool(f[r])
        detected += hit
        flagged_other += int(f.sum()) - int(hit)
        v = np.array([yc[r, c]], dtype=np.float32).view(np.uint32)
        fl = (v ^ np.uint32(1 << bt)).view(np.float32)[0]
        delta = abs(float(fl) - float(yc[r, c])) if np.isfinite(fl) else float("inf")
        if delta > 2 * half:
            detectable += 1
            detectable_hit += hit
    # campaign engine (kernels.packed_output_campaign): trials in distinct rows are independent
    # checks, packed into shared launches; verdicts must equal the per-trial ones
    faults = [K.Injection(row=int(r), col=int(c), bit=int(bt)) for r, c, bt in zip(rows, cols, bits)]
    det, n_launch = K.packed_output_campaign(x, w, b, faults, w_sum=ws, w_aux=aux, bias_sum=bsv, mu=mu, lo=lo, hi=hi)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        det, n_launch = K.packed_output_campaign(x, w, b, faults, w_sum=ws, w_aux=aux, bias_sum=bsv, mu=mu, lo=lo,
                                                 hi=hi)
    torch.cuda.synchronize()
    ms_b = (time.perf_counter() - t0) * 1e3 / 10
    det = det.cpu().numpy()
    same = all(bool(det[i]) == bool(results[i].flags.cpu().numpy()[rows[i]]) for i in range(n_trials))
    groups = [None] * n_launch
    emit({"config": "cfg1", "scope": "fp32 operands on tf32 tensor cores, fp64 checksum; one flip per launch",
          "batched_engine": {"launches": n_launch, "ms_for_all_trials_host_wall": ms_b,
                             "trials_per_s": n_trials / (ms_b * 1e-3), "verdicts_equal_per_trial": same},
          "shape": [M, N, Kd], "trials": n_trials, "ms_total": ms, "trials_per_s": n_trials / (ms * 1e-3),
          "us_per_trial": 1e3 * ms / n_trials, "epsilon": {"mu": mu, "half_width": half, "conf": 0.9999,
                                                          "clean_draws": 64},
          "detected": detected, "detection_rate": detected / n_trials,
          "flips_with_delta_over_2eps": detectable, "coverage_of_those": detectable_hit / max(detectable, 1),
          "false_flags_other_rows": flagged_other,
          "cpu_reference_ms_per_trial_BASELINE_md": 28.9}, out)


# ---------------------------------------------------------------- cfg2
def run_cfg2(out):
    hbm = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6548.5) if __import__("os").path.exists(
        "MEASURED_PEAKS.json") else 6548.5
    peak = PEAKS.get("int8") or 4500.0
    for Bi in (1, 8, 64, 256):
        for (Kd, N) in ((768, 768), (768, 2304), (768, 3072), (3072, 768)):
            M = 197 * Bi
            g = torch.Generator(device=DEV).manual_seed(Bi * 7 + N + Kd)
            x = torch.randint(-128, 128, (M, Kd), dtype=torch.int8, device=DEV, generator=g)
            w = torch.randint(-128, 128, (N, Kd), dtype=torch.int8, device=DEV, generator=g)
            b = torch.randint(-64, 65, (N,), dtype=torch.int32, device=DEV, generator=g)
            ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
            aux = K.checksum_aux(ws, torch.int8)
            bsv = int(bs.item())
            y = torch.empty(M, N, dtype=torch.int32, device=DEV)
            res = K.CheckResult.empty(M, True, DEV)
            fl = 2 * M * N * Kd
            reps = int(min(200, max(8, 2e-3 / (fl / 2e15 + 4e-6))))
            tu, tp = interleaved([lambda: K.protected_gemm(x, w, b, protect=False, out=y),
                                  lambda: K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, out=y,
                                                           result=res)], reps)
            torch.cuda.synchronize()
            ok = int(res.nflag.item()) == 0
            byts = M * Kd + N * Kd + 4 * M * N + 8 * Kd + 9 * M
            ai = fl / byts
            roof = min(peak, ai * hbm / 1e3)
            emit({"config": "cfg2", "M": M, "N": N, "K": Kd, "batch_images": Bi, "us_unprot": tu, "us_prot": tp,
                  "tops_prot": fl / (tp * 1e-6) / 1e12, "overhead_pct": 100 * (tp / tu - 1),
                  "arith_intensity": ai, "roofline_tops": roof, "frac_of_roofline": fl / (tp * 1e-6) / 1e12 / roof,
                  "clean_flags_zero": ok, "int8_peak_source": "measured (peaks line)" if "int8" in PEAKS else
                  "datasheet 4500 TOPS"}, out)


# ---------------------------------------------------------------- cfg4
def run_cfg4(out, dtype_name):
    dt = {"fp16": torch.float16, "tf32": torch.float32}[dtype_name]
    D, T, Bimg = 1024, 197, 256
    M = T * Bimg
    shapes = {"qkv": (3 * D, D), "proj": (D, D), "fc1": (4 * D, D), "fc2": (D, 4 * D)}
    per_layer = {}
    tot_trials = tot_us = 0.0
    for name, (N, Kd) in shapes.items():
        g = torch.Generator(device=DEV).manual_seed(N * 31 + Kd)
        w = (torch.randn(N, Kd, device=DEV, generator=g) / math.sqrt(Kd)).to(dt)
        b = 0.02 * torch.randn(N, device=DEV, generator=g)
        ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
        aux = K.checksum_aux(ws, dt)
        bsv = float(bs.item())
        xs = [torch.randn(M, Kd, device=DEV, generator=g).to(dt) for _ in range(3)]
        res = K.CheckResult.empty(M, False, DEV)

        def clean(i):
            K.protected_gemm(xs[i], w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, lo=-1e300, hi=1e300, result=res)
            return res
        mu, lo, hi = calibrate(clean, 2, 0.9999)
        x = xs[2]
        y_clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, mu=mu, lo=lo, hi=hi)
        torch.cuda.synchronize()
        clean_flags = int(r0.nflag.item())
        # one flip per image per launch: image j's row j*T + r_j; 8 launches of B trials each
        rng = np.random.default_rng(N + Kd)
        launches = 8
        inj_sets, meta = [], []
        top = 16 if dt == torch.float16 else 31
        for _ in range(launches):
            rr = rng.integers(0, T, Bimg) + np.arange(Bimg) * T
            cc = rng.integers(0, N, Bimg)
            bb = rng.integers(0, top - 1, Bimg)  # exclude the sign bit
            inj_sets.append(K.injections_to_device([K.Injection(row=int(r), col=int(c), bit=int(t))
                                                    for r, c, t in zip(rr, cc, bb)], DEV))
            meta.append((rr, cc, bb))
        y = torch.empty_like(y_clean)
        ress = [K.CheckResult.empty(M, False, DEV) for _ in range(launches)]

        def launch(i):
            K.protected_gemm(x, w, b, w_sum=ws, w_aux=aux, bias_sum=bsv, mu=mu, lo=lo, hi=hi,
                             injections=inj_sets[i], out=y, result=ress[i])
        for i in range(launches):
            launch(i)
        torch.cuda.synchronize()
        hits = detectable = detectable_hits = 0
        half = (hi - lo) / 2
        yc = y_clean.float().cpu().numpy()
        for i in range(launches):
            f = ress[i].flags.cpu().numpy()
            rr, cc, bb = meta[i]
            for r, c, t in zip(rr, cc, bb):
                hit = bool(f[r])
                hits += hit
                if dt == torch.float16:
                    v = np.array([yc[r, c]], dtype=np.float16).view(np.uint16)
                    flv = float((v ^ np.uint16(1 << int(t))).view(np.float16)[0])
                else:
                    v = np.array([yc[r, c]], dtype=np.float32).view(np.uint32)
                    flv = float((v ^ np.uint32(1 << int(t))).view(np.float32)[0])
                delta = abs(flv - float(yc[r, c])) if math.isfinite(flv) else float("inf")
                if delta > 2 * half:
                    detectable += 1
                    detectable_hits += hit
        reps = 8
        (tl,) = interleaved([lambda: launch(0)], reps, rounds=4)
        trials = Bimg
        per_layer[name] = {"N": N, "K": Kd, "us_per_launch": tl, "trials_per_launch": trials,
                           "trials_per_s": trials / (tl * 1e-6), "detection_rate": hits / (launches * Bimg),
                           "flips_delta_over_2eps": detectable,
                           "coverage_of_those": detectable_hits / max(detectable, 1), "clean_flags": clean_flags,
                           "eps_half_width": half}
        tot_trials += trials
        tot_us += tl
    emit({"config": "cfg4", "dtype": dtype_name, "scope": "GEMM-level campaign engine: ViT-L/16 block GEMM "
          "shapes, 256 images per launch, one output flip per image, detection at the injected layer "
          "(no suffix recompute)", "images_per_launch": Bimg, "layers": per_layer,
          "trials_per_s_mean_over_layer_types": tot_trials / (tot_us * 1e-6)}, out)


# ---------------------------------------------------------------- cfg5
def run_cfg5(out):
    Bimg = 32
    stages = [(3136, 128, 2), (784, 256, 2), (196, 512, 18), (49, 1024, 2)]
    layers = []
    for si, (tok, C, depth) in enumerate(stages):
        M = tok * Bimg
        for _ in range(depth):
            layers += [("qkv", M, 3 * C, C, torch.bfloat16), ("proj", M, C, C, torch.bfloat16),
                       ("fc1", M, 4 * C, C, torch.int8), ("fc2", M, C, 4 * C, torch.int8)]
        if si < 3:
            layers.append(("merge", tok // 4 * Bimg, 2 * C, 4 * C, torch.bfloat16))
    built = []
    for li, (name, M, N, Kd, dt) in enumerate(layers):
        g = torch.Generator(device=DEV).manual_seed(li)
        integer = dt == torch.int8
        if integer:
            x = torch.randint(-31, 32, (M, Kd), dtype=torch.int8, device=DEV, generator=g)
            w = torch.randint(-15, 16, (N, Kd), dtype=torch.int8, device=DEV, generator=g)
            b = torch.randint(-64, 65, (N,), dtype=torch.int32, device=DEV, generator=g)
            ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
            bsv = int(bs.item())
        else:
            x = torch.randn(M, Kd, device=DEV, generator=g).to(dt)
            w = (torch.randn(N, Kd, device=DEV, generator=g) / math.sqrt(Kd)).to(dt)
            b = None if name == "merge" else 0.02 * torch.randn(N, device=DEV, generator=g)
            ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
            bsv = float(bs.item()) if b is not None else 0.0
        aux = K.checksum_aux(ws, dt)
        y = torch.empty(M, N, dtype=K.default_out_dtype(dt), device=DEV)
        res = K.CheckResult.empty(M, integer, DEV)
        built.append(dict(name=name, x=x, w=w, b=b, ws=ws, aux=aux, bsv=bsv, y=y, res=res, integer=integer,
                          lo=0.0 if integer else -1e300, hi=0.0 if integer else 1e300, key=f"s{li}"))
    # float epsilon: one clean calibration pass per layer
    for ly in built:
        if not ly["integer"]:
            K.protected_gemm(ly["x"], ly["w"], ly["b"], w_sum=ly["ws"], w_aux=ly["aux"], bias_sum=ly["bsv"],
                             lo=-1e300, hi=1e300, out=ly["y"], result=ly["res"], ws_key=ly["key"])
            d = ly["res"].d.double()
            mu, sd = float(d.mean()), float(d.std())
            z = z_of(1 - 1e-9)
            ly["mu"], ly["lo"], ly["hi"] = mu, mu - z * sd, mu + z * sd
    target = next(i for i, ly in enumerate(built) if ly["name"] == "fc1" and ly["y"].shape[0] == 784 * Bimg)
    tl = built[target]
    inj = K.injections_to_device([K.Injection(row=12345, col=77, bit=30)], DEV)

    def launch(ly, injections=None):
        K.protected_gemm(ly["x"], ly["w"], ly["b"], w_sum=ly["ws"], w_aux=ly["aux"], bias_sum=ly["bsv"],
                         mu=ly.get("mu", 0.0), lo=ly["lo"], hi=ly["hi"], injections=injections, out=ly["y"],
                         result=ly["res"], ws_key=ly["key"])

    def step_clean():
        for ly in built:
            launch(ly)

    def step_inj_replay():
        for i, ly in enumerate(built):
            if i == target:
                launch(ly, inj)
                K.replay_tiles(ly["x"], ly["w"], ly["b"], ly["y"], ly["res"].flags, ly["res"], w_sum=ly["ws"],
                               w_aux=ly["aux"], bias_sum=ly["bsv"], lo=ly["lo"], hi=ly["hi"], ws_key=ly["key"])
            else:
                launch(ly)
    step_inj_replay()
    torch.cuda.synchronize()
    replayed_clean = int(tl["res"].nflag.item()) == 0
    # median of per-round ratios (each round times both graphs back to back, so the ratio is
    # insensitive to the slow clock drift of the power cap)
    rc, ri = interleaved([step_clean, step_inj_replay], 4, rounds=24, per_round=True)
    t_clean, t_inj = statistics.median(rc), statistics.median(ri)
    ratio = statistics.median(b / a for a, b in zip(rc, ri))
    # the replay's own cost: the target layer alone, clean vs injected + replayed
    def tgt_clean():
        launch(tl)

    def tgt_inj_replay():
        launch(tl, inj)
        K.replay_tiles(tl["x"], tl["w"], tl["b"], tl["y"], tl["res"].flags, tl["res"], w_sum=tl["ws"],
                       w_aux=tl["aux"], bias_sum=tl["bsv"], lo=tl["lo"], hi=tl["hi"], ws_key=tl["key"])
    rt_c, rt_i = interleaved([tgt_clean, tgt_inj_replay], 32, rounds=16, per_round=True)
    replay_us = statistics.median(b - a for a, b in zip(rt_c, rt_i))
    fl = sum(2 * ly["x"].shape[0] * ly["w"].shape[0] * ly["w"].shape[1] for ly in built)
    emit({"config": "cfg5", "scope": "Swin-B GEMM set (4 stages, depths 2/2/18/2, qkv/proj/merge bf16, "
          "fc1/fc2 int8), batch 32, one injected output error in a stage-2 fc1 detected and replayed "
          "(replay_tiles recomputes the flagged 256-row band only)", "gemms": len(built),
          "gflop_per_step": fl / 1e9, "ms_clean": t_clean / 1e3, "ms_inj_replay": t_inj / 1e3,
          "per_error_overhead_pct": 100 * (ratio - 1), "replay_us": replay_us,
          "replay_share_of_step_pct": 100 * replay_us / t_clean, "flags_clear_after_replay": replayed_clean,
          "target_pct": 2.0}, out)


# ---------------------------------------------------------------- calibration kernels (§8(f) 1)
def run_calib(out):
    from paper_2310_03841_b200 import calib
    hbm = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6548.5) if __import__("os").path.exists(
        "MEASURED_PEAKS.json") else 6548.5
    d = torch.randn(50432, device=DEV, dtype=torch.float64)
    st = calib.RunningStats(DEV)
    (t_stats,) = interleaved([lambda: st.update(d)], 50, rounds=4)
    y = torch.randn(50432, 3072, device=DEV).to(torch.bfloat16)
    rr = calib.RunningRange(DEV)
    (t_mm,) = interleaved([lambda: rr.update(y)], 20, rounds=4)
    gbs = y.numel() * 2 / (t_mm * 1e-6) / 1e9
    emit({"config": "calib", "scope": "device calibration kernels: running (n, mean, M2) of one ViT-B layer's d "
          "(50432 rows) and running min / max of a fc1 output (50432 x 3072 bf16)",
          "us_running_stats": t_stats, "us_minmax": t_mm, "minmax_gbs": gbs, "minmax_frac_of_hbm": gbs / hbm}, out)


# ---------------------------------------------------------------- int8 toy on the device (§8(f) 2)
def run_toy_int8(out):
    from paper_2310_03841_b200 import model as Mo
    from paper_2310_03841_b200 import toy_device as TD
    from paper_2310_03841_b200.numerics import Matrix2D
    model = Mo.build_toy_model(12, 768, 197, 1000, 0, "int8")
    rng = np.random.default_rng(1)
    inputs = [Matrix2D(rng.integers(-31, 32, (197, 768)), "int8") for _ in range(64)]
    TD.forward_batch(model, inputs[:4], protect=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outb = TD.forward_batch(model, inputs, protect=True)
    t_batch = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = Mo.forward(model, inputs[0], 0)
    t_host = time.perf_counter() - t0
    same = outb.logits[0].tolist() == ref.logits.tolist()
    emit({"config": "toy_int8_device", "scope": "integer toy with ViT-B dims (12 blocks, dim 768, 197 tokens, "
          "1000 classes; token mixing stands in for attention): batched device forward, every GEMM protected "
          "(int64-exact), host inputs in / logits out", "batch": len(inputs),
          "images_per_s_device_batch": len(inputs) / t_batch, "s_per_image_host_glue": t_host,
          "logits_identical_to_host_path": same, "flags_clean": all(not f.any() for f in outb.flagged.values()),
          "cpu_reference_s_per_image_BASELINE_md": 12.0}, out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="peaks,cfg1,cfg2,cfg4,cfg5,calib,toy")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    sel = a.only.split(",")
    if "peaks" in sel:
        run_peaks(a.out)
    if "cfg1" in sel:
        run_cfg1(a.out)
    if "cfg2" in sel:
        run_cfg2(a.out)
    if "cfg4" in sel:
        run_cfg4(a.out, "fp16")
        run_cfg4(a.out, "tf32")
    if "cfg5" in sel:
        run_cfg5(a.out)
    if "calib" in sel:
        run_calib(a.out)
    if "toy" in sel:
        run_toy_int8(a.out)


if __name__ == "__main__":
    main()
