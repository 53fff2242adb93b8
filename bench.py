"""Benchmark of the checksum-protected GEMM path (BASELINE.json metric).

Workload (configs[2] of BASELINE.json, the largest single-GPU config the
metric is quoted on): random-init ViT-B/16 inference at batch 256 in bf16
with all 50 Linear layers protected (`vit.ProtectedViT`: patch embed, 12 x
{qkv, proj, fc1 (+ fused GELU), fc2}, head), each with its own epsilon
calibrated on clean batches; attention (torch SDPA) and layer norms
unprotected.  Synthetic images (there is no network for
datasets or checkpoints).

One step = one full forward of the 256-image batch, captured once as a CUDA
graph and replayed.  Reported on one JSON line:

* value: protected ViT-B/16 images/s (whole job: all ranks), inputs resident;
* e2e: the same through the model API with the batch copied from pinned host
  memory every step and logits + per-layer flag counts read back;
* overhead_pct: against the same forward with every GEMM unprotected (the
  same kernel family), plus the GEMM-only view: the 50 protected launches on
  distinct per-layer buffers (protected_gemm_tflops, gemm_overhead_pct);
* roofline of the dominant kernel (K1, the protected GEMM) against the
  measured bf16 peak, and the whole-model fraction;
* coverage: a batched output bit-flip campaign (`campaign.ViTCampaign`: one
  trial per image, every protected layer) with the coverage of
  output-mismatching flips, its Wilson 95% interval and the clean false flags
  per image, at the bench's confidence and at c = 0.9999;
* cpu_baseline: the reference's CPU path (oracle port of numerics.gemm +
  guard._verify_arrays) on one image's protected GEMMs per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun): every rank runs its own batch-256 replica (weak
scaling, no collective on the hot path); campaign units are shared over the
ranks and their int64 counters all-reduced over NCCL (K5).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BATCH = 256
TOKENS = 197
D, MLP, BLOCKS, CLASSES = 768, 3072, 12, 1000
CONFIDENCE = 1.0 - 1e-9  # per-row checks: ~50k rows x 50 layers per step => keep false flags << 1 per step

# DRAM bytes (read + write) per protected launch, from `ncu --set full` captures of K1
# (profiles/r02/full_{proj,fc2}.ncu-rep and SUMMARY.md; profiles/ does not travel to the box)
NCU_DRAM_MB = {"qkv": 284.3, "proj": 115.6, "fc1": 369.0, "fc2": 382.4}  # profiles/r02/ncu_summaries (final)


def step_traffic_bytes() -> float:
    """DRAM traffic of the 50 protected GEMMs (ncu); patch embed ~ proj, head ~ 0."""
    per_block = sum(NCU_DRAM_MB[k] for k in ("qkv", "proj", "fc1", "fc2"))
    return 1e6 * (NCU_DRAM_MB["proj"] + BLOCKS * per_block)


def step_algorithmic_bytes(gemms) -> float:
    """Minimum bytes of the 50 GEMMs: A, B, C in bf16 plus d (8 B) and flags (1 B) per row."""
    return float(sum(2 * (M * K + N * K + M * N) + 9 * M for _, M, N, K in gemms))


def vit_b16_gemms(batch: int = BATCH):
    """(name, M, N, K) of the protected GEMMs of one ViT-B/16 forward."""
    m = batch * TOKENS
    g = [("patch_embed", batch * (TOKENS - 1), D, 3 * 16 * 16)]
    for b in range(BLOCKS):
        g += [(f"blk{b}.qkv", m, 3 * D, D), (f"blk{b}.proj", m, D, D), (f"blk{b}.fc1", m, MLP, D),
              (f"blk{b}.fc2", m, D, MLP)]
    g.append(("head", batch, CLASSES, D))
    return g


def gemm_flops(gemms) -> float:
    return float(sum(2 * M * N * K for _, M, N, K in gemms))


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------- reference (CPU) arm
def _ref_layer(args):
    """The reference algorithm (oracle port) on `rows` rows of one layer:
    numerics.gemm in binary16-emulated with binary32 accumulation (the
    reference's nearest precision to bf16) + guard._verify_arrays."""
    from oracle import gemmguard_oracle as O

    name, rows, N, K, seed = args
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, K)).astype(np.float16).astype(np.float64)
    wt = (rng.standard_normal((K, N)) / math.sqrt(K)).astype(np.float16).astype(np.float64)
    bias = (0.02 * rng.standard_normal(N)).astype(np.float16).astype(np.float64)
    w_sum, bsum = O.offline_checksum(wt, bias, "binary64")  # offline: outside the timed region
    t0 = time.perf_counter()
    y = O.gemm(x, wt, bias, "binary16-emulated", "binary32")
    O.verify(x, y, w_sum, bsum, "binary64", {"mu": 0.0, "threshold_low": -1e9, "threshold_high": 1e9})
    return time.perf_counter() - t0, 2.0 * rows * N * K


def reference_step(rows: int, workers: int, gemms) -> tuple[float, float]:
    """One bounded sample of the workload on the CPU: `rows` rows (one image) of
    every protected layer, layers spread over `workers` processes.  Returns (seconds, flops)."""
    jobs = [(name, min(rows, M), N, K, i) for i, (name, M, N, K) in enumerate(gemms)]
    t0 = time.perf_counter()
    if workers > 1:
        with ProcessPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(_ref_layer, jobs))
    else:
        res = [_ref_layer(j) for j in jobs]
    wall = time.perf_counter() - t0
    return wall, sum(f for _, f in res)


REF_SAMPLE = ("one image per step: 197 rows (1 for the head) of each of the 50 protected ViT-B/16 GEMMs, "
              "binary16-emulated x binary32 numerics.gemm + guard._verify_arrays (oracle port of the reference, "
              "which has no attention), layers over {w} processes")


def run_reference(args) -> dict:
    gemms = vit_b16_gemms(1)
    workers = os.cpu_count() or 1
    for _ in range(max(0, min(args.warmup, 1))):
        reference_step(TOKENS, workers, gemms)
    times = []
    for _ in range(args.steps):
        t, _ = reference_step(TOKENS, workers, gemms)
        times.append(t)
    total = sum(times)
    value = len(times) / total  # one image per step
    return {"metric": "vit_b16_protected_img_per_s", "value": value, "unit": "img/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16xf32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "vit_b16_b256_protected_inference", "images_per_step_sample": 1},
            "cpu_baseline": {"value": value, "unit": "img/s", "cores": workers, "kind": "port",
                             "sample": REF_SAMPLE.format(w=workers)},
            "e2e": {"value": value, "unit": "img/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_baseline(args) -> dict:
    workers = os.cpu_count() or 1
    t, _ = reference_step(TOKENS, workers, vit_b16_gemms(1))
    return {"value": 1.0 / t, "unit": "img/s", "cores": workers, "kind": "port",
            "sample": REF_SAMPLE.format(w=workers) + f", {t:.1f} s"}


# ------------------------------------------------------------------- ours
def _timed(fn, steps, warmup, world, dev, stream):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        fn()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
        torch.distributed.barrier()
    return ms


_CAPTURE_STREAM = None


def _interleaved(fa, fb, rounds, steps, warmup, world, dev, stream):
    """Median per-step times of two step functions timed in alternating rounds (A B, B A, ...)
    so that clock / power drift under the power cap hits both equally."""
    ta, tb = [], []
    for r in range(rounds):
        order = (fa, fb) if r % 2 == 0 else (fb, fa)
        for f in order:
            ms = _timed(f, steps, warmup if r == 0 else 1, world, dev, stream)
            (ta if f is fa else tb).append(ms)
    return statistics.median(ta), statistics.median(tb)


def _capture(fn):
    """CUDA graph of fn, warmed on the capture stream itself so that per-stream
    workspaces (kernels.workspace) are allocated and zeroed outside the graph."""
    import torch

    global _CAPTURE_STREAM
    if _CAPTURE_STREAM is None:
        _CAPTURE_STREAM = torch.cuda.Stream()
    s = _CAPTURE_STREAM
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


def gemm_only(args, dev, world, stream):
    """The 50 protected launches of one step on distinct per-layer buffers (>> L2): K1's
    own throughput and overhead against the unprotected instance of the same kernel."""
    import torch

    from paper_2310_03841_b200 import _lib as L
    from paper_2310_03841_b200 import calib
    from paper_2310_03841_b200 import kernels as K

    gemms = vit_b16_gemms()
    g = torch.Generator(device=dev).manual_seed(99)
    layers = []
    for name, M, N, Kd in gemms:
        w = (torch.randn(N, Kd, device=dev, generator=g) / math.sqrt(Kd)).to(torch.bfloat16)
        b = (0.02 * torch.randn(N, device=dev, generator=g)).float()
        x = torch.randn(M, Kd, device=dev, generator=g).to(torch.bfloat16)
        w_sum, bsum = K.offline_checksum(w, b, L.GG_P_F64)
        layers.append(dict(name=name, M=M, N=N, K=Kd, w=w, b=b, x=x, w_sum=w_sum, bsum=float(bsum.item()),
                           aux=K.checksum_aux(w_sum, torch.bfloat16), y=torch.empty(M, N, device=dev,
                                                                                    dtype=torch.bfloat16),
                           res=K.CheckResult.empty(M, False, dev), mu=0.0, lo=-1e300, hi=1e300))

    def launch(ly, protect=True):
        if protect:
            K.protected_gemm(ly["x"], ly["w"], ly["b"], w_sum=ly["w_sum"], w_aux=ly["aux"], bias_sum=ly["bsum"],
                             mu=ly["mu"], lo=ly["lo"], hi=ly["hi"], out=ly["y"], result=ly["res"],
                             ws_key=("gemm", ly["name"]))
        else:
            K.protected_gemm(ly["x"], ly["w"], ly["b"], protect=False, out=ly["y"])

    stats = {ly["name"]: calib.RunningStats(dev) for ly in layers}
    for ly in layers:
        launch(ly)
        stats[ly["name"]].update(ly["res"].d)
    for ly in layers:
        ly["mu"], ly["lo"], ly["hi"] = stats[ly["name"]].epsilon(CONFIDENCE)
    gp = _capture(lambda: [launch(ly, True) for ly in layers])
    gu = _capture(lambda: [launch(ly, False) for ly in layers])
    ms_p, ms_u = _interleaved(gp.replay, gu.replay, 6, max(3, args.steps // 2), args.warmup, world, dev, stream)
    # the library baseline: the same 50 GEMMs (+ bias) through cuBLAS, unprotected
    for ly in layers:
        ly["bb"] = ly["b"].to(torch.bfloat16)
    gc = _capture(lambda: [torch.addmm(ly["bb"], ly["x"], ly["w"].t(), out=ly["y"]) for ly in layers])
    ms_c = _timed(gc.replay, max(3, args.steps // 2), args.warmup, world, dev, stream)
    flops = gemm_flops(gemms)
    out = {"protected_gemm_tflops": flops / (ms_p * 1e-3) / 1e12, "unprotected_gemm_tflops": flops / (ms_u * 1e-3) / 1e12,
           "gemm_overhead_pct": 100.0 * (ms_p / ms_u - 1.0), "gemm_ms_per_step": ms_p,
           "cublas_unprotected_tflops": flops / (ms_c * 1e-3) / 1e12,
           "protected_vs_cublas_pct": 100.0 * (ms_p / ms_c - 1.0),
           "l2": f"distinct per-layer buffers, {sum(ly['x'].numel() + ly['y'].numel() for ly in layers) * 2 / 1e9:.1f} "
                 f"GB of activations per step (>> 126 MB L2)"}
    del layers, gp, gu, gc
    torch.cuda.empty_cache()
    return out


def run_ours(args, rank: int, world: int, local_rank: int) -> dict:
    import torch

    from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    cfg = VIT_B16
    model = ProtectedViT(cfg, dtype=torch.bfloat16, device=dev, seed=1234)  # same weights on every rank
    gen = torch.Generator(device=dev).manual_seed(4321 + rank)

    def images(n=BATCH):
        return torch.randn(n, 3, cfg.image, cfg.image, device=dev, generator=gen).to(torch.bfloat16)

    with torch.no_grad():
        # ---- per-layer epsilon from two clean calibration batches (device running moments)
        model.calibrate([images(), images()], CONFIDENCE)
        held = images()  # held-out batch, resident in HBM
        fwd_p = lambda: model(held, protect=True)  # noqa: E731
        fwd_u = lambda: model(held, protect=False)  # noqa: E731
        g_p = _capture(fwd_p)
        g_u = _capture(fwd_u)
        with ClockSampler(local_rank) as clk:
            ms_p = _timed(g_p.replay, args.steps, args.warmup, world, dev, stream)
        # overhead: protected vs unprotected forward in alternating rounds (median per step)
        ab_p, ab_u = _interleaved(g_p.replay, g_u.replay, 6, max(3, args.steps // 2), args.warmup, world, dev, stream)
        g_p.replay()
        flagged = model.flagged_rows(BATCH)  # held-out false flags of the timed batch (K5 over NCCL)
        if world > 1:
            torch.distributed.all_reduce(flagged)
        false_flags = int(flagged.sum().item())
        e2e = measure_e2e(model, g_p, held, dev, args, world)
        del g_p, g_u
        torch.cuda.empty_cache()
        gem = gemm_only(args, dev, world, stream)
        cov = {}
        if not args.no_campaign:
            cov = coverage_study(model, held, images, args, rank, world, dev)

    gemm_f, attn_f = cfg.flops_per_image()
    img_s = BATCH * world / (ms_p * 1e-3)
    img_s_u = BATCH * world / (ab_u * 1e-3)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("bf16_tflops_sustained") or 1400.0
    k1 = gem["protected_gemm_tflops"] / world
    model_tf = (gemm_f + attn_f) * img_s / world / 1e12
    layer_launches = len(model.linears)
    return {
        "metric": "vit_b16_protected_img_per_s", "value": img_s, "unit": "img/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_p, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic images, random-init ViT-B/16 weights",
        "config": {"workload": "vit_b16_b256_protected_inference", "model": "vit_b16", "global_batch": BATCH * world,
                   "seq_len": TOKENS, "protected_gemms": layer_launches, "parallelism": f"replicas{world}",
                   "epsilon": f"per-layer mu +/- z*sigma, c={CONFIDENCE}",
                   "l2": "one step moves ~15 GB of activations (>> 126 MB L2)"},
        "overhead_pct": 100.0 * (ab_p / ab_u - 1.0), "unprotected_img_per_s": img_s_u,
        "overhead_method": "protected vs unprotected forward graphs, 6 alternating rounds, median ms per step",
        "protected_gemm_tflops": gem["protected_gemm_tflops"], "gemm_overhead_pct": gem["gemm_overhead_pct"],
        "gemm_only": gem,
        "held_out_false_flags": false_flags,
        "roofline": {"bound": "tensor", "achieved": k1, "peak": peak, "unit": "TFLOP/s", "frac": k1 / peak,
                     "traffic": step_traffic_bytes(),
                     "traffic_unit": "DRAM bytes of the 50 protected launches of one step, ncu --set full",
                     "algorithmic_bytes": step_algorithmic_bytes(vit_b16_gemms()),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, back to back 4 s)",
                     "kernel": "gg_protected_gemm_pair_kernel<bf16> (K1): 2 * sum(M N K) of the 50 GEMMs / their "
                               "graph time on distinct buffers",
                     "model_tflops": model_tf, "model_frac": model_tf / peak,
                     "model_flops_per_image": gemm_f + attn_f},
        "coverage": cov,
        "e2e": e2e,
        "gpu_launches": (layer_launches + 2 * cfg.depth + 2) * args.steps,
        "gpu_launches_note": "per step: 50 K1 (protected GEMM) + gg_patchify + gg_embed_layernorm + 24 "
                             "gg_add_layernorm; torch SDPA not counted",
        "clocks": clk.summary(),
    }


def coverage_study(model, held, images, args, rank, world, dev) -> dict:
    """Batched output bit-flip campaigns (one trial per image, every protected layer):
    the bf16 model at the bench's c and at c = 0.9999, and the same architecture in
    fp16 (the paper's DeiT precision) at the bench's c."""
    import torch

    from paper_2310_03841_b200.campaign import ViTCampaign
    from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT

    from paper_2310_03841_b200.campaign import select_golden_images

    out = {}
    # golden set: images the bf16 model classifies like its fp32 teacher (profiler.select_golden's rule)
    teacher = ProtectedViT(VIT_B16, dtype=torch.float32, device=dev, seed=1234, f32_mode="3xtf32")
    golden, gstats = select_golden_images(model, teacher, images, BATCH)
    out["golden"] = gstats
    del teacher
    torch.cuda.empty_cache()

    from paper_2310_03841_b200.campaign_vit import calibrate_distributed

    def one(m, imgs, c, cal, tag, modes=("fp_exponent_bit", "fp_mantissa_bit")):
        calibrate_distributed(m, cal, c)  # every rank's batches, moments merged in rank order
        t0 = time.perf_counter()
        camp = ViTCampaign(m, imgs, seed=2310, modes=modes)
        tally = camp.run(args.campaign_blocks, rank=rank, world_size=world)
        torch.cuda.synchronize()
        s = tally.summary()
        s["trials_per_s"] = s["injections"] / (time.perf_counter() - t0)
        s["confidence"] = c
        s["modes"] = list(modes)
        s["by_role"] = tally.by_group(m.role_groups())
        out[tag] = s
        del camp

    cal = [images(), images()]
    one(model, golden, CONFIDENCE, cal, f"bf16 c={CONFIDENCE} bit flips")
    one(model, golden, CONFIDENCE, cal, f"bf16 c={CONFIDENCE} random values", ("random_value",))
    one(model, golden, 0.9999, cal, "bf16 c=0.9999 random values", ("random_value",))
    one(model, held, CONFIDENCE, cal, f"bf16 c={CONFIDENCE} bit flips, unfiltered images (near-ties kept)")
    model.calibrate(cal, CONFIDENCE)
    torch.cuda.empty_cache()
    m16 = ProtectedViT(VIT_B16, dtype=torch.float16, device=dev, seed=1234)
    one(m16, golden.to(torch.float16), CONFIDENCE, [c.to(torch.float16) for c in cal],
        f"fp16 c={CONFIDENCE} random values", ("random_value",))
    del m16
    torch.cuda.empty_cache()
    return out


def measure_e2e(model, graph, held, dev, args, world):
    """img/s through the model with the batch copied from pinned host memory every step
    (double-buffered on a side stream), logits + per-layer flag counts read back."""
    import torch

    host_x = torch.empty(held.shape, dtype=held.dtype, pin_memory=True)
    host_x.copy_(held.cpu())
    host_logits = torch.empty((BATCH, CLASSES), dtype=torch.bfloat16, pin_memory=True)
    host_flags = torch.empty(len(model.linears), dtype=torch.int64, pin_memory=True)
    copy_stream = torch.cuda.Stream(dev)
    compute = torch.cuda.current_stream(dev)
    staging = [torch.empty_like(held), torch.empty_like(held)]
    copied = [torch.cuda.Event(), torch.cuda.Event()]

    def prefetch(i):
        copy_stream.wait_stream(compute)
        with torch.cuda.stream(copy_stream):
            staging[i % 2].copy_(host_x, non_blocking=True)
            copied[i % 2].record(copy_stream)

    def step(i):
        compute.wait_event(copied[i % 2])
        held.copy_(staging[i % 2])  # the graph's input buffer (device-to-device)
        prefetch(i + 1)
        graph.replay()
        host_flags.copy_(model.flagged_rows(BATCH), non_blocking=True)
        host_logits.copy_(model.buffers(BATCH).logits, non_blocking=True)

    n_total = args.warmup + args.steps
    prefetch(0)
    for i in range(args.warmup):
        step(i)
        compute.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for i in range(args.warmup, n_total):
        step(i)
        compute.synchronize()  # the host consumes logits + flags every step
    compute.wait_stream(copy_stream)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    return {"value": BATCH * world / (ms * 1e-3), "unit": "img/s",
            "h2d_bytes_per_step": host_x.numel() * host_x.element_size(),
            "d2h_bytes_per_step": host_logits.numel() * host_logits.element_size() + host_flags.numel() * 8,
            "ms_per_step": ms, "host_wall_ms_per_step": 1e3 * (time.perf_counter() - t0) / args.steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-campaign", action="store_true")
    ap.add_argument("--campaign-blocks", type=int, default=1, help="trial blocks of 256 per protected layer")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    import torch

    if world > 1:
        # one rank per GPU over NCCL; GG_BENCH_BACKEND=gloo lets several ranks share one GPU to
        # exercise the N > 1 path where only one GPU is visible (tests / single-GPU boxes)
        backend = os.environ.get("GG_BENCH_BACKEND", "nccl")
        dev = torch.device("cuda", local_rank % torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines on stderr: one rank per GPU
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:
            torch.distributed.init_process_group(backend)
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
