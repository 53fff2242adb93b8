"""Benchmark of the checksum-protected GEMM path (BASELINE.json metric).

Workload (configs[2] of BASELINE.json, the largest single-GPU config the
metric is quoted on): the 50 protected GEMMs of one ViT-B/16 inference at
batch 256 in bf16 — patch embed 50176x768x768, 12 x (qkv 50432x2304x768,
attn proj 50432x768x768, mlp fc1 50432x3072x768, mlp fc2 50432x768x3072), and
the 1000-class head 256x1000x768 — every one a fused protected launch (K1)
with its own per-layer epsilon threshold calibrated on clean batches.
Random-init weights and synthetic activations of those shapes (there is no
network for checkpoints or datasets).  One step = one pass over the 50
GEMMs, captured once as a CUDA graph and replayed; every layer has its own
input and output buffers (13 GB working set per step, >> the 126 MB L2).

Reported: protected-GEMM TFLOP/s (value), the overhead against the
unprotected launch of the same kernel family, the implied ViT-B/16
protected-GEMM images/s, a roofline line for K1 against the measured bf16
peak, an end-to-end number through the public API with host buffers, the
reference's CPU path (the oracle port) timed on this host, and clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun): every rank runs its own batch-256 replica (weak
scaling, no collective on the hot path); the per-layer flagged-row counters
are all-reduced over NCCL once after the timed region.
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

# DRAM bytes (read + write) per protected launch, from `ncu --set full` captures of
# this kernel (profiles/r01/ncu_full_bf16_vitb.json; profiles/ does not travel to the box)
NCU_DRAM_MB = {"qkv": 282.1, "proj": 116.5, "fc1": 371.7, "fc2": 382.4}  # protected launches, ncu --set full (profiles/r01)


def step_traffic_bytes() -> float:
    """DRAM traffic of one step (50 launches) measured by ncu; patch embed ~ proj, head ~ 0."""
    per_block = sum(NCU_DRAM_MB[k] for k in ("qkv", "proj", "fc1", "fc2"))
    return 1e6 * (NCU_DRAM_MB["proj"] + BLOCKS * per_block)


def step_algorithmic_bytes(gemms) -> float:
    """Minimum bytes of one step: A, B, C of every GEMM in bf16 plus d (8 B) and flags (1 B) per row."""
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
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

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
    """One bounded sample of the workload on the CPU: `rows` rows of every
    layer, layers spread over `workers` processes.  Returns (seconds, flops)."""
    jobs = [(name, min(rows, M), N, K, i) for i, (name, M, N, K) in enumerate(gemms)]
    t0 = time.perf_counter()
    if workers > 1:
        with ProcessPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(_ref_layer, jobs))
    else:
        res = [_ref_layer(j) for j in jobs]
    wall = time.perf_counter() - t0
    return wall, sum(f for _, f in res)


def run_reference(args) -> dict:
    gemms = vit_b16_gemms()
    workers = os.cpu_count() or 1
    rows = args.ref_rows
    for _ in range(max(0, min(args.warmup, 1))):
        reference_step(rows, workers, gemms)
    times, flops = [], 0.0
    for _ in range(args.steps):
        t, flops = reference_step(rows, workers, gemms)
        times.append(t)
    total = sum(times)
    value = flops * len(times) / total / 1e12
    sample = f"{rows} rows (one image) of each of the 50 ViT-B/16 GEMMs per step, binary16-emulated x binary32 " \
             f"numerics.gemm + guard._verify_arrays (oracle port), layers over {workers} processes"
    return {"metric": "protected_gemm_tflops", "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16xf32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "vit_b16_b256_protected_gemms", "rows_per_layer_sample": rows},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": workers, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------- ours
def run_ours(args, rank: int, world: int, local_rank: int) -> dict | None:
    import torch

    from paper_2310_03841_b200 import _lib as L
    from paper_2310_03841_b200 import kernels as K

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    gemms = vit_b16_gemms()
    flops = gemm_flops(gemms)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    layers = []
    for name, M, N, Kd in gemms:
        w = (torch.randn(N, Kd, device=dev, generator=g) / math.sqrt(Kd)).to(torch.bfloat16)
        b = (0.02 * torch.randn(N, device=dev, generator=g)).float()
        x = torch.randn(M, Kd, device=dev, generator=g).to(torch.bfloat16)
        w_sum, bsum = K.offline_checksum(w, b, L.GG_P_F64)  # K2, offline
        aux = K.checksum_aux(w_sum, torch.bfloat16)
        y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        res = K.CheckResult.empty(M, False, dev)
        layers.append(dict(name=name, M=M, N=N, K=Kd, w=w, b=b, x=x, w_sum=w_sum, bsum=float(bsum.item()),
                           aux=aux, y=y, res=res, lo=-1e300, hi=1e300, mu=0.0, ws_key=name))

    def launch(ly, protect=True):
        if protect:
            K.protected_gemm(ly["x"], ly["w"], ly["b"], w_sum=ly["w_sum"], w_aux=ly["aux"], bias_sum=ly["bsum"],
                             mu=ly["mu"], lo=ly["lo"], hi=ly["hi"], out=ly["y"], result=ly["res"],
                             ws_key=ly["ws_key"])
        else:
            K.protected_gemm(ly["x"], ly["w"], ly["b"], protect=False, out=ly["y"])

    # ---- per-layer epsilon: two clean calibration batches (fresh activations each); the
    # fused check's d is folded into device-resident running moments (calib.RunningStats)
    from paper_2310_03841_b200 import calib
    stats = {ly["name"]: calib.RunningStats(dev) for ly in layers}
    for c in range(2):
        for ly in layers:
            if c:
                ly["x"].copy_(torch.randn(ly["M"], ly["K"], device=dev, generator=g).to(torch.bfloat16))
            launch(ly)
            stats[ly["name"]].update(ly["res"].d)
    for ly in layers:
        ly["mu"], ly["lo"], ly["hi"] = stats[ly["name"]].epsilon(CONFIDENCE)
        ly["x"].copy_(torch.randn(ly["M"], ly["K"], device=dev, generator=g).to(torch.bfloat16))  # held-out

    # ---- capture one step (50 launches) as a CUDA graph, protected and unprotected
    def capture(protect):
        for ly in layers:
            launch(ly, protect)  # warm: configures smem attributes, allocates workspaces
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for ly in layers:
                launch(ly, protect)
        return graph

    if args.eager:  # eager launches (programmatic dependent launch overlaps consecutive kernels)
        class _Eager:
            def __init__(self, protect):
                self.protect = protect

            def replay(self):
                for ly in layers:
                    launch(ly, self.protect)
        for ly in layers:
            launch(ly, True)
            launch(ly, False)
        torch.cuda.synchronize()
        g_prot, g_unprot = _Eager(True), _Eager(False)
    else:
        g_prot = capture(True)
        g_unprot = capture(False)
    stream = torch.cuda.current_stream(dev)

    def timed(graph, steps, warmup):
        for _ in range(warmup):
            graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            graph.replay()
        t1.record(stream)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        if world > 1:
            tt = torch.tensor([ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ms = float(tt.item())
            torch.distributed.barrier()
        return ms

    with ClockSampler(local_rank) as clk:
        ms_prot = timed(g_prot, args.steps, args.warmup)
    ms_unprot = timed(g_unprot, args.steps, args.warmup)

    # held-out false flags of the timed batches (K5 counter reduce over NCCL when world > 1)
    nflag = torch.stack([ly["res"].nflag[0].long() for ly in layers]).sum().reshape(1)
    if world > 1:
        torch.distributed.all_reduce(nflag)
    false_flags = int(nflag.item())

    # ---- end to end through the public API: pinned host input in, flags + logits out, per step
    e2e = measure_e2e(layers, launch, dev, args, world)

    act_gb = sum(ly["x"].numel() * 2 + ly["y"].numel() * 2 for ly in layers) / 1e9
    value = flops * world / (ms_prot * 1e-3) / 1e12
    unprot = flops * world / (ms_unprot * 1e-3) / 1e12
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("bf16_tflops_sustained") or 1400.0
    per_gpu = value / world
    out = {
        "metric": "protected_gemm_tflops", "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_prot, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, "
        "N(0,1) activations of ViT-B/16 GEMM shapes)",
        "config": {"workload": "vit_b16_b256_protected_gemms", "global_batch": BATCH * world, "seq_len": TOKENS,
                   "gemms_per_step": len(layers), "parallelism": f"replicas{world}",
                   "epsilon": f"per-layer mu +/- z*sigma, c={CONFIDENCE}",
                   "l2": f"inputs larger than L2 ({act_gb:.1f} GB of distinct activations per step)"},
        "overhead_pct": 100.0 * (ms_prot / ms_unprot - 1.0),
        "unprotected_tflops": unprot,
        "vit_b16_protected_gemm_img_per_s": BATCH * world / (ms_prot * 1e-3),
        "held_out_false_flags": false_flags,
        "roofline": {"bound": "tensor", "achieved": per_gpu, "peak": peak, "unit": "TFLOP/s",
                     "frac": per_gpu / peak, "traffic": step_traffic_bytes(),
                     "traffic_unit": "DRAM bytes per step (50 launches), ncu --set full",
                     "algorithmic_bytes": step_algorithmic_bytes(gemms),
                     "hbm_gbs_achieved": step_traffic_bytes() / (ms_prot * 1e-3) / 1e9,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, back to back 4 s)",
                     "kernel": "gg_protected_gemm_kernel<bf16,bf16,protect> (the only kernel in the step)"},
        "e2e": e2e,
        "gpu_launches": len(layers) * args.steps,
        "clocks": clk.summary(),
    }
    return out


def measure_e2e(layers, launch, dev, args, world):
    """Same metric through kernels.protected_gemm with the step's input batch
    copied from pinned host memory and the flags/summary + logits read back."""
    import torch

    first, head = layers[0], layers[-1]
    host_x = torch.empty_like(first["x"], device="cpu").pin_memory()
    host_x.copy_(first["x"].cpu())
    host_logits = torch.empty_like(head["y"], device="cpu").pin_memory()
    host_flags = torch.empty(len(layers), dtype=torch.int32).pin_memory()
    flops = gemm_flops([(ly["name"], ly["M"], ly["N"], ly["K"]) for ly in layers])

    # the next step's input batch is copied on a side stream while this step computes
    # (double-buffered layer-0 input); every step still moves its whole batch from pinned
    # host memory and the host consumes flags + logits before the next step
    x_bufs = [first["x"], torch.empty_like(first["x"])]
    copy_stream = torch.cuda.Stream(dev)
    compute = torch.cuda.current_stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]

    def prefetch(i):
        copy_stream.wait_stream(compute)  # the buffer's previous reader (step i - 2) has finished
        with torch.cuda.stream(copy_stream):
            x_bufs[i % 2].copy_(host_x, non_blocking=True)
            copied[i % 2].record(copy_stream)

    def step(i):
        compute.wait_event(copied[i % 2])
        first["x"] = x_bufs[i % 2]
        prefetch(i + 1)  # always: the timed region holds exactly one full batch copy per step
        for ly in layers:
            launch(ly)
        host_flags.copy_(torch.cat([ly["res"].nflag for ly in layers]), non_blocking=True)
        host_logits.copy_(head["y"], non_blocking=True)

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
        compute.synchronize()  # the host consumes flags + logits every step
    compute.wait_stream(copy_stream)
    ev1.record()
    torch.cuda.synchronize()
    first["x"] = x_bufs[0]
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    return {"value": flops * world / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": host_x.numel() * host_x.element_size(),
            "d2h_bytes_per_step": host_logits.numel() * host_logits.element_size() + host_flags.numel() * 4,
            "ms_per_step": ms, "host_wall_ms_per_step": 1e3 * (time.perf_counter() - t0) / args.steps}


def cpu_baseline(args) -> dict:
    workers = os.cpu_count() or 1
    t, f = reference_step(args.ref_rows, workers, vit_b16_gemms())
    return {"value": f / t / 1e12, "unit": "TFLOP/s", "cores": workers, "kind": "port",
            "sample": f"{args.ref_rows} rows (one image) of each of the 50 ViT-B/16 GEMMs, binary16-emulated x "
                      f"binary32 numerics.gemm + guard._verify_arrays (oracle port), {workers} processes, "
                      f"{t:.1f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--ref-rows", type=int, default=TOKENS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of one CUDA graph per step")
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
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
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
