"""Layer-vulnerability injection campaign on a protected ViT (BASELINE.json
configs[3]: ViT-L/16 fp16 / tf32, 1e6 trials sharded across GPUs, NCCL
counter reduce).

    python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype fp16 --trials 1000000
    torchrun --nproc-per-node 8 -m paper_2310_03841_b200.campaign_vit ...   (one rank per GPU)

Each rank builds the same random-init model (same seed) and golden batch,
calibrates the per-layer epsilon on its own clean batches (merged across ranks
in rank order: calib.merge_stats), takes its share of the (layer, block)
units (campaign.plan_units, balanced by suffix cost) and runs them as batched
trials (campaign.ViTCampaign: one trial per image, prefix reuse, device-side
mismatch / detection counters).  K5 all-reduces the int64 counters once at
the end; rank 0 prints one JSON line with trials/s (whole job, device-timed
as the max over ranks), the per-layer-role vulnerability (mismatch rate =
P_prop of analysis.compute_p_prop, analysis.py:101-106) and the coverage of
output-mismatching flips with its Wilson interval.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import time

import torch
import torch.distributed as dist

from . import calib
from .campaign import FIELDS, ViTCampaign, select_golden_images, wilson_interval
from .vit import VIT_B16, VIT_L16, ProtectedViT, ViTConfig

MODELS = {"vit_b16": VIT_B16, "vit_l16": VIT_L16}
DTYPES = {"bf16": (torch.bfloat16, "3xtf32"), "fp16": (torch.float16, "3xtf32"), "tf32": (torch.float32, "tf32"),
          "f32": (torch.float32, "3xtf32")}


def calibrate_distributed(model: ProtectedViT, batches, confidence: float) -> None:
    """Per-layer epsilon from every rank's clean batches (moments merged in rank order)."""
    stats = {lin.index: calib.RunningStats(model.device_) for lin in model.linears if not lin.integer}
    for lin in model.linears:
        lin.set_epsilon(0.0, -math.inf, math.inf)

    def hook(lin, res):
        if lin.index in stats:
            stats[lin.index].update(res.d)

    model.hooks.append(hook)
    try:
        with torch.no_grad():
            for b in batches:
                model.forward(b, protect=True)
    finally:
        model.hooks.remove(hook)
    z_lo_hi = calib.threshold_from_confidence
    for lin in model.linears:
        if lin.index in stats:
            m = calib.merge_stats(stats[lin.index])
            lo, hi = z_lo_hi(m.mean, m.sigma, confidence)
            lin.set_epsilon(m.mean, lo, hi)


def run(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    cfg: ViTConfig = MODELS[args.model]
    dtype, f32_mode = DTYPES[args.dtype]
    model = ProtectedViT(cfg, dtype=dtype, device=dev, seed=args.seed, f32_mode=f32_mode)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    gold_g = torch.Generator(device=dev).manual_seed(7)  # the same golden batch on every rank
    mk = lambda gen: torch.randn(args.batch, 3, cfg.image, cfg.image, device=dev, generator=gen).to(dtype)  # noqa: E731
    calibrate_distributed(model, [mk(g) for _ in range(args.cal_batches)], args.confidence)
    gstats = {"selection": "random synthetic images (no teacher filter)"}
    if args.teacher:
        teacher = ProtectedViT(cfg, dtype=torch.float32, device=dev, seed=args.seed, f32_mode="3xtf32")
        golden, gstats = select_golden_images(model, teacher, lambda: mk(gold_g), args.batch)
        del teacher
        torch.cuda.empty_cache()
    else:
        golden = mk(gold_g)
    camp = ViTCampaign(model, golden, seed=args.seed, modes=tuple(args.modes.split(",")))
    n_layers = cfg.n_layers
    per_layer = math.ceil(args.trials / n_layers)
    n_blocks = math.ceil(per_layer / args.batch)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    tally = camp.run(n_blocks, rank=rank, world_size=world)  # K5 inside
    ev1.record()
    torch.cuda.synchronize()
    s = ev0.elapsed_time(ev1) / 1e3
    wall = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([s, wall], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        s, wall = t.tolist()
    if rank != 0:
        return None
    summ = tally.summary()
    c = tally.counters
    roles = {}
    for name, idx in model.role_groups().items():
        inj = int(c[idx, FIELDS.index("injections")].sum())
        mm = int(c[idx, FIELDS.index("mismatches")].sum())
        tp = int(c[idx, FIELDS.index("true_positives")].sum())
        fn = int(c[idx, FIELDS.index("false_negatives")].sum())
        roles[name] = {"injections": inj, "mismatches": mm, "p_prop": mm / inj if inj else 0.0,
                       "coverage": tp / (tp + fn) if tp + fn else 1.0, "wilson95": wilson_interval(tp, tp + fn)}
    gemm_f, attn_f = cfg.flops_per_image()
    return {"config": "cfg4", "model": cfg.name, "dtype": args.dtype, "n_gpus": world, "trials": summ["injections"],
            "skipped": summ["skipped"], "blocks_per_layer": n_blocks, "images_per_block": args.batch,
            "device_s": s, "wall_s": wall, "trials_per_s": summ["injections"] / s,
            "full_forward_flop_per_trial": gemm_f + attn_f, "confidence": args.confidence,
            "summary": summ, "by_role": roles, "golden": gstats, "modes": args.modes,
            "scope": "one output bit flip per image of a 256-image batch at one protected layer, prefix reuse "
                     "(forward resumed at the layer), range-constrained exponent/mantissa flips, mismatch = "
                     "argmax change vs the clean prediction"}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--model", choices=sorted(MODELS), default="vit_l16")
    ap.add_argument("--dtype", choices=sorted(DTYPES), default="fp16")
    ap.add_argument("--trials", type=int, default=1_000_000)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--cal-batches", type=int, default=2)
    ap.add_argument("--confidence", type=float, default=1.0 - 1e-9)
    ap.add_argument("--seed", type=int, default=2310)
    ap.add_argument("--modes", default="fp_exponent_bit,fp_mantissa_bit",
                    help="comma-separated sample_injection modes (bit modes or random_value)")
    ap.add_argument("--teacher", action=argparse.BooleanOptionalAction, default=True,
                    help="golden set = images the model classifies like its fp32 teacher (profiler.select_golden)")
    args = ap.parse_args()
    out = run(args)
    if out is not None:
        print(json.dumps(out), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
