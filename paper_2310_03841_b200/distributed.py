"""Multi-GPU plumbing of the protected path: sharding and counter reduction.

Batched inference and injection campaigns are independent units (SURVEY.md
§8(e)): every rank works on its own images / layers and nothing is exchanged
on the hot path.  The only collective is K5, one all-reduce(SUM) of the int64
campaign counters at the end (`guard.py:767-792`, `injector.py:335-345`);
integer sums are order-independent, so the result does not depend on the
number of ranks.  Floating-point loss sums are NOT reduced here (their order
would vary); gather records instead and sum them in (layer, k) order.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

COUNTER_FIELDS = ("injections", "mismatches", "true_positives", "false_negatives", "benign_detections",
                  "true_negatives", "skipped", "clean_checks", "clean_false_positive_checks",
                  "clean_false_positive_inferences", "flagged_rows")


def world() -> tuple[int, int]:
    """(rank, world_size); (0, 1) without an initialised process group."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(n: int, rank: int, world_size: int) -> range:
    """Contiguous share of n units for `rank` (sizes differ by at most one)."""
    lo = n * rank // world_size
    hi = n * (rank + 1) // world_size
    return range(lo, hi)


def counters_tensor(per_layer: dict[int, dict[str, int]], n_layers: int, device=None) -> torch.Tensor:
    """Pack per-layer integer tallies into an int64 [n_layers, len(COUNTER_FIELDS)] tensor."""
    t = torch.zeros((n_layers, len(COUNTER_FIELDS)), dtype=torch.int64, device=device)
    for layer, tally in per_layer.items():
        for j, name in enumerate(COUNTER_FIELDS):
            t[layer, j] = int(tally.get(name, 0))
    return t


def reduce_counters(t: torch.Tensor) -> torch.Tensor:
    """K5: all-reduce(SUM) of the int64 counter tensor across ranks (NCCL on GPUs, gloo on CPU)."""
    if t.dtype != torch.int64:
        raise ValueError("campaign counters are int64 (order-independent sums)")
    r, w = world()
    if w > 1:
        if t.is_cuda and dist.get_backend() == "gloo":  # gloo reduces host tensors
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def unpack_counters(t: torch.Tensor) -> dict[int, dict[str, int]]:
    out = {}
    for layer in range(t.shape[0]):
        row = t[layer].tolist()
        if any(row):
            out[layer] = {name: int(v) for name, v in zip(COUNTER_FIELDS, row)}
    return out
