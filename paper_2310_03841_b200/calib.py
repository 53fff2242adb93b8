"""Device-resident calibration and range profiling.

The reference collects every clean discrepancy of a layer on the host and takes
mean and std(ddof=1) (``guard.calibrate_epsilon``, guard.py:300-355), and
profiles each layer's output range with a host min/max pass
(``profiler.profile_ranges``, profiler.py:62-80).  For batched B200 runs those
host passes are replaced by two C-ABI kernels whose state stays on the device:

* ``RunningStats.update(d)``: ``gg_running_stats`` merges a batch of the fused
  check's d into (count, mean, M2).  The merge is deterministic: fixed chunks
  and a fixed tree.
* ``RunningRange.update(y)``: ``gg_minmax`` folds a layer output into
  (min, max, non-finite count).

Across ranks, ``merge_stats`` / ``merge_ranges`` combine all-gathered states in
rank order, so a sharded calibration gives the same ε on every world size up
to the associativity of Chan's merge.  Thresholds use the reference's own
``threshold_from_confidence``.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib as L
from .guard import threshold_from_confidence
from .kernels import _require_cuda, _stream

_TOP = 1 << 63
_MASK = (1 << 64) - 1


def _key_to_float(key: int) -> float:
    """Inverse of the kernel's order-preserving double -> uint64 map."""
    key &= _MASK
    bits = (key ^ _TOP) if key & _TOP else (~key & _MASK)
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def _float_to_key(v: float) -> int:
    """The kernel's map (gg_minmax), for tests and host-side merges."""
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    return (~bits & _MASK) if bits >> 63 else (bits | _TOP)


@dataclass
class Moments:
    count: float
    mean: float
    m2: float

    @property
    def sigma(self) -> float:
        return math.sqrt(self.m2 / (self.count - 1)) if self.count > 1 else 0.0


def merge_moments(parts: list[Moments]) -> Moments:
    """Chan's pairwise merge, left to right (same formula as the kernel)."""
    acc = Moments(0.0, 0.0, 0.0)
    for b in parts:
        if b.count == 0:
            continue
        if acc.count == 0:
            acc = Moments(b.count, b.mean, b.m2)
            continue
        n = acc.count + b.count
        delta = b.mean - acc.mean
        acc = Moments(n, acc.mean + delta * (b.count / n), acc.m2 + b.m2 + delta * delta * (acc.count * b.count / n))
    return acc


class RunningStats:
    """Streaming (count, mean, M2) of a layer's clean discrepancies, on the device."""

    def __init__(self, device):
        self.state = torch.zeros(3, dtype=torch.float64, device=device)

    def update(self, d: torch.Tensor) -> None:
        dev = _require_cuda(d)
        if d.dtype != torch.float64 or d.dim() != 1 or not d.is_contiguous():
            raise ValueError("running stats take a contiguous 1-D float64 discrepancy vector")
        L.check(L.load().gg_running_stats(d.data_ptr(), d.numel(), self.state.data_ptr(), _stream(dev)),
                "gg_running_stats")

    def moments(self) -> Moments:
        n, mean, m2 = self.state.tolist()
        return Moments(n, mean, m2)

    def epsilon(self, confidence: float) -> tuple[float, float, float]:
        """(mu, lo, hi) with the reference's z-quantile rule."""
        m = self.moments()
        lo, hi = threshold_from_confidence(m.mean, m.sigma, confidence)
        return m.mean, lo, hi


class RunningRange:
    """Streaming min / max (finite values) and non-finite count of a layer's outputs."""

    def __init__(self, device):
        self.state = torch.tensor([-1, 0, 0], dtype=torch.int64, device=device)  # {~0, 0, 0}

    def update(self, y: torch.Tensor) -> None:
        dev = _require_cuda(y)
        dt = {torch.bfloat16: L.GG_BF16, torch.float16: L.GG_F16, torch.float32: L.GG_F32,
              torch.int32: L.GG_I32}.get(y.dtype)
        if dt is None or y.dim() != 2 or y.stride(1) != 1:
            raise ValueError("range profiling takes a 2-D row-major bf16 / f16 / f32 / i32 layer output")
        L.check(L.load().gg_minmax(dt, y.data_ptr(), y.shape[0], y.shape[1], y.stride(0), self.state.data_ptr(),
                                   _stream(dev)), "gg_minmax")

    def bounds(self) -> tuple[float, float, int]:
        lo_k, hi_k, bad = (v & _MASK for v in self.state.tolist())
        if lo_k == _MASK and hi_k == 0:
            return math.inf, -math.inf, bad
        return _key_to_float(lo_k), _key_to_float(hi_k), bad


def merge_stats(local: RunningStats) -> Moments:
    """All-gather every rank's moments and merge them in rank order (identity on one process)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local.moments()
    t = local.state.detach().to(torch.float64)
    if dist.get_backend() == "gloo":  # gloo gathers host tensors
        t = t.cpu()
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return merge_moments([Moments(*p.tolist()) for p in parts])


def merge_ranges(local: RunningRange) -> tuple[float, float, int]:
    """All-reduce MIN / MAX / SUM of the order keys across ranks."""
    lo, hi, bad = local.bounds()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return lo, hi, bad
    dev = local.state.device
    t_lo = torch.tensor([lo], dtype=torch.float64, device=dev)
    t_hi = torch.tensor([hi], dtype=torch.float64, device=dev)
    t_bad = torch.tensor([bad], dtype=torch.int64, device=dev)
    dist.all_reduce(t_lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(t_hi, op=dist.ReduceOp.MAX)
    dist.all_reduce(t_bad, op=dist.ReduceOp.SUM)
    return t_lo.item(), t_hi.item(), int(t_bad.item())
