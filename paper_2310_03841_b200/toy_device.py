"""Batched, device-resident forward of the integer toy pipeline.

``model.forward`` (model.py:359-391) runs one sample at a time, with the glue
between GEMMs (``finish_layer_output``, model.py:307-331) in NumPy on the host.
For integer models that glue is integer arithmetic, so it moves onto the
device bit-exactly (``gg_int_finish``):

* B samples go through each layer as one [B*T, K] protected GEMM;
* the hidden state stays in HBM between layers;
* the head reads each sample's class token;
* only the logits, plus the per-layer flags and ranges when asked for, come back.

Float models keep the host path: their layer norm and tanh-GELU would need the
reference's libm to be bit-identical.

``forward_batch`` returns the same logits, predictions and losses as
``model.forward`` per sample. With ``protect=True`` every layer runs the fused
int64-exact check (ε = 0, guard.py:148-152). With ``ranges=`` each layer's raw
output is folded into a ``calib.RunningRange``, which is the device
``profile_ranges``.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .calib import RunningRange
from .model import ModelGraph, _requant_shift, device_layer, loss_from_logits
from .numerics import Matrix2D


@dataclass
class BatchForward:
    logits: np.ndarray  # [B, classes] float64 (int32 logits widened, as model.forward does)
    predicted: np.ndarray  # [B] int
    losses: np.ndarray | None  # [B] softmax cross-entropy when labels are given
    flagged: dict[int, np.ndarray] | None  # protect=True: layer -> [B] bool (any flagged row of the sample)
    flagged_rows: dict[int, np.ndarray] | None = None  # protect=True: layer -> [B] flagged rows of the sample
    max_disc: dict[int, np.ndarray] | None = None  # protect=True: layer -> [B] max |d| over the sample's rows


def output_injection(spec_mode: str, bit, value, row: int, col: int) -> K.Injection:
    """An output fault of sample_injection as an in-epilogue descriptor (bit flip or value)."""
    if bit is not None and spec_mode not in ("random_value", "fixed_value"):
        return K.Injection(row=row, col=col, bit=int(bit))
    return K.Injection(row=row, col=col, mode=L.GG_INJ_SET_VALUE, value=float(value))


_CHK: dict[int, tuple[torch.Tensor, int]] = {}  # id(weight Matrix2D) -> (w_sum, bias_sum), dropped with the weight


def _checksum(layer, w_nk: torch.Tensor, bias: torch.Tensor):
    key = id(layer.weight)
    got = _CHK.get(key)
    if got is None:
        ws, bs = K.offline_checksum(w_nk, bias, L.GG_P_I64)
        got = (ws, int(bs.item()))
        _CHK[key] = got
        # a reused id must never find a dead weight's checksum (model._DEV does the same)
        weakref.finalize(layer.weight, _CHK.pop, key, None)
    return got


def forward_batch(model: ModelGraph, inputs: Sequence[Matrix2D], labels: Sequence[int] | None = None, *,
                  protect: bool = False, ranges: dict[int, RunningRange] | None = None,
                  device: torch.device | str = "cuda", injections: dict | None = None,
                  chks: dict | None = None) -> BatchForward:
    """Batched integer forward.  `injections`: {layer: [K.Injection]} output faults applied in
    that layer's GEMM epilogue (rows of the batched output: sample * rows_per_sample + row)."""
    if not model.is_integer:
        raise NotImplementedError("device glue covers integer models; float models use model.forward")
    if len(inputs) == 0:
        raise ValueError("forward_batch needs at least one input")
    dev = torch.device(device)
    B, T, D = len(inputs), model.tokens, model.input_dim
    for x in inputs:
        if x.dtype != model.dtype or x.shape != (T, D):
            raise ValueError(f"input must be {model.dtype} with shape ({T}, {D})")
    host = np.stack([np.asarray(x.data, dtype=np.int8) for x in inputs]).reshape(B * T, D)
    h = torch.from_numpy(host).to(dev)
    lib = L.load()
    stream = torch.cuda.current_stream(dev).cuda_stream
    flags = {} if protect else None
    nrows = {} if protect else None
    maxd = {} if protect else None
    logits = None
    for layer in model.layers:
        ent = device_layer(layer, model.dtype, "tensor")
        bias = ent.bias[("tensor", id(layer.bias))]
        head = layer.kind == "head"
        xin = h.view(B, T, -1)[:, 0, :].contiguous() if head else h
        inj = injections.get(layer.index) if injections else None
        # elementwise glue (relu + requantisation) fused into K1's epilogue: the check runs on the
        # int32 output, the int8 hidden state is what is stored; qkv's head mixing and the range
        # profile (which needs the int32 output) keep the separate gg_int_finish pass
        fuse = not head and layer.kind != "qkv" and ranges is None
        rq = dict(out_dtype=torch.int8, requant_shift=_requant_shift(layer.in_dim),
                  act=L.GG_ACT_RELU if layer.activation == "relu" else L.GG_ACT_NONE) if fuse else {}
        if protect:
            if chks is not None and layer.index in chks:  # the caller's offline checksums (guard.WeightChecksum)
                ws, bs = chks[layer.index].w_sum_device(), int(chks[layer.index].bias_sum)
            else:
                ws, bs = _checksum(layer, ent.w_nk, bias)
            y, res = K.protected_gemm(xin, ent.w_nk, bias, w_sum=ws, bias_sum=bs, lo=0, hi=0, injections=inj, **rq)
            rows = res.flags.view(B, -1) if not head else res.flags.view(B, 1)
            flags[layer.index] = rows.bool().any(dim=1)
            nrows[layer.index] = rows.to(torch.int32).sum(dim=1)
            maxd[layer.index] = res.d.view(B, -1).abs().max(dim=1).values
        else:
            y, _ = K.protected_gemm(xin, ent.w_nk, bias, protect=False, injections=inj, **rq)
        if fuse:
            h = y
            continue
        if ranges is not None:
            ranges.setdefault(layer.index, RunningRange(dev)).update(y)
        if head:
            logits = y
            break
        N = y.shape[1]
        qkv = layer.kind == "qkv"
        out = torch.empty((B * T, N // 3 if qkv else N), dtype=torch.int8, device=dev)
        L.check(lib.gg_int_finish(y.data_ptr(), B, T, N, y.stride(0), int(layer.activation == "relu"),
                                  _requant_shift(layer.in_dim), int(qkv), out.data_ptr(), stream), "gg_int_finish")
        h = out
    lg = logits.to(torch.float64).cpu().numpy()
    pred = lg.argmax(axis=1)
    losses = None if labels is None else np.array([loss_from_logits(lg[i], int(labels[i])) for i in range(B)])
    fl = None if flags is None else {i: f.cpu().numpy() for i, f in flags.items()}
    nr = None if nrows is None else {i: f.cpu().numpy() for i, f in nrows.items()}
    md = None if maxd is None else {i: f.cpu().numpy() for i, f in maxd.items()}
    return BatchForward(logits=lg, predicted=pred, losses=losses, flagged=fl, flagged_rows=nr, max_disc=md)
