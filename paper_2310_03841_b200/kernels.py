"""Torch-tensor front end of the C-ABI kernels (device memory in, device memory out).

torch is plumbing here: it owns device memory and the current stream; every
computation runs in ``libgemmguard_b200.so``.  Functions raise ValueError for
bad shapes/dtypes (the reference's convention) and never fall back to a CPU
path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib as L

TORCH_TO_GG = {
    torch.float64: L.GG_F64,
    torch.float32: L.GG_F32,
    torch.float16: L.GG_F16,
    torch.bfloat16: L.GG_BF16,
    torch.int8: L.GG_I8,
    torch.int32: L.GG_I32,
    torch.int64: L.GG_I64,
}
PREC_TORCH = {
    L.GG_P_F16: torch.float16,
    L.GG_P_F32: torch.float32,
    L.GG_P_F64: torch.float64,
    L.GG_P_I64: torch.int64,
}

INJ_DTYPE = np.dtype(
    [("row", "<i8"), ("col", "<i4"), ("bit", "<i4"), ("target", "<i4"), ("mode", "<i4"), ("value", "<f8")]
)
assert INJ_DTYPE.itemsize == ctypes.sizeof(L.GGInjection)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(*ts: torch.Tensor | None) -> torch.device:
    dev = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("device kernels take CUDA tensors (no CPU fallback)")
        dev = t.device if dev is None else dev
    if dev is None:
        raise ValueError("no CUDA tensor given")
    return dev


@dataclass
class Injection:
    """One fault for the protected-GEMM epilogue (gg_injection)."""

    row: int
    col: int
    bit: int = 0
    target: int = L.GG_INJ_OUTPUT
    mode: int = L.GG_INJ_BITFLIP
    value: float = 0.0


def injections_to_device(injs: Sequence[Injection], device: torch.device) -> torch.Tensor:
    """Pack injections for the epilogue, sorted by row as the C-ABI requires (stable)."""
    arr = np.zeros(len(injs), dtype=INJ_DTYPE)
    for i, f in enumerate(injs):
        arr[i] = (f.row, f.col, f.bit, f.target, f.mode, f.value)
    arr = arr[np.argsort(arr["row"], kind="stable")]
    return torch.from_numpy(arr.view(np.uint8).copy()).to(device, non_blocking=False)


@dataclass
class CheckResult:
    """Device-resident outcome of one protected launch (guard.DetectionOutcome)."""

    d: torch.Tensor  # [M] f64 or i64
    flags: torch.Tensor  # [M] u8
    max_disc: torch.Tensor  # [1] f64
    nflag: torch.Tensor  # [1] i32
    triggered: torch.Tensor  # [1] u8

    @classmethod
    def empty(cls, M: int, integer: bool, device) -> "CheckResult":
        return cls(
            d=torch.empty(M, dtype=torch.int64 if integer else torch.float64, device=device),
            flags=torch.empty(M, dtype=torch.uint8, device=device),
            max_disc=torch.empty(1, dtype=torch.float64, device=device),
            nflag=torch.empty(1, dtype=torch.int32, device=device),
            triggered=torch.empty(1, dtype=torch.uint8, device=device),
        )


_WS: dict[tuple, torch.Tensor] = {}


def workspace(M: int, N: int, device: torch.device, key=None) -> torch.Tensor:
    """Zero-initialised workspace for (M, N); every launch leaves it re-zeroed.

    One workspace per (device, shape, key, stream): launches on one stream are
    ordered, so they may share it (a replay finds its launch's band summaries),
    while launches on different streams never race on the same counters."""
    nbytes = int(L.load().gg_protected_gemm_workspace_bytes(M, N))
    k = (device, M, N, key, torch.cuda.current_stream(device).cuda_stream)
    ws = _WS.get(k)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _WS[k] = ws
    return ws


def _pad_k(t: torch.Tensor) -> torch.Tensor:
    """Row pitch must be a multiple of 16 bytes for TMA: pad storage, keep K."""
    K = t.shape[1]
    es = t.element_size()
    if t.stride(1) == 1 and (t.stride(0) * es) % 16 == 0 and t.data_ptr() % 16 == 0 and t.stride(0) >= K:
        return t
    step = 16 // es
    Kp = (K + step - 1) // step * step
    buf = torch.zeros((t.shape[0], Kp), dtype=t.dtype, device=t.device)
    buf[:, :K] = t
    return buf[:, :K]


def build_desc(
    x: torch.Tensor,
    w: torch.Tensor,
    y: torch.Tensor,
    bias: torch.Tensor | None,
    *,
    protect: bool,
    w_sum: torch.Tensor | None = None,
    w_aux: torch.Tensor | None = None,
    bias_sum: float | int = 0,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    statistic: int = L.GG_PER_SAMPLE,
    result: CheckResult | None = None,
    inj_dev: torch.Tensor | None = None,
    n_inj: int = 0,
    ws: torch.Tensor | None = None,
    replay_rows: torch.Tensor | None = None,
    changed: torch.Tensor | None = None,
    act: int = L.GG_ACT_NONE,
    pred_in: torch.Tensor | None = None,
    requant_shift: int = 0,
    residual: torch.Tensor | None = None,
) -> L.GGGemmDesc:
    M, K = x.shape
    N = w.shape[0]
    d = L.GGGemmDesc()
    d.ab_kind = TORCH_TO_GG[x.dtype]
    d.c_dtype = TORCH_TO_GG[y.dtype]
    d.M, d.N, d.K = M, N, K
    d.A, d.lda = x.data_ptr(), x.stride(0)
    d.B, d.ldb = w.data_ptr(), w.stride(0)
    d.bias = _ptr(bias)
    d.C, d.ldc = y.data_ptr(), y.stride(0)
    d.protect = 1 if protect else 0
    integer = x.dtype == torch.int8
    d.chk_prec = L.GG_P_I64 if integer else {torch.float32: L.GG_P_F32, torch.float16: L.GG_P_F16}.get(
        None if w_sum is None else w_sum.dtype, L.GG_P_F64)
    if protect:
        d.w_sum = _ptr(w_sum)
        d.w_aux = _ptr(w_aux)
        if integer:
            d.bias_sum_i = int(bias_sum)
        else:
            d.bias_sum_f = float(bias_sum)
        d.mu, d.lo, d.hi, d.statistic = float(mu), float(lo), float(hi), int(statistic)
        d.d = result.d.data_ptr()
        d.flags = result.flags.data_ptr()
        d.max_disc = result.max_disc.data_ptr()
        d.nflag = result.nflag.data_ptr()
        d.triggered = result.triggered.data_ptr()
        d.workspace = ws.data_ptr()
        d.workspace_bytes = ws.numel()
    d.inj = _ptr(inj_dev)
    d.n_inj = int(n_inj)
    d.replay_rows = _ptr(replay_rows)
    d.changed = _ptr(changed)
    d.epilogue_act = int(act)
    d.pred_in = _ptr(pred_in) if protect else None
    d.requant_shift = int(requant_shift)
    if residual is not None:
        if residual.shape != y.shape or residual.dtype != y.dtype or residual.stride(1) != 1:
            raise ValueError("residual must be [M, N] of the output dtype with contiguous rows")
        if residual.data_ptr() == y.data_ptr():
            raise ValueError("residual must not alias the output (a replay re-reads it)")
        d.residual, d.ld_res = residual.data_ptr(), residual.stride(0)
    return d


F32_MODES = ("3xtf32", "tf32")


def _f32_mode(mode: str) -> str:
    if mode not in F32_MODES:
        raise ValueError(f"f32_mode must be one of {F32_MODES}, got {mode!r}")
    return mode


def tf32x3_segment(K: int) -> int:
    """Width of one K segment of a 3xTF32 expansion (K rounded up to 32)."""
    return (K + 31) // 32 * 32


def split_tf32x3(t: torch.Tensor, role: int) -> torch.Tensor:
    """gg_split_tf32x3: fp32 [rows, K] -> [rows, 3*Ks]; role 0 (X): [hi|lo|hi],
    role 1 (W [N, K]): [lo|hi|hi].  A tf32 launch over the expanded operands
    computes the binary32 GEMM to ~2^-21 per product (3xTF32), the small
    cross terms accumulated first."""
    dev = _require_cuda(t)
    if t.dtype != torch.float32 or t.dim() != 2:
        raise ValueError("split_tf32x3 takes a 2-D float32 tensor")
    if t.stride(1) != 1:
        t = t.contiguous()
    rows, K = t.shape
    Ks = tf32x3_segment(K)
    out = torch.empty((rows, 3 * Ks), dtype=torch.float32, device=dev)
    L.check(L.load().gg_split_tf32x3(t.data_ptr(), rows, K, t.stride(0), int(role), out.data_ptr(), out.stride(0),
                                     _stream(dev)), "gg_split_tf32x3")
    return out


def checksum_aux(w_sum: torch.Tensor, ab_dtype: torch.dtype, f32_mode: str = "3xtf32") -> torch.Tensor | None:
    """Side-path encoding of w_sum for the fused checksum (gg_checksum_aux):
    fp32(w_sum) for float operands (bf16 / fp16 / tf32; [w | 0 | w] over the
    three segments of a 3xTF32 launch), signed base-256 digit planes for int8.
    Computed once per weight."""
    dev = _require_cuda(w_sum)
    kind = TORCH_TO_GG[ab_dtype]
    if ab_dtype == torch.float32 and _f32_mode(f32_mode) == "3xtf32":
        kind = L.GG_TF32X3
    K = w_sum.numel()
    nbytes = int(L.load().gg_checksum_aux_bytes(kind, K))
    if nbytes == 0:
        return None
    if kind != L.GG_I8 and w_sum.dtype != torch.float64:  # binary16 / binary32 checksum precisions
        w_sum = w_sum.to(torch.float64)
    aux = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    L.check(L.load().gg_checksum_aux(kind, w_sum.data_ptr(), K, aux.data_ptr(), _stream(dev)), "gg_checksum_aux")
    return aux


def _check_gemm_operands(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None):
    if x.dim() != 2 or w.dim() != 2:
        raise ValueError("protected_gemm requires 2-D operands")
    if x.shape[1] != w.shape[1]:
        raise ValueError(f"gemm dims mismatch: X is {tuple(x.shape)}, W is {tuple(w.shape)} ([N, K])")
    if x.dtype != w.dtype:
        raise ValueError(f"gemm operand dtypes differ: {x.dtype} vs {w.dtype}")
    if x.dtype not in (torch.bfloat16, torch.float16, torch.float32, torch.int8):
        raise ValueError(f"tensor-core path takes bf16, fp16, fp32 (tf32) or int8 operands, got {x.dtype}")
    if bias is not None:
        want = torch.int32 if x.dtype == torch.int8 else torch.float32
        if bias.dtype != want or bias.dim() != 1 or bias.shape[0] != w.shape[0]:
            raise ValueError(f"bias must be a [{w.shape[0]}] {want} tensor")


def default_out_dtype(ab: torch.dtype) -> torch.dtype:
    """Result rounded to the operand dtype (numerics.py:289); int8 -> int32."""
    return {torch.bfloat16: torch.bfloat16, torch.float16: torch.float16, torch.float32: torch.float32,
            torch.int8: torch.int32}[ab]


def _check_pred(pred_in: torch.Tensor | None, M: int) -> torch.Tensor | None:
    if pred_in is not None and (pred_in.dtype != torch.int64 or pred_in.numel() < M or not pred_in.is_contiguous()):
        raise ValueError("pred_in must be a contiguous int64 (fp32 pair bits) tensor with one entry per row")
    return pred_in


def _prepare_operands(x, w, w_sum, w_aux, protect, f32_mode, w_split):
    """TMA-ready operands (16-byte pitches) and the matching checksum encoding;
    fp32 operands are expanded for 3xTF32 unless f32_mode="tf32"."""
    if x.dtype == torch.float32 and _f32_mode(f32_mode) == "3xtf32":
        xs = split_tf32x3(x, 0)
        ws = w_split if w_split is not None else split_tf32x3(w, 1)
        if ws.shape != (w.shape[0], xs.shape[1]):
            raise ValueError("w_split does not match the weight's 3xTF32 expansion")
        if protect and w_aux is None and w_sum is not None:
            w_aux = checksum_aux(w_sum, torch.float32, "3xtf32")
    else:
        xs, ws = _pad_k(x), _pad_k(w)
        if protect and w_aux is None and w_sum is not None:
            w_aux = checksum_aux(w_sum, x.dtype, f32_mode)
    if protect and w_aux is not None:
        need = int(L.load().gg_checksum_aux_bytes(TORCH_TO_GG[xs.dtype], xs.shape[1]))
        if w_aux.numel() * w_aux.element_size() < need:
            raise ValueError("w_aux does not match this launch's operand kind (3xTF32 vs tf32?)")
    return xs, ws, w_aux


def protected_gemm(
    x: torch.Tensor,
    w: torch.Tensor,
    bias: torch.Tensor | None = None,
    *,
    out_dtype: torch.dtype | None = None,
    protect: bool = True,
    w_sum: torch.Tensor | None = None,
    w_aux: torch.Tensor | None = None,
    bias_sum: float | int = 0,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    statistic: int = L.GG_PER_SAMPLE,
    injections: Sequence[Injection] | torch.Tensor | None = None,
    out: torch.Tensor | None = None,
    result: CheckResult | None = None,
    ws_key=None,
    f32_mode: str = "3xtf32",
    w_split: torch.Tensor | None = None,
    act: int = L.GG_ACT_NONE,
    pred_in: torch.Tensor | None = None,
    requant_shift: int = 0,
    residual: torch.Tensor | None = None,
) -> tuple[torch.Tensor, CheckResult | None]:
    """K1: y = x @ w.T + bias with the fused checksum check (one launch).

    x [M, K], w [N, K] (torch Linear layout), bias [N] (f32, or i32 for int8).
    fp32 operands run as 3xTF32 (binary32 accuracy; `w_split` may hold the
    weight's cached `split_tf32x3(w, 1)`) unless f32_mode="tf32" (one tf32 pass).
    act=GG_ACT_GELU_TANH stores GELU(y) (16-bit outputs) after the check of y.
    pred_in [M] (uint64 fp32 (hi, lo) pairs): the predicted row sums x . w_sum
    computed by x's producer (add_layernorm's pred_out); K1 then skips its own.
    int8 operands with out_dtype=torch.int8 and requant_shift s store the requantised hidden
    state clip(((relu ? max(y, 0) : y) + 2^(s-1)) >> s, -128, 127) of the checked int32 y
    (act=GG_ACT_RELU for the relu; model.finish_layer_output's elementwise part).
    residual [M, N] (16-bit outputs): the stored output is round(residual + y) of the checked y
    (a transformer block's residual update fused; act becomes GG_ACT_RESIDUAL).
    Returns (y, CheckResult or None when protect=False).
    """
    dev = _require_cuda(x, w, bias)
    _check_gemm_operands(x, w, bias)
    x, w, w_aux = _prepare_operands(x, w, w_sum, w_aux, protect, f32_mode, w_split)
    M, N = x.shape[0], w.shape[0]
    odt = out_dtype or default_out_dtype(x.dtype)
    y = out if out is not None else torch.empty((M, N), dtype=odt, device=dev)
    if protect:
        if w_sum is None:
            raise ValueError("protect=True needs the offline checksum w_sum")
        result = result or CheckResult.empty(M, x.dtype == torch.int8, dev)
        ws = workspace(M, N, dev, ws_key)
    else:
        ws = None
    if isinstance(injections, torch.Tensor):
        inj_dev, n_inj = injections, injections.numel() // INJ_DTYPE.itemsize
    elif injections:
        inj_dev, n_inj = injections_to_device(injections, dev), len(injections)
    else:
        inj_dev, n_inj = None, 0
    desc = build_desc(x, w, y, bias, protect=protect, w_sum=w_sum, w_aux=w_aux, bias_sum=bias_sum, mu=mu, lo=lo,
                      hi=hi, statistic=statistic, result=result, inj_dev=inj_dev, n_inj=n_inj, ws=ws, act=act,
                      pred_in=_check_pred(pred_in, M), requant_shift=requant_shift, residual=residual)
    if residual is not None:
        desc.epilogue_act = L.GG_ACT_RESIDUAL
    L.check(L.load().gg_protected_gemm(ctypes.byref(desc), _stream(dev)), "gg_protected_gemm")
    return y, (result if protect else None)


def protected_gemm_wt(
    x: torch.Tensor,
    wt: torch.Tensor,
    bias: torch.Tensor | None = None,
    *,
    protect: bool = True,
    w_sum: torch.Tensor | None = None,
    w_aux: torch.Tensor | None = None,
    bias_sum: float | int = 0,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    statistic: int = L.GG_PER_SAMPLE,
    out: torch.Tensor | None = None,
    result: CheckResult | None = None,
    ws_key=None,
    f32_mode: str = "tf32",
) -> tuple[torch.Tensor, CheckResult | None]:
    """K1 on the reference's weight layout Wt [K, N] (numerics.gemm's `Wt`, model.py:43):
    the descriptor's b_layout = GG_B_KN, so the launcher transposes Wt into a scratch buffer
    and runs the K-major kernel -- results identical to protected_gemm(x, Wt.T.contiguous()).
    fp32 operands take the single-pass tf32 engine here (3xTF32 splits a [N, K] weight)."""
    dev = _require_cuda(x, wt, bias)
    if x.dim() != 2 or wt.dim() != 2 or x.shape[1] != wt.shape[0]:
        raise ValueError(f"gemm dims mismatch: X is {tuple(x.shape)}, Wt is {tuple(wt.shape)} ([K, N])")
    _check_gemm_operands(x, wt.t(), bias)
    if x.dtype == torch.float32 and _f32_mode(f32_mode) != "tf32":
        raise ValueError("protected_gemm_wt: fp32 operands need f32_mode='tf32' (3xTF32 splits [N, K] weights)")
    if wt.stride(1) != 1:
        raise ValueError("protected_gemm_wt: Wt rows must be contiguous")
    xs = _pad_k(x)
    M, N = x.shape[0], wt.shape[1]
    lib = L.load()
    scratch = torch.empty(int(lib.gg_b_scratch_bytes(TORCH_TO_GG[x.dtype], N, x.shape[1])), dtype=torch.uint8,
                          device=dev)
    y = out if out is not None else torch.empty((M, N), dtype=default_out_dtype(x.dtype), device=dev)
    if protect:
        if w_sum is None:
            raise ValueError("protect=True needs the offline checksum w_sum")
        if w_aux is None:
            w_aux = checksum_aux(w_sum, x.dtype, f32_mode)
        result = result or CheckResult.empty(M, x.dtype == torch.int8, dev)
        ws = workspace(M, N, dev, ws_key)
    else:
        ws = None
    desc = build_desc(xs, wt.t(), y, bias, protect=protect, w_sum=w_sum, w_aux=w_aux, bias_sum=bias_sum, mu=mu,
                      lo=lo, hi=hi, statistic=statistic, result=result, ws=ws)
    desc.ldb = wt.stride(0)
    desc.b_layout = L.GG_B_KN
    desc.b_scratch = scratch.data_ptr()
    desc.b_scratch_bytes = scratch.numel()
    L.check(lib.gg_protected_gemm(ctypes.byref(desc), _stream(dev)), "gg_protected_gemm")
    return y, (result if protect else None)


def packed_output_campaign(
    x: torch.Tensor,
    w: torch.Tensor,
    bias: torch.Tensor | None,
    faults: Sequence[Injection],
    *,
    w_sum: torch.Tensor,
    w_aux: torch.Tensor | None = None,
    bias_sum: float | int = 0,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    f32_mode: str = "3xtf32",
) -> tuple[torch.Tensor, int]:
    """Campaign engine for independent single-fault trials on one layer input:
    fault i is detected iff its row is flagged by a launch that injects it.

    The check is per row (guard.py:188-215), so faults in distinct rows do not
    interact. They are packed greedily into as few protected launches as there
    are faults per row. Returns (detected [len(faults)] bool on the device,
    number of launches); the verdicts equal one launch per fault."""
    dev = _require_cuda(x, w, bias)
    groups: list[list[int]] = []
    used: list[set[int]] = []
    for i, f in enumerate(faults):
        for g, u in zip(groups, used):
            if f.row not in u:
                u.add(f.row)
                g.append(i)
                break
        else:
            groups.append([i])
            used.append({f.row})
    detected = torch.zeros(len(faults), dtype=torch.bool, device=dev)
    M = x.shape[0]
    res = CheckResult.empty(M, x.dtype == torch.int8, dev)
    y = torch.empty((M, w.shape[0]), dtype=default_out_dtype(x.dtype), device=dev)
    for g in groups:
        inj = injections_to_device([faults[i] for i in g], dev)
        protected_gemm(x, w, bias, w_sum=w_sum, w_aux=w_aux, bias_sum=bias_sum, mu=mu, lo=lo, hi=hi, injections=inj,
                       out=y, result=res, f32_mode=f32_mode)
        idx = torch.tensor(g, dtype=torch.int64, device=dev)
        rows = torch.tensor([faults[i].row for i in g], dtype=torch.int64, device=dev)
        detected[idx] = res.flags[rows].bool()
    return detected, len(groups)


def replay_tiles(
    x: torch.Tensor,
    w: torch.Tensor,
    bias: torch.Tensor | None,
    y: torch.Tensor,
    replay_rows: torch.Tensor,
    result: CheckResult,
    *,
    w_sum: torch.Tensor,
    w_aux: torch.Tensor | None = None,
    bias_sum: float | int = 0,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    statistic: int = L.GG_PER_SAMPLE,
    changed: torch.Tensor | None = None,
    ws_key=None,
    f32_mode: str = "3xtf32",
    w_split: torch.Tensor | None = None,
    act: int = L.GG_ACT_NONE,
    pred_in: torch.Tensor | None = None,
    requant_shift: int = 0,
    residual: torch.Tensor | None = None,
) -> torch.Tensor:
    """K4: recompute only the M-bands holding a flagged row, in place in y.

    Must use the same operands, f32_mode and ws_key as the launch it replays.
    Returns the device scalar count of outputs whose bytes changed (0 means
    the recompute reproduced the flagged output: guard.py:590-594).
    """
    dev = _require_cuda(x, w, y, replay_rows)
    _check_gemm_operands(x, w, bias)
    x, w, w_aux = _prepare_operands(x, w, w_sum, w_aux, True, f32_mode, w_split)
    M, N = x.shape[0], w.shape[0]
    changed = changed if changed is not None else torch.zeros(1, dtype=torch.int32, device=dev)
    ws = workspace(M, N, dev, ws_key)
    desc = build_desc(x, w, y, bias, protect=True, w_sum=w_sum, w_aux=w_aux, bias_sum=bias_sum, mu=mu, lo=lo, hi=hi,
                      statistic=statistic, result=result, ws=ws, replay_rows=replay_rows, changed=changed, act=act,
                      pred_in=_check_pred(pred_in, M), requant_shift=requant_shift, residual=residual)
    if residual is not None:
        desc.epilogue_act = L.GG_ACT_RESIDUAL
    L.check(L.load().gg_replay_tiles(ctypes.byref(desc), _stream(dev)), "gg_replay_tiles")
    return changed


BAND_ROWS, TILE_COLS = 128, 256  # K1's row band (one CTA) and column tile (one CTA pair)


def locate_tiles(
    x: torch.Tensor,
    w: torch.Tensor,
    bias: torch.Tensor | None,
    y: torch.Tensor,
    result: CheckResult,
    *,
    mu: float = 0.0,
    frac: float = 0.5,
    with_columns: bool = False,
) -> tuple[torch.Tensor, torch.Tensor | None]:
    """Column checksums of the flagged bands (gg_locate_tiles): which 256-column tiles of
    each 128-row band hold the fault its row check flagged.

    Returns (tile_mask [ceil(M/128), ceil(N/256)] uint8, col_disc [ceil(M/128), N] or None):
    the column discrepancies e^T (X W^T + b) - e^T C of the flagged bands (int64 for int8,
    fp64 otherwise; zero rows for bands without a flag)."""
    dev = _require_cuda(x, w, bias, y)
    _check_gemm_operands(x, w, bias)
    if x.stride(1) != 1 or w.stride(1) != 1 or y.stride(1) != 1:
        raise ValueError("locate_tiles: rows must be contiguous")
    M, K = x.shape
    N = w.shape[0]
    mt, nt = (M + BAND_ROWS - 1) // BAND_ROWS, (N + TILE_COLS - 1) // TILE_COLS
    mask = torch.empty((mt, nt), dtype=torch.uint8, device=dev)
    integer = x.dtype == torch.int8
    cols = torch.zeros((mt, N), dtype=torch.int64 if integer else torch.float64, device=dev) if with_columns else None
    lib = L.load()
    ws = torch.empty(int(lib.gg_locate_workspace_bytes(M, K)), dtype=torch.uint8, device=dev)
    L.check(
        lib.gg_locate_tiles(
            TORCH_TO_GG[x.dtype], x.data_ptr(), M, K, x.stride(0), w.data_ptr(), N, w.stride(0), _ptr(bias),
            TORCH_TO_GG[bias.dtype] if bias is not None else 0, TORCH_TO_GG[y.dtype], y.data_ptr(), y.stride(0),
            result.flags.data_ptr(), result.d.data_ptr(), float(mu), float(frac), mask.data_ptr(), _ptr(cols),
            ws.data_ptr(), ws.numel(), _stream(dev),
        ),
        "gg_locate_tiles",
    )
    return mask, cols


def replay_located(
    x: torch.Tensor,
    w: torch.Tensor,
    bias: torch.Tensor | None,
    y: torch.Tensor,
    result: CheckResult,
    *,
    w_sum: torch.Tensor,
    bias_sum: float | int,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    f32_mode: str = "3xtf32",
    w_split: torch.Tensor | None = None,
    frac: float = 0.5,
    **band_kw,
) -> tuple[torch.Tensor, int]:
    """Tile-granular replay: locate the faulty (band, column tile) pairs by column checksums,
    recompute only those tiles with the clean weight (K1 on the tile's rows and columns:
    per-element the same MMA sequence, so a clean tile reproduces its bytes), then re-check
    the touched bands' rows (gg_verify_rows) and re-derive the launch summary.  A band whose
    rows still flag (a fault the columns did not place) falls back to K4 on its rows.

    Per-sample statistic and no fused epilogue activation (the check needs the raw output).
    Returns (changed outputs [1] int32 on the device, tiles recomputed)."""
    dev = _require_cuda(x, w, bias, y)
    integer = x.dtype == torch.int8
    mask, _ = locate_tiles(x, w, bias, y, result, mu=mu, frac=frac)
    tiles = mask.nonzero().tolist()
    changed = torch.zeros(1, dtype=torch.int32, device=dev)
    M, N = x.shape[0], w.shape[0]
    prec = L.GG_P_I64 if integer else L.GG_P_F64
    bsum = torch.tensor([bias_sum], dtype=torch.int64 if integer else torch.float64, device=dev)
    bands = sorted({b for b, _ in tiles})
    for b, t in tiles:
        r0, r1 = b * BAND_ROWS, min(M, (b + 1) * BAND_ROWS)
        c0, c1 = t * TILE_COLS, min(N, (t + 1) * TILE_COLS)
        view = y[r0:r1, c0:c1]
        old = view.clone()
        protected_gemm(x[r0:r1], w[c0:c1], None if bias is None else bias[c0:c1], protect=False, out=view,
                       f32_mode=f32_mode, w_split=None if w_split is None else w_split[c0:c1])
        bits = torch.int16 if view.element_size() == 2 else torch.int32
        changed += (view.view(bits) != old.view(bits)).sum().to(torch.int32)
    for b in bands:  # re-check the touched bands' rows in the reference order
        r0, r1 = b * BAND_ROWS, min(M, (b + 1) * BAND_ROWS)
        rb = verify_rows(x[r0:r1], y[r0:r1], w_sum, bsum, prec, mu=mu, lo=lo, hi=hi)
        result.d[r0:r1] = rb.d
        result.flags[r0:r1] = rb.flags
    keep = result.flags.clone()
    if bool(keep.any()):  # the columns did not place every fault: K4 on the rows still flagged
        replay_tiles(x, w, bias, y, keep, result, w_sum=w_sum, bias_sum=bias_sum, mu=mu, lo=lo, hi=hi,
                     changed=changed, f32_mode=f32_mode, w_split=w_split, **band_kw)
    _resummarise(result, mu, integer)  # from the rows (K4's standing band summaries predate the tile fix)
    return changed, len(tiles)


def _resummarise(result: CheckResult, mu: float, integer: bool) -> None:
    """nflag / triggered / max_disc over every row (the kernels' rule: the largest |d - mu|
    ignoring NaN, +inf when every d is NaN)."""
    f = result.flags
    n = f.to(torch.int32).sum()
    result.nflag.copy_(n.view(1))
    result.triggered.copy_((n > 0).to(torch.uint8).view(1))
    g = result.d.double().abs() if integer else (result.d - mu).abs()
    g = torch.where(torch.isnan(g), torch.full_like(g, -1.0), g)
    m = g.max()
    result.max_disc.copy_(torch.where(m < 0, torch.full_like(m, float("inf")), m).view(1))


def offline_checksum(
    w: torch.Tensor, bias: torch.Tensor | None, prec: int, *, layout: int = 0
) -> tuple[torch.Tensor, torch.Tensor]:
    """K2: (w_sum [K], bias_sum [1]) in precision `prec` (bit-exact, guard.py:142-160).

    layout 0: w is [N, K] (torch); layout 1: w is Wt [K, N] (reference)."""
    dev = _require_cuda(w, bias)
    w = w.contiguous()
    if layout == 0:
        N, K = w.shape
    else:
        K, N = w.shape
    pt = PREC_TORCH[prec]
    w_sum = torch.empty(K, dtype=pt, device=dev)
    bsum = torch.empty(1, dtype=pt, device=dev)
    b = None if bias is None else bias.contiguous()
    L.check(
        L.load().gg_offline_checksum(
            TORCH_TO_GG[w.dtype], w.data_ptr(), K, N, w.stride(0), layout, _ptr(b),
            TORCH_TO_GG[b.dtype] if b is not None else 0, prec, w_sum.data_ptr(), bsum.data_ptr(), _stream(dev),
        ),
        "gg_offline_checksum",
    )
    return w_sum, bsum


def verify_rows(
    x: torch.Tensor,
    y: torch.Tensor,
    w_sum: torch.Tensor,
    bias_sum: torch.Tensor,
    prec: int,
    *,
    mu: float = 0.0,
    lo: float = 0.0,
    hi: float = 0.0,
    statistic: int = L.GG_PER_SAMPLE,
) -> CheckResult:
    """Reference-exact guard._discrepancies + _verify_arrays on a given (X, Y)."""
    dev = _require_cuda(x, y, w_sum, bias_sum)
    x = x.contiguous()
    y = y.contiguous()
    M, K = x.shape
    N = y.shape[1]
    res = CheckResult.empty(M, prec == L.GG_P_I64, dev)
    L.check(
        L.load().gg_verify_rows(
            TORCH_TO_GG[x.dtype], x.data_ptr(), M, K, x.stride(0), TORCH_TO_GG[y.dtype], y.data_ptr(), N,
            y.stride(0), prec, w_sum.data_ptr(), bias_sum.data_ptr(), float(mu), float(lo), float(hi),
            int(statistic), res.d.data_ptr(), res.flags.data_ptr(), res.max_disc.data_ptr(),
            res.nflag.data_ptr(), res.triggered.data_ptr(), _stream(dev),
        ),
        "gg_verify_rows",
    )
    return res


def flip_bits(buf: torch.Tensor, elem_idx: torch.Tensor, bit_idx: torch.Tensor) -> None:
    """K3: in-place XOR of bit bit_idx[i] of element elem_idx[i] (involution)."""
    dev = _require_cuda(buf, elem_idx, bit_idx)
    if elem_idx.dtype != torch.int64 or bit_idx.dtype != torch.int32:
        raise ValueError("flip_bits: elem_idx must be int64 and bit_idx int32")
    n = elem_idx.numel()
    L.check(
        L.load().gg_flip_bits(buf.data_ptr(), buf.element_size(), elem_idx.data_ptr(), bit_idx.data_ptr(), n,
                              _stream(dev)),
        "gg_flip_bits",
    )


def gemm_exact(x: torch.Tensor, wt: torch.Tensor, bias: torch.Tensor | None, accum: int) -> torch.Tensor:
    """Bit-exact numerics.gemm on CUDA cores: x [M,K], wt [K,N] (reference layout)."""
    dev = _require_cuda(x, wt, bias)
    x = x.contiguous()
    wt = wt.contiguous()
    M, K = x.shape
    N = wt.shape[1]
    odt = torch.int32 if x.dtype in (torch.int8, torch.int32) else x.dtype
    y = torch.empty((M, N), dtype=odt, device=dev)
    b = None if bias is None else bias.contiguous()
    L.check(
        L.load().gg_gemm_exact(TORCH_TO_GG[x.dtype], accum, x.data_ptr(), M, K, wt.data_ptr(), N, _ptr(b),
                               y.data_ptr(), _stream(dev)),
        "gg_gemm_exact",
    )
    return y


def reduce(a: torch.Tensor, axis: int) -> torch.Tensor:
    """numerics.reduce_rows (axis=1) / reduce_cols (axis=0), ascending folds."""
    dev = _require_cuda(a)
    a = a.contiguous()
    rows, cols = a.shape
    integer = a.dtype in (torch.int8, torch.int32, torch.int64)
    out = torch.empty(rows if axis == 1 else cols, dtype=torch.int64 if integer else torch.float64, device=dev)
    L.check(L.load().gg_reduce(TORCH_TO_GG[a.dtype], a.data_ptr(), rows, cols, axis, out.data_ptr(), _stream(dev)),
            "gg_reduce")
    return out


def patchify(images: torch.Tensor, P: int, out: torch.Tensor) -> None:
    """gg_patchify: images [B, C, H, W] -> out [B * (H/P) * (W/P), C * P * P] (row (b, gy, gx),
    column (c, py, px)), the patch-embedding GEMM's input."""
    dev = _require_cuda(images, out)
    B, C, H, W = images.shape
    if not images.is_contiguous() or not out.is_contiguous() or out.dtype != images.dtype or \
            out.shape != (B * (H // P) * (W // P), C * P * P):
        raise ValueError("patchify: contiguous images [B, C, H, W] and out [B * H/P * W/P, C * P * P] of one dtype")
    L.check(L.load().gg_patchify(TORCH_TO_GG[images.dtype], images.data_ptr(), B, C, H, W, P, out.data_ptr(),
                                 _stream(dev)), "gg_patchify")


def embed_layernorm(e: torch.Tensor, pos: torch.Tensor, cls: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor,
                    eps: float, h_out: torch.Tensor, ln_out: torch.Tensor, w_pred: torch.Tensor | None = None,
                    pred_out: torch.Tensor | None = None) -> None:
    """gg_embed_layernorm: h_out[b, 0] = cls + pos[0], h_out[b, t] = e[b, t - 1] + pos[t] (rounded like
    torch's add), ln_out = LN(h_out) * gamma + beta (+ the consumer's predicted sums)."""
    dev = _require_cuda(e, pos, cls, gamma, beta, h_out, ln_out)
    T, D = pos.shape
    rows = h_out.shape[0]
    if rows % T or e.shape != (rows // T * (T - 1), D) or cls.shape != (D,) or ln_out.shape != (rows, D):
        raise ValueError("embed_layernorm: e [B*(T-1), D], pos [T, D], cls [D], h_out / ln_out [B*T, D]")
    for t in (e, pos, cls, h_out, ln_out):
        if not t.is_contiguous() or t.dtype != e.dtype:
            raise ValueError("embed_layernorm takes contiguous tensors of one dtype")
    L.check(L.load().gg_embed_layernorm(TORCH_TO_GG[e.dtype], e.data_ptr(), pos.data_ptr(), cls.data_ptr(),
                                        rows // T, T, D, gamma.data_ptr(), beta.data_ptr(), float(eps),
                                        h_out.data_ptr(), ln_out.data_ptr(), _ptr(w_pred), _ptr(pred_out),
                                        _stream(dev)),
            "gg_embed_layernorm")


def add_layernorm(h: torch.Tensor, y: torch.Tensor | None, gamma: torch.Tensor, beta: torch.Tensor, eps: float,
                  ln_out: torch.Tensor, h_out: torch.Tensor | None = None, w_pred: torch.Tensor | None = None,
                  pred_out: torch.Tensor | None = None) -> None:
    """gg_add_layernorm: h_out = h + y (if y is given; h_out may be h), ln_out = LN(.) * gamma + beta,
    and with w_pred (the consumer's fp32 checksum_aux) pred_out[row] = ln_out[row] . w_pred as
    fp32 (hi, lo) pair bits (the consumer launch's pred_in)."""
    dev = _require_cuda(h, y, gamma, beta, ln_out, h_out)
    rows, D = h.shape
    for t in (h, y, ln_out, h_out):
        if t is not None and (not t.is_contiguous() or t.shape != (rows, D) or t.dtype != h.dtype):
            raise ValueError("add_layernorm takes contiguous [rows, D] tensors of one dtype")
    if w_pred is not None and (w_pred.dtype != torch.uint8 and w_pred.dtype != torch.float32):
        raise ValueError("w_pred is the consumer's fp32 checksum_aux vector")
    L.check(L.load().gg_add_layernorm(TORCH_TO_GG[h.dtype], h.data_ptr(), _ptr(y), rows, D, gamma.data_ptr(),
                                      beta.data_ptr(), float(eps), _ptr(h_out), ln_out.data_ptr(), _ptr(w_pred),
                                      _ptr(pred_out), _stream(dev)),
            "gg_add_layernorm")
