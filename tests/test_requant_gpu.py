"""Fused int8 requantisation (descriptor requant_shift, c_dtype GG_I8; SURVEY §8(b) "epilogue
options (activation, int8 requant shift for the fused path)").

The check runs on the int32 GEMM output (guard.py:170), the stored output is
model.finish_layer_output's elementwise requantisation of it (model.py:312-316):
clip(((relu ? max(y, 0) : y) + 2^(s-1)) >> s, -128, 127) with int32 wrap-around."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402


def _requant_ref(y32: torch.Tensor, shift: int, relu: bool) -> torch.Tensor:
    h = y32.long()
    if relu:
        h = h.clamp(min=0)
    h = ((h + (1 << (shift - 1)) + (1 << 31)) % (1 << 32)) - (1 << 31)  # int32 wrap, as NumPy
    return torch.clamp(h >> shift, -128, 127).to(torch.int8)


def _ops(M, N, Kd, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randint(-128, 128, (M, Kd), generator=g, dtype=torch.int8).cuda()
    w = torch.randint(-128, 128, (N, Kd), generator=g, dtype=torch.int8).cuda()
    b = torch.randint(-2000, 2001, (N,), generator=g, dtype=torch.int32).cuda()
    ws, bs = K.offline_checksum(w, b, L.GG_P_I64)
    return x, w, b, ws, int(bs.item())


@pytest.mark.parametrize("shape", [(197, 768, 768), (1000, 300, 200), (4096, 3072, 768)])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("shift", [1, 9, 17])
def test_fused_requant_equals_int32_then_requant(shape, relu, shift):
    M, N, Kd = shape
    x, w, b, ws, bs = _ops(M, N, Kd, M + N + shift)
    act = L.GG_ACT_RELU if relu else L.GG_ACT_NONE
    y32, r32 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0)
    h, rh = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0, out_dtype=torch.int8,
                             requant_shift=shift, act=act)
    torch.cuda.synchronize()
    assert h.dtype == torch.int8
    assert torch.equal(h, _requant_ref(y32, shift, relu))
    assert torch.equal(rh.d, r32.d) and int(rh.nflag.item()) == 0  # the same exact check of y
    hu, _ = K.protected_gemm(x, w, b, protect=False, out_dtype=torch.int8, requant_shift=shift, act=act)
    assert torch.equal(hu, h)


def test_fused_requant_fault_detected_and_replayed():
    M, N, Kd = 2048, 768, 768
    x, w, b, ws, bs = _ops(M, N, Kd, 5)
    clean, _ = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0, out_dtype=torch.int8, requant_shift=9,
                                act=L.GG_ACT_RELU)
    rows = [3, 700, 2047]
    injs = [K.Injection(row=r, col=(5 * r) % N, bit=28) for r in rows]
    h, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0, out_dtype=torch.int8, requant_shift=9,
                              act=L.GG_ACT_RELU, injections=injs)
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == rows
    diff = int((h != clean).sum().item())  # the requantised bytes the faults moved
    changed = K.replay_tiles(x, w, b, h, res.flags.clone(), res, w_sum=ws, bias_sum=bs, lo=0, hi=0,
                             act=L.GG_ACT_RELU, requant_shift=9)
    torch.cuda.synchronize()
    assert torch.equal(h, clean)
    assert int(changed.item()) == diff and int(res.nflag.item()) == 0


def test_requant_argument_checks():
    x, w, b, ws, bs = _ops(64, 64, 64, 1)
    with pytest.raises(ValueError, match="requant shift"):
        K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, out_dtype=torch.int8, requant_shift=0)
    with pytest.raises(NotImplementedError, match="ReLU"):
        xb = x.to(torch.bfloat16)
        wb = w.to(torch.bfloat16)
        wsb, bsb = K.offline_checksum(wb, b.float(), L.GG_P_F64)
        K.protected_gemm(xb, wb, b.float(), w_sum=wsb, bias_sum=float(bsb.item()), act=L.GG_ACT_RELU)
