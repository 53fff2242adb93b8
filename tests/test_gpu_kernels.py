"""GPU tests of the tcgen05 protected GEMM (K1), replay (K4) and flips (K3)
against fp32/fp64 torch references computed from the same operands."""

import pytest
import torch

# Fused d for bf16/fp16 operands (worst case, u = 2^-24): w = fp32(w_sum) adds u per
# predicted term; each K-block is 4 fp32 FMA chains of 16 products plus a 4-way fp32
# sum (18u), folded exactly by TwoSum; observed sums are 4 fp32 chains of <= 32
# stored outputs per thread (32u), folded in fp64.  Hence
# |d_fused - d_fp64| <= 2^-24 (20 sum|x w_sum| + 32 sum|y|) <= 2^-19 sum|terms|.
# tf32 operands / fp32 outputs: fp32 FMA chains of 8 products and fp32 chains of 8
# outputs per 32-column chunk, folded by TwoSum: 2^-24 (10 sum|x w_sum| + 8 sum|y|).
FUSED_D_REL = 2.0**-19

pytestmark = pytest.mark.gpu

from paper_2310_03841_b200 import _lib as L
from paper_2310_03841_b200 import kernels as K


def _operands(M, N, Kd, dtype, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    if dtype == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), generator=g, dtype=torch.int8)
        w = torch.randint(-128, 128, (N, Kd), generator=g, dtype=torch.int8)
        b = torch.randint(-64, 65, (N,), generator=g, dtype=torch.int32)
    else:
        x = torch.randn(M, Kd, generator=g).to(dtype)
        w = (torch.randn(N, Kd, generator=g) / Kd**0.5).to(dtype)
        b = (0.02 * torch.randn(N, generator=g)).float()
    return x.cuda(), w.cuda(), b.cuda()


def _ref_y(x, w, b, out_dtype):
    if x.dtype == torch.int8:
        y = x.cpu().long() @ w.cpu().long().T + b.cpu().long()
        return y.to(torch.int32)
    y = x.double() @ w.double().T + b.double()
    return y


SHAPES = [(128, 256, 64), (300, 520, 200), (197, 768, 768), (1, 8, 16), (517, 1000, 3072)]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int8])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_matches_reference(dtype, shape):
    M, N, Kd = shape
    x, w, b = _operands(M, N, Kd, dtype)
    y, _ = K.protected_gemm(x, w, b, protect=False)
    torch.cuda.synchronize()
    ref = _ref_y(x, w, b, y.dtype)
    if dtype == torch.int8:
        assert torch.equal(y.cpu(), ref), "int8 GEMM must be bit-exact"
    else:
        # fp32 accumulation over K terms + output rounding
        scale = (x.double().abs() @ w.double().abs().T + b.double().abs()).cpu()
        u_out = {torch.bfloat16: 2.0**-8, torch.float16: 2.0**-11, torch.float32: 2.0**-24}[dtype]
        u_in = 2.0**-11 if dtype == torch.float32 else 0.0  # tf32 operands
        tol = scale * (Kd * 2.0**-23 + 2 * u_in) + ref.abs().cpu() * u_out
        err = (y.double().cpu() - ref.cpu()).abs()
        assert bool((err <= tol + 1e-30).all()), float((err - tol).max())


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int8])
@pytest.mark.parametrize("shape", SHAPES)
def test_protected_checksum_matches_fp64(dtype, shape):
    M, N, Kd = shape
    x, w, b = _operands(M, N, Kd, dtype, seed=1)
    integer = dtype == torch.int8
    prec = L.GG_P_I64 if integer else L.GG_P_F64
    w_sum, bsum = K.offline_checksum(w, b, prec)
    y0, _ = K.protected_gemm(x, w, b, protect=False)
    y, res = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.uint8) if y.dtype != torch.int32 else y, y0.view(torch.uint8) if y0.dtype != torch.int32 else y0)
    if integer:
        pred = x.cpu().long() @ w_sum.cpu() + int(bsum.item())
        obs = y.cpu().long().sum(1)
        bad = torch.nonzero(res.d.cpu() != pred - obs).flatten()
        assert bad.numel() == 0, (bad[:10].tolist(), res.d.cpu()[bad[:5]].tolist(), (pred - obs)[bad[:5]].tolist(),
                                  (x.cpu().long() @ w_sum.cpu())[bad[:5]].tolist(), obs[bad[:5]].tolist())
        assert int(res.nflag.item()) == int((pred != obs).sum())
    else:
        pred = x.double() @ w_sum + bsum.double()
        obs = y.double().sum(1)
        d_ref = (pred - obs).cpu()
        mag = ((x.double().abs() @ w_sum.abs()) + y.double().abs().sum(1)).cpu()
        rel = FUSED_D_REL
        err = (res.d.cpu() - d_ref).abs()
        assert bool((err <= mag * rel + 1e-300).all()), (float(err.max()), float((err / mag).max()))
        assert int(res.nflag.item()) == 0 and int(res.triggered.item()) == 0
        gap = (res.d.cpu()).abs().max().item()
        assert abs(res.max_disc.item() - gap) <= 1e-12 * max(gap, 1e-300)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int8])
def test_output_flip_is_detected_and_replayed(dtype):
    M, N, Kd = 300, 520, 256
    x, w, b = _operands(M, N, Kd, dtype, seed=2)
    integer = dtype == torch.int8
    prec = L.GG_P_I64 if integer else L.GG_P_F64
    w_sum, bsum = K.offline_checksum(w, b, prec)
    _, cal = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    thr = 0.0 if integer else 4.0 * float(cal.d.abs().max().item()) + 1e-12
    clean, res0 = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-thr, hi=thr)
    clean = clean.clone()
    torch.cuda.synchronize()
    assert int(res0.nflag.item()) == 0
    top = {torch.bfloat16: 14, torch.float16: 14, torch.float32: 30, torch.int8: 30}[dtype]
    inj = [K.Injection(row=257, col=300, bit=top), K.Injection(row=3, col=5, bit=top)]
    y, res = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-thr, hi=thr, injections=inj)
    torch.cuda.synchronize()
    flagged = torch.nonzero(res.flags.cpu()).flatten().tolist()
    assert flagged == [3, 257]
    assert int(res.nflag.item()) == 2 and int(res.triggered.item()) == 1
    changed = K.replay_tiles(x, w, b, y, res.flags, res, w_sum=w_sum, bias_sum=bsum.item(), lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert int(changed.item()) == 2
    assert torch.equal(y.cpu(), clean.cpu())
    assert int(res.nflag.item()) == 0 and int(res.triggered.item()) == 0


def test_accumulator_flip_detected_bf16():
    M, N, Kd = 256, 512, 128
    x, w, b = _operands(M, N, Kd, torch.bfloat16, seed=3)
    w_sum, bsum = K.offline_checksum(w, b, L.GG_P_F64)
    inj = [K.Injection(row=100, col=400, bit=30, target=L.GG_INJ_ACCUMULATOR)]
    y, res = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-0.5, hi=0.5, injections=inj)
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == [100]


def test_flip_bits_involution():
    t = torch.randn(1000, dtype=torch.float32, device="cuda")
    orig = t.clone()
    idx = torch.tensor([0, 5, 999], dtype=torch.int64, device="cuda")
    bits = torch.tensor([31, 3, 23], dtype=torch.int32, device="cuda")
    K.flip_bits(t, idx, bits)
    assert t[0].item() == -orig[0].item()
    assert not torch.equal(t, orig)
    K.flip_bits(t, idx, bits)
    assert torch.equal(t.view(torch.int32), orig.view(torch.int32))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int8])
@pytest.mark.parametrize("shape", [(50432, 768, 768), (50432, 768, 3072), (4096, 3072, 768), (1024, 3072, 768),
                                   (512, 8192, 256), (50432, 1024, 256), (50432, 2048, 256)])
def test_fused_check_is_deterministic_and_accurate_at_scale(dtype, shape):
    """Full-size launches (many tiles per CTA pair, split and local bands; contiguous,
    strided and one-tile schedules, and tf32's claimed folds in the first two):
    bit-identical d across launches, and d within the stated bound of the fp64
    discrepancy of the same outputs (a race in the stage hand-off shows up here)."""
    M, N, Kd = shape
    x, w, b = _operands(M, N, Kd, dtype, seed=5)
    integer = dtype == torch.int8
    w_sum, bsum = K.offline_checksum(w, b, L.GG_P_I64 if integer else L.GG_P_F64)
    y1, r1 = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-1e30, hi=1e30)
    d1 = r1.d.clone()
    y2, r2 = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=bsum.item(), lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(d1.view(torch.int64) if not integer else d1, r2.d.view(torch.int64) if not integer else r2.d)
    if integer:
        ref = (x.cpu().long() @ w_sum.cpu() + int(bsum.item())) - y1.cpu().long().sum(1)  # int64 matmul: CPU
        assert torch.equal(d1.cpu(), ref)
    else:
        ref = (x.double() @ w_sum + bsum.double()) - y1.double().sum(1)
        mag = (x.double().abs() @ w_sum.abs()) + y1.double().abs().sum(1)
        assert bool(((d1 - ref).abs() <= mag * FUSED_D_REL + 1e-300).all())
