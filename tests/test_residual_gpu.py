"""Fused residual update (epilogue_act GG_ACT_RESIDUAL): the stored output is round(residual + y)
of the checked GEMM output y -- bytes identical to the separate add, the check unchanged, faults
in y detected and replayed (the residual is read-only, so the replay reproduces the bytes)."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shape", [(197, 768, 768), (5000, 1000, 320), (50432, 768, 3072)])
def test_residual_epilogue_equals_separate_add(dtype, shape):
    M, N, Kd = shape
    g = torch.Generator(device="cuda").manual_seed(M + N)
    x = torch.randn(M, Kd, device="cuda", generator=g).to(dtype)
    w = (torch.randn(N, Kd, device="cuda", generator=g) / Kd**0.5).to(dtype)
    b = 0.02 * torch.randn(N, device="cuda", generator=g)
    h = torch.randn(M, N, device="cuda", generator=g).to(dtype)
    ws, bs = K.offline_checksum(w, b, L.GG_P_F64)
    y, r = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30)
    hy, rh = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-1e30, hi=1e30, residual=h)
    torch.cuda.synchronize()
    assert torch.equal(hy.view(torch.uint8), (h + y).view(torch.uint8))  # torch's add rounds the fp32 sum once
    assert torch.equal(rh.d.view(torch.int64), r.d.view(torch.int64))  # the check is on y
    hu, _ = K.protected_gemm(x, w, b, protect=False, residual=h)
    assert torch.equal(hu, hy)
    thr = 4 * float(r.d.abs().max().item()) + 1e-6
    rows = [0, M // 2, M - 1]
    injs = [K.Injection(row=rr, col=(3 * rr) % N, bit=14) for rr in rows]
    hf, rf = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs.item(), lo=-thr, hi=thr, residual=h, injections=injs)
    torch.cuda.synchronize()
    assert torch.nonzero(rf.flags.cpu()).flatten().tolist() == rows
    changed = K.replay_tiles(x, w, b, hf, rf.flags.clone(), rf, w_sum=ws, bias_sum=bs.item(), lo=-thr, hi=thr,
                             residual=h)
    torch.cuda.synchronize()
    assert torch.equal(hf, hy) and int(rf.nflag.item()) == 0
    assert int(changed.item()) >= 1


def test_residual_must_not_alias_the_output():
    x = torch.randn(64, 64, device="cuda").bfloat16()
    w = torch.randn(64, 64, device="cuda").bfloat16()
    y = torch.empty(64, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="alias"):
        K.protected_gemm(x, w, None, protect=False, out=y, residual=y)


def test_vit_with_fused_residual_equals_the_separate_adds():
    """ProtectedViT with proj / fc2 storing h + y (fused_residual) gives the same logits, checks and
    replay results as with the layer norms adding the residual."""
    from paper_2310_03841_b200.vit import ProtectedViT, ViTConfig

    cfg = ViTConfig(name="vit_s_test", dim=256, depth=2, heads=4, mlp=1024, classes=10)
    m = ProtectedViT(cfg, seed=5)
    g = torch.Generator(device="cuda").manual_seed(11)
    m.calibrate([torch.randn(8, 3, cfg.image, cfg.image, device="cuda", generator=g) for _ in range(2)],
                confidence=1 - 1e-9)
    imgs = torch.randn(8, 3, cfg.image, cfg.image, device="cuda", generator=g)
    assert m.fused_residual
    fused = m(imgs).clone()
    d_fused = {i: m.buffers(8).results[i].d.clone() for i in range(cfg.n_layers)}
    m.fused_residual = False
    m._bufs = {}
    plain = m(imgs).clone()
    assert torch.equal(fused.view(torch.uint8), plain.view(torch.uint8))
    for i in range(cfg.n_layers):
        assert torch.equal(m.buffers(8).results[i].d.view(torch.int64), d_fused[i].view(torch.int64))
    m.fused_residual = True
    m._bufs = {}
    clean = m(imgs).clone()
    layer = 8  # fc2 of block 1: residual fused
    inj = K.injections_to_device([K.Injection(row=3 * cfg.tokens + 7, col=11, bit=14)], torch.device("cuda"))
    m.enable_replay()
    fixed = m(imgs, injections={layer: inj}).clone()
    m.disable_replay()
    assert torch.equal(fixed, clean)
    assert m.replay_events == [(layer, "replay", 1)]
    # resume from a cached prefix reproduces the forward
    cache = {}
    m(imgs, cache=cache)
    for start in (2, 3, 4, 7, 8):
        assert torch.equal(m.resume(start, cache, 8, protect=True).view(torch.uint8), clean.view(torch.uint8))
