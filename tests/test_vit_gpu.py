"""ProtectedLinear / ProtectedViT / the batched campaign engine on the B200.

Numerics bars: the model against a plain-PyTorch fp32 forward of the same
parameters (bf16 storage between layers: logits within a few percent of their
spread); fused GELU within one output ulp of GELU applied to the checked
output; the fused add + layer norm against torch within bf16 rounding;
resume / replay / batched campaigns bit-identical to the plain forward."""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.nn.functional as F  # noqa: E402

from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402
from paper_2310_03841_b200.campaign import FIELDS, ViTCampaign  # noqa: E402
from paper_2310_03841_b200.vit import VIT_B16, ProtectedLinear, ProtectedViT, ViTConfig  # noqa: E402

SMALL = ViTConfig(name="vit_s_test", dim=256, depth=2, heads=4, mlp=1024, classes=10)


def _images(B, cfg=VIT_B16, seed=0, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(B, 3, cfg.image, cfg.image, device="cuda", generator=g).to(dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("D", [256, 768, 1024])
def test_add_layernorm_matches_torch(dtype, D):
    g = torch.Generator(device="cuda").manual_seed(1)
    rows = 1000
    h = torch.randn(rows, D, device="cuda", generator=g).to(dtype)
    y = torch.randn(rows, D, device="cuda", generator=g).to(dtype)
    gam = 1 + 0.1 * torch.randn(D, device="cuda", generator=g)
    bet = 0.1 * torch.randn(D, device="cuda", generator=g)
    ln = torch.empty_like(h)
    hn = h.clone()
    K.add_layernorm(hn, y, gam, bet, 1e-6, ln_out=ln, h_out=hn)
    want_h = (h.float() + y.float()).to(dtype)
    assert torch.equal(hn, want_h)
    want = F.layer_norm(want_h.float(), (D,), gam, bet, 1e-6)
    tol = {torch.bfloat16: 2**-7, torch.float16: 2**-10, torch.float32: 1e-5}[dtype]
    assert torch.allclose(ln.float(), want, atol=tol * 4, rtol=tol * 2)
    ln2 = torch.empty_like(h)
    K.add_layernorm(h, None, gam, bet, 1e-6, ln_out=ln2)
    assert torch.allclose(ln2.float(), F.layer_norm(h.float(), (D,), gam, bet, 1e-6), atol=tol * 4, rtol=tol * 2)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_fused_gelu_is_gelu_of_the_checked_output(dtype):
    """The check covers the raw GEMM output (d identical with and without the
    activation); the stored value is tanh-GELU of it, within one output ulp
    plus the MUFU tanh's absolute error (<= 2^-10.9) scaled by 0.5 |x|."""
    g = torch.Generator(device="cuda").manual_seed(2)
    lin = ProtectedLinear(0, "fc1", 768, 3072, dtype=dtype, device="cuda", generator=g, act=L.GG_ACT_GELU_TANH)
    x = torch.randn(50432 // 8, 768, device="cuda", generator=g).to(dtype)
    y_act = lin(x).clone()
    r_act = lin.result
    lin.act = L.GG_ACT_NONE
    y_raw = lin(x).clone()
    r_raw = lin.result
    assert torch.equal(r_act.d, r_raw.d) and torch.equal(r_act.flags, r_raw.flags)
    want = F.gelu(y_raw.float(), approximate="tanh")
    ulp = {torch.bfloat16: 2**-7, torch.float16: 2**-10}[dtype]
    err = (y_act.float() - want).abs()
    tanh_err = 0.5 * y_raw.float().abs() * 2.0**-10.9
    assert bool((err <= ulp * want.abs() + tanh_err + 1e-3 * ulp).all()), float(err.max())


def _torch_reference(model, images):
    """Plain PyTorch fp32 forward of the same parameters."""
    c = model.cfg
    B, P, G, D = images.shape[0], c.patch, c.grid, c.dim
    x = images.float().view(B, 3, G, P, G, P).permute(0, 2, 4, 1, 3, 5).reshape(B * G * G, -1)

    def lin(i, t):
        ly = model.layer(i)
        return t @ ly.weight.float().T + ly.bias

    def ln(j, t):
        return F.layer_norm(t, (D,), model.ln_g[j], model.ln_b[j], c.ln_eps)

    e = lin(0, x).view(B, G * G, D)
    h = torch.cat([(model.cls.float() + model.pos[0].float()).expand(B, 1, D), e + model.pos[1:].float()], dim=1)
    H, hd = c.heads, D // c.heads
    for b in range(c.depth):
        base = 1 + 4 * b
        a = ln(2 * b, h).reshape(B * c.tokens, D)
        qkv = lin(base, a).view(B, c.tokens, 3, H, hd)
        q, k, v = (qkv[:, :, j].transpose(1, 2) for j in range(3))
        o = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B * c.tokens, D)
        h = h + lin(base + 1, o).view(B, c.tokens, D)
        a = ln(2 * b + 1, h).reshape(B * c.tokens, D)
        f = F.gelu(lin(base + 2, a), approximate="tanh")
        h = h + lin(base + 3, f).view(B, c.tokens, D)
    a = ln(2 * c.depth, h)
    return lin(c.n_layers - 1, a[:, 0])


def test_vit_b16_forward_matches_a_plain_torch_forward():
    model = ProtectedViT(VIT_B16, seed=3)
    imgs = _images(4)
    got = model(imgs).float()
    want = _torch_reference(model, imgs)
    spread = float(want.std())
    assert float((got - want).abs().max()) <= 0.05 * spread + 1e-3, (float((got - want).abs().max()), spread)
    cos = F.cosine_similarity(got.flatten(), want.flatten(), dim=0)
    assert float(cos) > 0.999
    # every protected layer ran its check, nothing flagged (thresholds not calibrated: +-inf)
    assert int(model.flagged_rows(4).sum()) == 0
    assert len(model.linears) == 50


def test_resume_reproduces_the_forward_bit_for_bit():
    model = ProtectedViT(SMALL, seed=4)
    imgs = _images(3, SMALL)
    cache = {}
    full = model(imgs, cache=cache).clone()
    for start in range(SMALL.n_layers):
        again = model.resume(start, cache, 3)
        assert torch.equal(again, full), start


def test_calibrated_vit_flags_faults_and_replay_restores_the_clean_logits():
    model = ProtectedViT(SMALL, seed=5)
    cal = [_images(8, SMALL, seed=s) for s in (10, 11, 12)]
    eps = model.calibrate(cal, confidence=1 - 1e-9)
    assert len(eps) == SMALL.n_layers
    imgs = _images(8, SMALL, seed=13)
    clean = model(imgs).clone()
    assert int(model.flagged_rows(8).sum()) == 0  # held-out clean batch: no false flag at c = 1 - 1e-9
    # a large output fault in fc1 of block 1 (layer 7), row 5 of image 2: bit 14 = exponent MSB of bf16
    layer, row = 7, 2 * SMALL.tokens + 5
    inj = K.injections_to_device([K.Injection(row=row, col=17, bit=14)], torch.device("cuda"))
    bad = model(imgs, injections={layer: inj}).clone()
    res = model.buffers(8).results[layer]
    assert int(res.nflag.item()) >= 1 and bool(res.flags[row].item())
    model.enable_replay()
    fixed = model(imgs, injections={layer: inj}).clone()
    model.disable_replay()
    assert torch.equal(fixed, clean)
    assert model.replay_events == [(layer, "replay", 1)]
    del bad  # (GELU of a huge negative value is 0: this flip need not change the logits)


@pytest.mark.parametrize("modes", [("fp_exponent_bit", "fp_mantissa_bit"), ("random_value",)])
def test_campaign_batched_trials_equal_single_trial_forwards(modes):
    """One trial per image: each image's outcome equals a forward carrying only its own fault."""
    model = ProtectedViT(SMALL, seed=6)
    model.calibrate([_images(8, SMALL, seed=s) for s in (20, 21)], confidence=1 - 1e-9)
    imgs = _images(8, SMALL, seed=22)
    camp = ViTCampaign(model, imgs, seed=7, keep_records=True, modes=modes)
    counters = torch.zeros((SMALL.n_layers, len(FIELDS)), dtype=torch.int64, device="cuda")
    for layer in (0, 3, 5, SMALL.n_layers - 1):
        rec = camp.run_block(layer, 0, counters)
        rows = model.rows_per_image(layer)
        for i in range(8):
            if rec["element"][i] < 0:
                continue
            N = model.layer(layer).out_features
            r, c = i * rows + rec["element"][i] // N, rec["element"][i] % N
            f = (K.Injection(row=int(r), col=int(c), bit=int(rec["bit"][i])) if rec["bit"][i] >= 0 else
                 K.Injection(row=int(r), col=int(c), mode=L.GG_INJ_SET_VALUE, value=float(rec["value"][i])))
            inj = K.injections_to_device([f], torch.device("cuda"))
            logits = model.resume(layer, camp.cache, 8, injections={layer: inj})
            mism = bool(logits[i].float().argmax() != camp.clean_pred[i])
            res = model.buffers(8).results[layer]
            det = bool(res.flags.view(8, rows)[i].any())
            assert mism == bool(rec["mismatch"][i]) and det == bool(rec["detected"][i]), (layer, i)
    c = counters.cpu().numpy()
    for layer in (0, 3, 5, SMALL.n_layers - 1):
        inj, mm, tp, fn, ben, tn, sk, _loss = c[layer]
        assert inj + sk == 8 and tp + fn == mm and tp + fn + ben + tn == inj


def test_campaign_sampler_follows_the_reference_rules():
    """Elements / bits are in range, flips are never no-ops and stay inside the layer's clean range."""
    model = ProtectedViT(SMALL, seed=8)
    imgs = _images(4, SMALL, seed=30)
    camp = ViTCampaign(model, imgs, seed=9)
    for layer in (1, 4, 9):
        y = camp._raw_output(layer)
        ks = np.arange(4)
        elem, bit, mode, _ = camp._sample(layer, ks, y)
        lo, hi = camp.ranges[layer]
        rows = model.rows_per_image(layer)
        N = y.shape[1]
        for i, (e, b) in enumerate(zip(elem, bit)):
            assert 0 <= e < rows * N and 0 <= b < 15
            v = y[i * rows + e // N, e % N].view(torch.int16).item() & 0xFFFF
            f = torch.tensor([(v ^ (1 << int(b))) - (65536 if (v ^ (1 << int(b))) >= 32768 else 0)],
                             dtype=torch.int16).view(torch.bfloat16).float().item()
            o = y[i * rows + e // N, e % N].float().item()
            assert f != o and lo <= f <= hi
        # the same (seed, layer, k) draws the same trial
        e2, b2, _, _ = camp._sample(layer, ks, y)
        assert np.array_equal(elem, e2) and np.array_equal(bit, b2)


def test_layernorm_supplied_predicted_sums_match_the_kernels_own():
    """pred_in from gg_add_layernorm (over the stored LN output) gives the same d as K1's own
    predicted side within the fused-d bound, and the same flags at a calibrated epsilon."""
    model = ProtectedViT(SMALL, seed=9)
    cal = [_images(8, SMALL, seed=s) for s in (40, 41)]
    model.calibrate(cal, confidence=0.9999)
    imgs = _images(8, SMALL, seed=42)
    ds = {}
    for flag in (True, False):
        model.producer_pred = flag  # off by default (a wash on ViT-B), must stay correct
        logits = model(imgs).clone()
        ds[flag] = ({i: model.buffers(8).results[i].d.clone() for i in range(SMALL.n_layers)},
                    {i: model.buffers(8).results[i].flags.clone() for i in range(SMALL.n_layers)}, logits)
    assert torch.equal(ds[True][2], ds[False][2])  # the GEMM outputs do not depend on it
    for i in range(SMALL.n_layers):
        a, b = ds[True][0][i], ds[False][0][i]
        scale = a.abs().max().item() + 1.0
        assert float((a - b).abs().max()) <= 2.0**-16 * scale * SMALL.mlp, i
        assert torch.equal(ds[True][1][i], ds[False][1][i]), i
