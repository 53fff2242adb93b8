"""Protected Swin (int8 MLP + bf16 attention projections) on the B200.

Against a plain-PyTorch fp32 forward of the same parameters and the same
int8 quantisation (loose: bf16 storage and int8 rounding boundaries); the
int8 layers' exact check flags every output fault; detect-then-replay
restores the clean logits bit for bit."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.nn.functional as F  # noqa: E402

from paper_2310_03841_b200 import kernels as K  # noqa: E402
from paper_2310_03841_b200.swin import SWIN_B, ProtectedSwin, SwinConfig  # noqa: E402

TINY = SwinConfig(name="swin_tiny_test", embed=32, depths=(2, 2, 2, 2), heads=(1, 2, 4, 8), classes=10)


def _imgs(B, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(B, 3, 224, 224, device="cuda", generator=g)


def _reference(m: ProtectedSwin, images):
    """fp32 torch forward: same weights, same fake-quantisation of the int8 layers."""
    c0 = m.cfg
    B, P, r0 = images.shape[0], c0.patch, c0.image // c0.patch

    def ln(x, j, d):
        return F.layer_norm(x, (d,), m.ln_g[j, :d], m.ln_b[j, :d], c0.ln_eps)

    def lin(pl, x):
        q = m.quant.get(pl.index)
        if q is None:
            return x @ pl.weight.float().T + pl.bias
        xq = torch.clamp(torch.round(x / q.s_x), -127, 127)
        return (xq.double() @ pl.weight.double().T + pl.bias.double()).float() * (q.s_x * q.s_w)

    x = images.float().view(B, 3, r0, P, r0, P).permute(0, 2, 4, 1, 3, 5).reshape(B * r0 * r0, -1)
    h = ln(lin(m.embed, x.to(torch.bfloat16).float()), 0, c0.embed)
    for s, ((r, c), stage) in enumerate(zip(c0.stage_dims(), m.blocks)):
        for blk in stage:
            a = ln(h, blk["ln1"], c)
            qkv = lin(blk["qkv"], a)
            o = m._attention(qkv.to(torch.bfloat16), B, r, c, blk["heads"], blk["shift"], blk["bias"]).float()
            h = h + lin(blk["proj"], o)
            f = F.gelu(lin(blk["fc1"], ln(h, blk["ln2"], c)), approximate="tanh")
            h = h + lin(blk["fc2"], f)
        if s < len(m.merges):
            mg = m.merges[s]
            v = h.view(B, r, r, c)
            cat = torch.cat([v[:, 0::2, 0::2], v[:, 1::2, 0::2], v[:, 0::2, 1::2], v[:, 1::2, 1::2]], dim=-1)
            h = lin(mg["lin"], ln(cat.reshape(-1, 4 * c), mg["ln"], 4 * c))
    r, c = c0.stage_dims()[-1]
    hf = ln(h, m.final_ln, c).view(B, r * r, c).mean(dim=1)
    return lin(m.head, hf)


def test_swin_gemm_inventory():
    g = SWIN_B.gemms(1)
    assert len(g) == 101
    assert sum(1 for x in g if x[4] == "int8") == 48


def test_swin_forward_matches_plain_torch():
    m = ProtectedSwin(TINY, seed=1)
    imgs = _imgs(4, 2)
    got = m(imgs).float()
    want = _reference(m, imgs)
    cos = F.cosine_similarity(got.flatten(), want.flatten(), dim=0)
    assert float(cos) > 0.99, float(cos)
    assert m.flagged_rows() == {}  # int8 exact checks clean; bf16 thresholds not calibrated yet


def test_swin_int8_faults_detected_exactly_and_replayed():
    m = ProtectedSwin(TINY, seed=3)
    m.calibrate([_imgs(8, s) for s in (4, 5, 7, 8)], 1 - 1e-9)  # >= 30 samples for the 1-row-per-image head
    imgs = _imgs(4, 6)
    clean = m(imgs).clone()
    # per-layer scalar epsilon (guard.EpsilonModel) on a few calibration images: at most a stray
    # false flag in a bf16 layer; the int8 layers' exact checks are silent
    false = m.flagged_rows()
    assert sum(false.values()) <= 2 and not any(m.linears[i].integer for i in false)
    fc1 = m.blocks[1][0]["fc1"]
    assert fc1.integer
    for bit in (0, 5, 17, 30):  # any flipped bit of an int32 output changes its row sum: exact detection
        inj = K.injections_to_device([K.Injection(row=100, col=3, bit=bit)], torch.device("cuda"))
        m(imgs, injections={fc1.index: inj})
        res = fc1.result
        assert bool(res.triggered.item()) and res.flags.nonzero().flatten().tolist() == [100]
    m.enable_replay(layers=[fc1.index])
    fixed = m(imgs, injections={fc1.index: inj}).clone()
    m.disable_replay()
    assert torch.equal(fixed, clean)
    assert m.replay_events == [(fc1.index, "replay", 1)]
