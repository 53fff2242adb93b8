"""gg_embed_layernorm: the ViT embedding's position add, class token and first layer norm in
one pass -- the residual stream bit-identical to torch's adds, the normalised rows identical
to gg_add_layernorm on that stream (and its predicted sums)."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import kernels as K  # noqa: E402


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("B,T,D", [(3, 197, 768), (2, 50, 1024), (1, 2, 256)])
def test_embed_layernorm_matches_torch_adds_then_layernorm(dtype, B, T, D):
    g = torch.Generator(device="cuda").manual_seed(B * T + D)
    e = torch.randn(B * (T - 1), D, device="cuda", generator=g).to(dtype)
    pos = (0.02 * torch.randn(T, D, device="cuda", generator=g)).to(dtype)
    cls = (0.02 * torch.randn(D, device="cuda", generator=g)).to(dtype)
    gamma = 1 + 0.1 * torch.randn(D, device="cuda", generator=g)
    beta = 0.1 * torch.randn(D, device="cuda", generator=g)
    w = torch.randn(D, device="cuda", generator=g)
    h = torch.empty(B * T, D, dtype=dtype, device="cuda")
    a = torch.empty_like(h)
    pred = torch.empty(B * T, dtype=torch.int64, device="cuda")
    K.embed_layernorm(e, pos, cls, gamma, beta, 1e-6, h_out=h, ln_out=a, w_pred=w, pred_out=pred)
    want = torch.empty_like(h)
    wv = want.view(B, T, D)
    torch.add(e.view(B, T - 1, D), pos[1:], out=wv[:, 1:])
    wv[:, 0] = cls + pos[0]
    assert torch.equal(h.view(torch.uint8), want.view(torch.uint8))
    a2 = torch.empty_like(h)
    pred2 = torch.empty_like(pred)
    K.add_layernorm(want, None, gamma, beta, 1e-6, ln_out=a2, w_pred=w, pred_out=pred2)
    assert torch.equal(a.view(torch.uint8), a2.view(torch.uint8))
    assert torch.equal(pred, pred2)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("B,H,P", [(2, 224, 16), (3, 64, 8), (1, 32, 32)])
def test_patchify_matches_the_permuted_copy(dtype, B, H, P):
    if (P * torch.tensor([], dtype=dtype).element_size()) % 16:
        pytest.skip("16-byte pieces")
    g = torch.Generator(device="cuda").manual_seed(B * H + P)
    img = torch.randn(B, 3, H, H, device="cuda", generator=g).to(dtype)
    G = H // P
    out = torch.empty(B * G * G, 3 * P * P, dtype=dtype, device="cuda")
    K.patchify(img, P, out)
    want = img.view(B, 3, G, P, G, P).permute(0, 2, 4, 1, 3, 5).reshape(B * G * G, 3 * P * P)
    assert torch.equal(out, want)
