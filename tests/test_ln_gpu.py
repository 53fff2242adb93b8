"""The persistent layer norm (gg_add_layernorm without a residual add at D = 768 / 1024, the ViT-B / ViT-L widths)
against the one-pass kernel it replaces: adding a zero residual routes the same rows through
add_layernorm_kernel, whose sums are the same in the same order, so the normalised rows and the
consumer's predicted sums must be bit-identical; plus torch fp32 within bf16 / fp16 rounding, and
ragged row counts (fewer rows than one block, not a multiple of the grid's warps)."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import kernels as K  # noqa: E402


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("rows", [1, 7, 1001, 50432])
@pytest.mark.parametrize("pred", [False, True])
@pytest.mark.parametrize("D", [768, 1024])
def test_stream_layernorm_matches_the_one_pass_kernel(dtype, rows, pred, D):
    g = torch.Generator(device="cuda").manual_seed(rows + 3 * pred)
    h = (2.0 * torch.randn(rows, D, device="cuda", generator=g) + 0.5).to(dtype)
    gm = 1.0 + 0.1 * torch.randn(D, device="cuda", generator=g)
    bt = 0.1 * torch.randn(D, device="cuda", generator=g)
    w = torch.randn(D, device="cuda", generator=g) if pred else None
    a1 = torch.empty_like(h)
    p1 = torch.empty(rows, dtype=torch.int64, device="cuda") if pred else None
    K.add_layernorm(h, None, gm, bt, 1e-6, ln_out=a1, w_pred=w, pred_out=p1)  # persistent kernel
    a2, h2 = torch.empty_like(h), torch.empty_like(h)
    p2 = torch.empty(rows, dtype=torch.int64, device="cuda") if pred else None
    K.add_layernorm(h, torch.zeros_like(h), gm, bt, 1e-6, ln_out=a2, h_out=h2, w_pred=w, pred_out=p2)
    torch.cuda.synchronize()
    assert torch.equal(h2, h)
    assert torch.equal(a1.view(torch.int16), a2.view(torch.int16))
    if pred:
        assert torch.equal(p1, p2)
        # the predicted sum is fp32 bits of sum(stored a * w): check against fp64 over the same bytes
        got = torch.tensor(p1.cpu().numpy().astype("uint32").view("float32"), dtype=torch.float64)
        want = (a1.double() @ w.double()).cpu()
        bound = (a1.double().abs() @ w.double().abs()).cpu() * (D / 32 + 5) * 2.0**-24
        assert bool(((got - want).abs() <= bound).all())
    ref = torch.nn.functional.layer_norm(h.float(), (D,), gm, bt, 1e-6)
    ulp = 2.0**-7 if dtype == torch.bfloat16 else 2.0**-10
    assert bool(((a1.float() - ref).abs() <= ulp * ref.abs() + 1e-3).all())


def test_layernorm_output_must_not_alias_its_input():
    h = torch.randn(16, 768, device="cuda").to(torch.bfloat16)
    gm, bt = torch.ones(768, device="cuda"), torch.zeros(768, device="cuda")
    with pytest.raises(ValueError, match="alias"):
        K.add_layernorm(h, None, gm, bt, 1e-6, ln_out=h)
    with pytest.raises(ValueError, match="alias"):
        K.add_layernorm(h, torch.zeros_like(h), gm, bt, 1e-6, ln_out=h, h_out=h)
