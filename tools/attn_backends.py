"""SDPA backends for the ViT-B/16 b256 attention shape (B=256, H=12, T=197, hd=64, bf16)."""
import sys, torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel
B, H, T, hd = 256, 12, 197, 64
qkv = torch.randn(B, T, 3, H, hd, device='cuda', dtype=torch.bfloat16)
q, k, v = (qkv[:, :, j].transpose(1, 2) for j in range(3))
def bench(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
flops = 4 * B * H * T * T * hd
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    try:
        with sdpa_kernel(be):
            us = bench(lambda: F.scaled_dot_product_attention(q, k, v))
        print(f"{be}: {us:.1f} us  {flops / us / 1e6:.0f} TFLOP/s")
    except Exception as e:
        print(be, 'unavailable:', str(e)[:100])
try:
    from flash_attn import flash_attn_qkvpacked_func
    us = bench(lambda: flash_attn_qkvpacked_func(qkv))
    print(f"flash_attn package: {us:.1f} us {flops / us / 1e6:.0f} TFLOP/s")
except Exception as e:
    print('flash_attn package unavailable:', str(e)[:200])
try:
    import flashinfer
    print('flashinfer', flashinfer.__version__)
except Exception as e:
    print('flashinfer', str(e)[:100])
