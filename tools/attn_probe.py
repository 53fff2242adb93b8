"""Attention libraries on the ViT-B/16 b256 shape (B=256, H=12, T=197, hd=64, bf16, non-causal):
torch SDPA (cuDNN), flash_attn, flashinfer's cuDNN / trtllm-gen paths where they load without JIT."""
import time, traceback, torch
import torch.nn.functional as F
B, H, T, hd = 256, 12, 197, 64
dev = 'cuda'
qkv = torch.randn(B, T, 3, H, hd, device=dev, dtype=torch.bfloat16)
q, k, v = (qkv[:, :, j] for j in range(3))  # [B, T, H, hd]
flops = 4 * B * H * T * T * hd
ref = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2)).transpose(1, 2)

def bench(name, fn, n=30):
    try:
        t0 = time.time(); out = fn(); torch.cuda.synchronize(); first = time.time() - t0
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        err = (out.float() - ref.float()).abs().max().item() if out is not None and out.shape == ref.shape else float('nan')
        print(f"{name:40s} {us:8.1f} us  {flops/us/1e6:7.1f} TF/s  max|err| {err:.3g}  first call {first:.1f}s", flush=True)
    except Exception as e:
        print(f"{name:40s} FAILED: {type(e).__name__}: {str(e)[:200]}", flush=True)

bench("torch sdpa (default)", lambda: F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2)).transpose(1, 2))
try:
    from flash_attn import flash_attn_func
    bench("flash_attn 2 flash_attn_func", lambda: flash_attn_func(q, k, v))
except Exception as e:
    print("flash_attn import failed", e)
try:
    import flashinfer
    qf, kf, vf = q.reshape(B * T, H, hd), k.reshape(B * T, H, hd), v.reshape(B * T, H, hd)
    indptr = torch.arange(0, (B + 1) * T, T, device=dev, dtype=torch.int32)
    for backend in ("cutlass", "fa2", "trtllm-gen", "cudnn"):
        try:
            ws = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
            w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=backend)
            w.plan(indptr, indptr, H, H, hd, causal=False, q_data_type=torch.bfloat16)
            bench(f"flashinfer ragged prefill [{backend}]", lambda: w.run(qf, kf, vf).reshape(B, T, H, hd))
        except Exception as e:
            print(f"flashinfer [{backend}] FAILED: {type(e).__name__}: {str(e)[:300]}", flush=True)
except Exception:
    traceback.print_exc()
