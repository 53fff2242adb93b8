import statistics, torch
h = torch.randn(50432, 768, device='cuda').bfloat16(); o = torch.empty_like(h)
big = torch.empty(2 * 1024**3 // 2, dtype=torch.bfloat16, device='cuda'); big2 = torch.empty_like(big)
gm = torch.ones(768, device='cuda', dtype=torch.bfloat16); bt = torch.zeros(768, device='cuda', dtype=torch.bfloat16)
def t(fn, n=40):
    for _ in range(5): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)
us = t(lambda: o.copy_(h)); print(f"copy 77MB: {us:.1f} us {2*h.numel()*2/us/1e3:.0f} GB/s")
us = t(lambda: big2.copy_(big), 10); print(f"copy 2GB: {us:.1f} us {2*big.numel()*2/us/1e3:.0f} GB/s")
us = t(lambda: torch.nn.functional.layer_norm(h, (768,), gm, bt, 1e-6)); print(f"torch layer_norm bf16: {us:.1f} us {2*h.numel()*2/us/1e3:.0f} GB/s")
us = t(lambda: torch.add(h, 1.0, out=o)); print(f"torch add scalar: {us:.1f} us {2*h.numel()*2/us/1e3:.0f} GB/s")
