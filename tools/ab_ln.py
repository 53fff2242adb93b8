"""The plain layer norm on a ViT-B b256 residual stream (50432 x 768 bf16, no residual add):
median of CUDA-event-timed launches and a hash of the output, per library ($GEMMGUARD_LIB)."""
import hashlib, os, statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200 import kernels as K
D = int(sys.argv[1]) if len(sys.argv) > 1 else 768
dt = {'bf16': torch.bfloat16, 'f16': torch.float16}[sys.argv[2] if len(sys.argv) > 2 else 'bf16']
g = torch.Generator(device='cuda').manual_seed(5)
h = torch.randn(50432, D, device='cuda', generator=g).to(dt)
ln = torch.empty_like(h)
gm = 1 + 0.1 * torch.randn(D, device='cuda', generator=g)
bt = 0.1 * torch.randn(D, device='cuda', generator=g)
for _ in range(5):
    K.add_layernorm(h, None, gm, bt, 1e-6, ln_out=ln)
ts = []
for _ in range(60):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); K.add_layernorm(h, None, gm, bt, 1e-6, ln_out=ln); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
us = statistics.median(ts)
ref = torch.nn.functional.layer_norm(h.float(), (D,), gm, bt, 1e-6)
print(os.environ.get('GEMMGUARD_LIB', 'default').split('/')[-1], D, dt, f"{us:.1f} us {2 * h.numel() * 2 / us / 1e3:.0f} GB/s",
      hashlib.sha256(ln.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:12], f"max|err| vs torch fp32 {(ln.float() - ref).abs().max().item():.3g}")
