"""ViT-B/16 b256 protected forward with the predicted sums of qkv / fc1 formed by the
layer norm (pred_in) vs by K1's checksum warps; CUDA graphs, alternating rounds."""
import statistics, sys, torch
sys.path.insert(0, '.')
from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT
m = ProtectedViT(VIT_B16, seed=1)
g = torch.Generator(device='cuda').manual_seed(3)
x = torch.randn(256, 3, 224, 224, device='cuda', generator=g).bfloat16()
m.calibrate([x], 1 - 1e-9)
def graph(flag, protect=True):
    m.producer_pred = flag
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): m(x, protect=protect)
    torch.cuda.synchronize(); gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s): m(x, protect=protect)
    return gr
gs = {"pred_in": graph(True), "in-kernel": graph(False), "unprotected": graph(False, False)}
def timed(gr, n=10):
    for _ in range(3): gr.replay()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): gr.replay()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
t = {k: [] for k in gs}
for r in range(6):
    for k in (list(gs) if r % 2 == 0 else list(gs)[::-1]): t[k].append(timed(gs[k]))
med = {k: statistics.median(v) for k, v in t.items()}
print({k: round(v, 3) for k, v in med.items()}, "overhead pred_in %.1f%% in-kernel %.1f%%" % (
    100 * (med["pred_in"] / med["unprotected"] - 1), 100 * (med["in-kernel"] / med["unprotected"] - 1)))
