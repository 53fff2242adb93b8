"""ViT-B/16 b256 bf16 protected forward graphs with the layer norms forming qkv / fc1's predicted
sums (producer_pred) vs K1's own predicted side, plus the unprotected forward, alternating rounds
on one box."""
import statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT  # noqa: E402
m = ProtectedViT(VIT_B16, seed=1)
g = torch.Generator(device="cuda").manual_seed(2)
x = torch.randn(256, 3, 224, 224, device="cuda", generator=g).to(torch.bfloat16)
graphs = {}
for fr, prot in ((True, True), (False, True), (False, False)):
    if True:
        m.producer_pred = fr
        m._bufs = {}
        s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                m(x, protect=prot)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            m(x, protect=prot)
        graphs[(fr, prot)] = (gr, m._bufs)
t = {k: [] for k in graphs}
for r in range(8):
    for k in (list(graphs) if r % 2 == 0 else list(reversed(list(graphs)))):
        gr = graphs[k][0]
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            gr.replay()
        e1.record(); torch.cuda.synchronize()
        t[k].append(e0.elapsed_time(e1) / 10)
for k, v in t.items():
    ms = statistics.median(v)
    print(f"producer_pred={k[0]!s:5s} protect={k[1]!s:5s} {ms:7.3f} ms  {256 / ms * 1e3:8.0f} img/s")
