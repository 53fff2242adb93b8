"""Where a ViT-L/16 fp16 campaign block's time goes: host sampling, the suffix forward's host
launches and its device time (no teacher filter; 24 blocks spread over the layers)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200.campaign import ViTCampaign  # noqa: E402
from paper_2310_03841_b200.vit import VIT_L16, ProtectedViT  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
cfg = VIT_L16
model = ProtectedViT(cfg, dtype=torch.float16, device=dev, seed=3)
g = torch.Generator(device=dev).manual_seed(7)
imgs = torch.randn(256, 3, cfg.image, cfg.image, device=dev, generator=g).half()
camp = ViTCampaign(model, imgs, seed=1)
torch.cuda.synchronize()
rows = []
for li in list(range(0, cfg.n_layers, 4)) * 2:
    ks = np.arange(0, 256, dtype=np.int64)
    t0 = time.perf_counter()
    y = camp._raw_output(li)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    elem, bit, mode_ix, value = camp._sample(li, ks, y)
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    inj = K.injections_to_device([K.Injection(row=int(i * camp.model.rows_per_image(li)), col=0, bit=3) for i in range(256)], dev)
    e0.record()
    model.resume(li, camp.cache, 256, protect=True, injections={li: inj})
    e1.record()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    rows.append((li, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, e0.elapsed_time(e1), (t4 - t2) * 1e3))
for r in rows[len(rows) // 2:]:
    print(f"layer {r[0]:3d}: raw out {r[1]:6.2f} ms  sample {r[2]:6.2f} ms  forward launch (host) {r[3]:6.2f} ms  "
          f"forward device {r[4]:6.2f} ms  forward wall {r[5]:6.2f} ms")
