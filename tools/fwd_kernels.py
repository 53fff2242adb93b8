"""One ViT-B/16 b256 protected forward (eager, after a warm-up) for a kernel listing under ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200.vit import VIT_B16, ProtectedViT  # noqa: E402

m = ProtectedViT(VIT_B16, seed=1)
g = torch.Generator(device="cuda").manual_seed(2)
x = torch.randn(256, 3, 224, 224, device="cuda", generator=g).to(torch.bfloat16)
m(x)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("fwd")
m(x)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
