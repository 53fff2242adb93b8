"""3xTF32 segment orders on the tf32 tensor pipe (cfg1 inputs): row-sum error
of Y against fp64 for each order of the hi*hi / hi*lo / lo*hi segments."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200 import kernels as K  # noqa: E402
from tests.golden_io import cfg1_inputs  # noqa: E402

x, wt, bias = cfg1_inputs()
y64 = x.astype(np.float64) @ wt.astype(np.float64) + bias
w = np.ascontiguousarray(wt.T)


def split(a):
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000).astype(np.uint32).view(np.float32)
    return r, (a - r).astype(np.float32)


xh, xl = split(x)
wh, wl = split(w)
segs = {"hh": (xh, wh), "hl": (xh, wl), "lh": (xl, wh), "ll": (xl, wl)}
bd = torch.from_numpy(bias.astype(np.float32)).cuda()
for order in (["hh", "hl", "lh"], ["hl", "lh", "hh"], ["lh", "hl", "hh"], ["ll", "hl", "lh", "hh"]):
    A = np.concatenate([segs[s][0] for s in order], axis=1)
    B = np.concatenate([segs[s][1] for s in order], axis=1)
    y, _ = K.protected_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), bd, protect=False,
                            f32_mode="tf32")
    e = y.double().cpu().numpy() - y64
    print(f"{'+'.join(order):14s} rms {np.sqrt(np.mean(e**2)):.3e} row-sum err std {np.std(e.sum(1)):.3e}")
