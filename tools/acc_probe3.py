"""3xTF32 on the tf32 pipe with the K-blocks dealt over 2 / 4 accumulation chains (the tensor
core's fp32 accumulator truncates at every step; shorter chains shrink the bias): row-sum
error of Y against fp64 on cfg1's inputs, chains summed in fp32 round-to-nearest."""
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
A = np.concatenate([xh, xl, xh], axis=1)  # hi*lo, lo*hi, hi*hi (small terms first)
B = np.concatenate([wl, wh, wh], axis=1)
A = np.concatenate([A[:, 1024:2048], A[:, :1024], A[:, 2048:]], axis=1)
B = np.concatenate([B[:, 1024:2048], B[:, :1024], B[:, 2048:]], axis=1)
bd = torch.from_numpy(bias.astype(np.float32)).cuda()
zero = torch.zeros_like(bd)
BK = 32
nb = A.shape[1] // BK
for chains in (1, 2, 4):
    y = None
    for c in range(chains):
        cols = np.concatenate([np.arange(b * BK, (b + 1) * BK) for b in range(c, nb, chains)])
        yc, _ = K.protected_gemm(torch.from_numpy(np.ascontiguousarray(A[:, cols])).cuda(),
                                 torch.from_numpy(np.ascontiguousarray(B[:, cols])).cuda(), bd if c == 0 else zero,
                                 protect=False, f32_mode="tf32")
        y = yc if y is None else y + yc
    e = y.double().cpu().numpy() - y64
    print(f"chains {chains}: rms {np.sqrt(np.mean(e**2)):.3e} row-sum err std {np.std(e.sum(1)):.3e} "
          f"mean(err*sign y) {np.mean(e * np.sign(y64)):.3e}")
