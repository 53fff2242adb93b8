"""Probe of the tensor core's fp32 accumulation on 3xTF32 (cfg1 inputs):
error of Y against an fp64 GEMM, its correlation with sign(Y) (a truncating
accumulator leaves a bias toward zero), versus the reference's fp32 fold."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03841_b200 import kernels as K  # noqa: E402
from paper_2310_03841_b200.numerics import Matrix2D, Precision, gemm  # noqa: E402
from tests.golden_io import cfg1_inputs  # noqa: E402

x, wt, bias = cfg1_inputs()
y64 = x.astype(np.float64) @ wt.astype(np.float64) + bias
ref = gemm(Matrix2D(x, "binary32"), Matrix2D(wt, "binary32"), bias=bias, accum=Precision.BINARY32,
           engine="exact").widened()
xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(np.ascontiguousarray(wt.T)).cuda()
bd = torch.from_numpy(bias.astype(np.float32)).cuda()
for mode in ("3xtf32", "tf32"):
    y, _ = K.protected_gemm(xd, wd, bd, protect=False, f32_mode=mode)
    y = y.double().cpu().numpy()
    for name, a in ((mode, y), ("reference fp32 fold", ref)):
        e = a - y64
        rel_bias = float(np.mean(e * np.sign(y64)) / np.mean(np.abs(y64)))
        print(f"{name:22s} rms err {np.sqrt(np.mean(e**2)):.3e}  mean(err*sign(y))/mean|y| {rel_bias:+.3e}  "
              f"row-sum err std {np.std(e.sum(1)):.3e}")
# the same with K split in 4 chunks summed on the host (fewer accumulation steps per accumulator)
parts = []
for c in range(4):
    sl = slice(256 * c, 256 * (c + 1))
    yc, _ = K.protected_gemm(xd[:, sl].contiguous(), wd[:, sl].contiguous(), None, protect=False)
    parts.append(yc.double().cpu().numpy())
ys = sum(parts) + bias
e = ys - y64
print(f"3xtf32 4 K-chunks      rms err {np.sqrt(np.mean(e**2)):.3e}  row-sum err std {np.std(e.sum(1)):.3e}")
