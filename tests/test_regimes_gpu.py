"""K1's fold regimes side by side: tiny launches (one launch-wide count, every row folded by
the last CTA), launches of at most two tiles per pair (split bands finished at the kernel end
by the completing CTA), contiguous ranges (whole bands folded locally, cut bands through the
workspace) and the strided long-K schedule.  In each: d equals a plain fp64 reference within
the fused-d bound (int8 exactly), repeated launches give identical d, faults in several bands
are flagged exactly and replay restores the clean bytes and the summary."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402

BOUND = 2.0**-19

SHAPES = {
    "tiny": (197, 2304, 768),          # 9 pair tiles, 2 bands
    "few_tiles": (9000, 3072, 256),    # 18 x 12 = 216 pair tiles: at most two per pair
    "contiguous": (20000, 1024, 512),  # ~8 tiles per pair, cut and whole bands
    "long_k": (8192, 768, 4096),       # strided schedule
}


def _ops(M, N, Kd, dtype, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    if dtype == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), generator=g, dtype=torch.int8)
        w = torch.randint(-128, 128, (N, Kd), generator=g, dtype=torch.int8)
        b = torch.randint(-64, 65, (N,), generator=g, dtype=torch.int32)
        prec = L.GG_P_I64
    else:
        x = torch.randn(M, Kd, generator=g).to(dtype)
        w = (torch.randn(N, Kd, generator=g) / Kd**0.5).to(dtype)
        b = (0.02 * torch.randn(N, generator=g)).float()
        prec = L.GG_P_F64
    x, w, b = x.cuda(), w.cuda(), b.cuda()
    ws, bs = K.offline_checksum(w, b, prec)
    return x, w, b, ws, bs.item()


@pytest.mark.parametrize("regime", sorted(SHAPES))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.int8])
def test_fold_regimes(regime, dtype):
    M, N, Kd = SHAPES[regime]
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, M + N)
    integer = dtype == torch.int8
    y, r = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    # d against fp64 over the same stored outputs
    pred = x.double() @ ws.double() + float(bs)
    obs = y.double().sum(dim=1)
    if integer:
        # exact in fp64 here (|x . w_sum| < 2^53); torch has no integer matmul on the device
        want = (x.double() @ ws.double()).round().long() + int(bs) - y.long().sum(dim=1)
        assert torch.equal(r.d, want)
    else:
        terms = (x.double().abs() @ ws.double().abs()) + y.double().abs().sum(dim=1) + abs(float(bs))
        assert bool(((r.d - (pred - obs)).abs() <= BOUND * terms).all())
    _, r2 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    assert torch.equal(r2.d.view(torch.int64), r.d.view(torch.int64))  # deterministic folds
    clean = y.clone()
    thr = 0.0 if integer else 4 * float(r.d.abs().max().item()) + 1e-6
    rows = sorted({0, M // 3, M // 2 + 1, M - 1})
    injs = [K.Injection(row=rr, col=(7 * rr) % N, bit=30 if integer else 14) for rr in rows]
    y3, r3 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr, injections=injs)
    torch.cuda.synchronize()
    assert torch.nonzero(r3.flags.cpu()).flatten().tolist() == rows
    assert int(r3.nflag.item()) == len(rows) and int(r3.triggered.item()) == 1
    changed = K.replay_tiles(x, w, b, y3, r3.flags.clone(), r3, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert int(changed.item()) == len(rows)
    assert torch.equal(y3.view(torch.uint8), clean.view(torch.uint8))
    assert int(r3.nflag.item()) == 0 and int(r3.triggered.item()) == 0
    assert torch.equal(r3.d.view(torch.int64), r.d.view(torch.int64))  # replayed d = the clean launch's
