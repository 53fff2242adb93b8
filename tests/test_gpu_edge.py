"""GPU edge cases of the protected GEMM's epilogue and replay machinery:
campaign-style launches with many unsorted injections (including repeated
flips of one element), tiny and ragged shapes with faults in partial column
chunks, replay with nothing flagged, and replay under the strided (long-K)
schedule at full scale."""

import numpy as np
import pytest
import torch

from paper_2310_03841_b200 import _lib as L
from paper_2310_03841_b200 import kernels as K

pytestmark = pytest.mark.gpu


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


def _flip(y, r, c, bit):
    v = y.view(torch.int16 if y.element_size() == 2 else torch.int32)
    v[r, c] ^= (1 << bit) if bit < 8 * y.element_size() - 1 else -(1 << bit)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.int8])
def test_many_unsorted_injections_with_repeats(dtype):
    M, N, Kd = 2048, 768, 256
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, 11)
    clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    thr = 0.0 if dtype == torch.int8 else 4 * float(r0.d.abs().max().item())
    rng = np.random.default_rng(5)
    rows = rng.choice(M, 300, replace=False)
    injs = [K.Injection(row=int(r), col=int(rng.integers(0, N)), bit=int(rng.integers(8, 14))) for r in rows]
    injs += [K.Injection(row=injs[i].row, col=injs[i].col, bit=injs[i].bit) for i in range(0, 60)]  # cancel 60
    order = rng.permutation(len(injs))
    injs = [injs[i] for i in order]
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr, injections=injs)
    want = clean.clone()
    odd = {}
    for f in injs:
        key = (f.row, f.col, f.bit)
        odd[key] = not odd.get(key, False)
    for (r, c, bit), on in odd.items():
        if on:
            _flip(want, r, c, bit)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.uint8), want.view(torch.uint8))
    flagged = set(torch.nonzero(res.flags.cpu()).flatten().tolist())
    faulted = {r for (r, _, _), on in odd.items() if on}
    assert flagged <= faulted  # no clean row flags
    delta = (want.double() - clean.double()).abs().sum(dim=1).cpu()
    must = {r for r in faulted if delta[r] > 2 * thr}  # exact for int8 (thr = 0): every fault
    assert must <= flagged
    assert must == faulted if dtype == torch.int8 else len(must) >= 20


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.int8])
@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 33, 7), (129, 257, 65), (300, 40, 1000)])
def test_tiny_and_ragged_shapes_with_partial_chunk_fault(dtype, shape):
    M, N, Kd = shape
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, sum(shape))
    clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    integer = dtype == torch.int8
    thr = 0.0 if integer else 4 * float(r0.d.abs().max().item()) + 1e-6
    r, c = M - 1, N - 1  # last row, last column: the partial chunk / band
    top = {torch.bfloat16: 14, torch.float16: 14, torch.float32: 30, torch.int8: 30}[dtype]
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr,
                              injections=[K.Injection(row=r, col=c, bit=top)])
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == [r]
    changed = K.replay_tiles(x, w, b, y, res.flags, res, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert int(changed.item()) == 1
    assert torch.equal(y.view(torch.uint8), clean.view(torch.uint8))
    assert int(res.nflag.item()) == 0 and int(res.triggered.item()) == 0


def test_replay_with_nothing_flagged_keeps_outputs_and_summary():
    M, N, Kd = 1024, 512, 256
    x, w, b, ws, bs = _ops(M, N, Kd, torch.bfloat16, 3)
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    before = y.clone()
    md = float(res.max_disc.item())
    changed = K.replay_tiles(x, w, b, y, torch.zeros(M, dtype=torch.uint8, device="cuda"), res, w_sum=ws,
                             bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    assert int(changed.item()) == 0
    assert torch.equal(y, before)
    assert int(res.nflag.item()) == 0 and int(res.triggered.item()) == 0
    assert float(res.max_disc.item()) == md


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.int8])
def test_replay_under_strided_schedule_at_scale(dtype):
    """M = 50432, K = 3072: the long-K shape walks tiles strided and every band
    folds through the workspace; faults in three bands are detected, replayed,
    and the result equals the clean launch byte for byte."""
    M, N, Kd = 50432, 768, 3072
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, 9)
    clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    integer = dtype == torch.int8
    thr = 0.0 if integer else 4 * float(r0.d.abs().max().item())
    top = 14 if dtype == torch.bfloat16 else 30
    rows = [5, 25000, M - 1]
    if dtype == torch.float32:
        _, r1 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
        torch.cuda.synchronize()
        assert torch.equal(r1.d.view(torch.int64), r0.d.view(torch.int64))  # claimed folds: same association
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr,
                              injections=[K.Injection(row=r, col=100 + r % 500, bit=top) for r in rows])
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == rows
    changed = K.replay_tiles(x, w, b, y, res.flags, res, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert int(changed.item()) == 3
    assert torch.equal(y.view(torch.uint8), clean.view(torch.uint8))
    assert int(res.nflag.item()) == 0


def test_concurrent_streams_same_shape_do_not_share_counters():
    M, N, Kd = 4096, 768, 768
    x, w, b, ws, bs = _ops(M, N, Kd, torch.bfloat16, 21)
    x2 = torch.randn(M, Kd, device="cuda").to(torch.bfloat16)
    ref1, r1 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    ref2, r2 = K.protected_gemm(x2, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    d1, d2 = r1.d.clone(), r2.d.clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(20):
        with torch.cuda.stream(s1):
            ya, ra = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
        with torch.cuda.stream(s2):
            yb, rb = K.protected_gemm(x2, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
        outs.append((ya, ra, yb, rb))
    torch.cuda.synchronize()
    for ya, ra, yb, rb in outs:
        assert torch.equal(ya, ref1) and torch.equal(yb, ref2)
        assert torch.equal(ra.d, d1) and torch.equal(rb.d, d2)
        assert int(ra.nflag.item()) == 0 and int(rb.nflag.item()) == 0


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.int8])
def test_packed_output_campaign_equals_one_launch_per_fault(dtype):
    M, N, Kd = 512, 384, 256
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, 33)
    _, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    thr = 0.0 if dtype == torch.int8 else 4 * float(r0.d.abs().max().item())
    rng = np.random.default_rng(8)
    faults = [K.Injection(row=int(rng.integers(0, M)), col=int(rng.integers(0, N)), bit=int(rng.integers(0, 15)))
              for _ in range(400)]  # repeated rows force several launches
    got, launches = K.packed_output_campaign(x, w, b, faults, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    assert 1 < launches < 20
    want = []
    for f in faults:
        _, r = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr, injections=[f])
        want.append(bool(r.flags[f.row].item()))
    assert got.cpu().tolist() == want


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.int8])
@pytest.mark.parametrize("shape", [(1024, 3072, 768), (512, 8192, 256)])
def test_one_tile_per_pair_launch_end_fold(dtype, shape):
    """At most one tile per CTA pair: every band is split and folded at the end of the
    kernel by all threads of the CTA completing it (more than four bands), or every row
    by the launch's last CTA (tiny).  Faults in several bands are flagged exactly, and
    replay restores the clean bytes."""
    M, N, Kd = shape
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, 41)
    clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    integer = dtype == torch.int8
    thr = 0.0 if integer else 4 * float(r0.d.abs().max().item()) + 1e-6
    top = {torch.bfloat16: 14, torch.float32: 30, torch.int8: 30}[dtype]
    rows = [0, 130, 255, 300, M - 1]
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr,
                              injections=[K.Injection(row=r, col=(37 * r) % N, bit=top) for r in rows])
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == rows
    assert int(res.nflag.item()) == len(rows)
    changed = K.replay_tiles(x, w, b, y, res.flags, res, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert int(changed.item()) == len(rows)
    assert torch.equal(y.view(torch.uint8), clean.view(torch.uint8))
    assert int(res.nflag.item()) == 0


@pytest.mark.parametrize("shape", [(8192, 3072, 768), (50432, 2048, 256)])
def test_tf32_claimed_folds_replay(shape):
    """tf32 launches with >= 8 tiles per band fold their split bands through the claimed
    path (strided and contiguous schedules, and replay's active-band list): faults in
    several bands are flagged exactly, replay restores the clean bytes, and d repeats."""
    M, N, Kd = shape
    x, w, b, ws, bs = _ops(M, N, Kd, torch.float32, 17)
    clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    d0 = r0.d.clone()
    _, r1 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    assert torch.equal(r1.d.view(torch.int64), d0.view(torch.int64))
    thr = 4 * float(d0.abs().max().item()) + 1e-6
    rows = [3, 700, 4100, M - 2]
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr,
                              injections=[K.Injection(row=r, col=(11 * r) % N, bit=30) for r in rows])
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == rows
    changed = K.replay_tiles(x, w, b, y, res.flags, res, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert int(changed.item()) == len(rows)
    assert torch.equal(y.view(torch.uint8), clean.view(torch.uint8))
    assert int(res.nflag.item()) == 0
