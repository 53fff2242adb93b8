"""Tile localisation by column checksums (gg_locate_tiles) and tile-granular replay.

North-star kernel (1) asks for column checksums e^T A next to the row check so a fault
can be placed in its (row band, column tile); the reference checks rows only and
replays the whole layer (guard.py:575-604).  A fault at (r, n) moves row r's check and
column n's check by the same amount: int8 column discrepancies are exact, float ones
are compared with half the smallest flagged row discrepancy of the band."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402
from paper_2310_03841_b200.vit import ProtectedViT, ViTConfig  # noqa: E402

DT = [torch.bfloat16, torch.float16, torch.float32, torch.int8]
TOP = {torch.bfloat16: 14, torch.float16: 14, torch.float32: 30, torch.int8: 30}


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


def _faulted(dtype, M=1000, N=1000, Kd=300, seed=3, cells=((5, 40), (300, 700), (310, 999), (999, 260))):
    x, w, b, ws, bs = _ops(M, N, Kd, dtype, seed)
    clean, r0 = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-1e30, hi=1e30)
    torch.cuda.synchronize()
    thr = 0.0 if dtype == torch.int8 else 4 * float(r0.d.abs().max().item()) + 1e-6
    injs = [K.Injection(row=r, col=c, bit=TOP[dtype]) for r, c in cells]
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr, injections=injs)
    torch.cuda.synchronize()
    assert sorted(torch.nonzero(res.flags.cpu()).flatten().tolist()) == sorted(r for r, _ in cells)
    return x, w, b, ws, bs, thr, clean, y, res


@pytest.mark.parametrize("dtype", DT)
def test_locate_marks_exactly_the_faulty_tiles(dtype):
    cells = ((5, 40), (300, 700), (310, 999), (999, 260))
    x, w, b, ws, bs, thr, clean, y, res = _faulted(dtype, cells=cells)
    mask, cols = K.locate_tiles(x, w, b, y, res, with_columns=True)
    torch.cuda.synchronize()
    want = {(r // 128, c // 256) for r, c in cells}
    got = {tuple(t) for t in mask.nonzero().tolist()}
    assert got == want
    if dtype == torch.int8:  # exact: e[b, c] = true - stored at the faulty columns, 0 elsewhere
        delta = (clean.long() - y.long()).cpu().numpy()
        e = cols.cpu().numpy()
        for bnd in {r // 128 for r, _ in cells}:
            np.testing.assert_array_equal(e[bnd], delta[bnd * 128:(bnd + 1) * 128].sum(axis=0))


@pytest.mark.parametrize("dtype", DT)
def test_tile_replay_restores_clean_bytes_and_summary(dtype):
    cells = ((5, 40), (300, 700), (310, 999), (999, 260))
    x, w, b, ws, bs, thr, clean, y, res = _faulted(dtype, cells=cells)
    d_before = res.d.clone()
    changed, tiles = K.replay_located(x, w, b, y, res, w_sum=ws, bias_sum=bs, lo=-thr, hi=thr)
    torch.cuda.synchronize()
    assert tiles == 4  # of 4 x 4 = 16 band tiles of the flagged bands a band replay recomputes
    assert int(changed.item()) == len(cells)
    assert torch.equal(y.view(torch.uint8), clean.view(torch.uint8))
    assert int(res.nflag.item()) == 0 and int(res.triggered.item()) == 0
    assert not bool(res.flags.any())
    untouched = torch.ones(1000, dtype=torch.bool, device="cuda")
    for bnd in {r // 128 for r, _ in cells}:
        untouched[bnd * 128:(bnd + 1) * 128] = False
    assert torch.equal(res.d[untouched], d_before[untouched])  # other bands keep the fused d
    if dtype == torch.int8:  # exact d: the re-check agrees with a clean protected launch
        _, rc = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0)
        assert torch.equal(res.d, rc.d)


def test_cancelling_faults_in_one_column_fall_back_to_band_replay():
    """Two int8 faults of opposite sign in one column of one band leave that column's
    check at 0: the columns place nothing there, the rows stay flagged, and K4 replays
    their band."""
    M, N, Kd = 512, 512, 128
    x, w, b, ws, bs = _ops(M, N, Kd, torch.int8, 8)
    clean, _ = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0)
    torch.cuda.synchronize()
    v1, v2 = int(clean[10, 77].item()), int(clean[20, 77].item())
    injs = [K.Injection(row=10, col=77, mode=L.GG_INJ_SET_VALUE, value=float(v1 + 1000)),
            K.Injection(row=20, col=77, mode=L.GG_INJ_SET_VALUE, value=float(v2 - 1000))]
    y, res = K.protected_gemm(x, w, b, w_sum=ws, bias_sum=bs, lo=0, hi=0, injections=injs)
    torch.cuda.synchronize()
    assert torch.nonzero(res.flags.cpu()).flatten().tolist() == [10, 20]
    mask, _ = K.locate_tiles(x, w, b, y, res)
    assert int(mask.sum().item()) == 0
    changed, tiles = K.replay_located(x, w, b, y, res, w_sum=ws, bias_sum=bs, lo=0, hi=0)
    torch.cuda.synchronize()
    assert tiles == 0 and int(changed.item()) == 2
    assert torch.equal(y, clean)
    assert int(res.nflag.item()) == 0


def test_vit_tile_granular_replay_restores_the_clean_logits():
    cfg = ViTConfig(name="vit_s_test", dim=256, depth=2, heads=4, mlp=1024, classes=10)
    model = ProtectedViT(cfg, seed=5)
    g = torch.Generator(device="cuda").manual_seed(10)
    cal = [torch.randn(8, 3, cfg.image, cfg.image, device="cuda", generator=g) for _ in range(3)]
    model.calibrate(cal, confidence=1 - 1e-9)
    imgs = torch.randn(8, 3, cfg.image, cfg.image, device="cuda", generator=g)
    clean = model(imgs).clone()
    layer, row = 8, 2 * cfg.tokens + 5  # fc2 of block 1 (no fused activation): tile replay applies
    assert model.linears[layer].act == L.GG_ACT_NONE
    inj = K.injections_to_device([K.Injection(row=row, col=200, bit=14)], torch.device("cuda"))
    model.enable_replay(granularity="tile")
    fixed = model(imgs, injections={layer: inj}).clone()
    model.disable_replay()
    assert torch.equal(fixed, clean)
    assert model.replay_events == [(layer, "replay", 1)]

