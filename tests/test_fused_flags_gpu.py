"""Fused-check flags against the reference rule at calibrated thresholds.

For every operand kind and the cfg2 / cfg3 GEMM shapes (one 197-token image
and a batch of 256 images of ViT-B/16), epsilon is calibrated the reference's
way (per-row mean / std(ddof=1) of clean d, guard.py:300-360) at c = 0.9999
and c = 1 - 1e-9, then a held-out launch with injected output faults is
checked by the fused epilogue (K1) and by guard._verify_arrays' rule on the
SAME stored Y (reference-order folds: `gg_verify_rows`, bit-identical to the
oracle, which is re-run on a slice of rows here).

Bars:
* int8: d, flags, nflag, triggered and max_disc bit-exact;
* floats: a row's flag may differ only where the reference d lies within
  the fused d's stated error bound of a threshold, |d_ref - lo|, |d_ref - hi|
  <= 2^-19 * sum|terms| (include/gemmguard_b200.h); such rows
  are counted and reported (expected 0); nflag / triggered follow; max_disc
  within the same bound; the batch_mean statistic equals the reference's
  NumPy pairwise mean rule.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import gemmguard_oracle as O  # noqa: E402
from paper_2310_03841_b200 import _lib as L  # noqa: E402
from paper_2310_03841_b200 import kernels as K  # noqa: E402

KINDS = {
    "bf16": (torch.bfloat16, "3xtf32"),
    "fp16": (torch.float16, "3xtf32"),
    "f32": (torch.float32, "3xtf32"),
    "tf32": (torch.float32, "tf32"),
    "int8": (torch.int8, "3xtf32"),
}
SHAPES = [(50432, 2304, 768), (50432, 768, 768), (50432, 3072, 768), (50432, 768, 3072),
          (197, 768, 768), (197, 2304, 768), (197, 3072, 768), (197, 768, 3072)]
CONFIDENCES = (0.9999, 1.0 - 1e-9)
BOUND = 2.0**-19


def _operands(kind, M, N, Kd, seed):
    dt, _ = KINDS[kind]
    g = torch.Generator(device="cuda").manual_seed(seed)
    if dt == torch.int8:
        x = torch.randint(-128, 128, (M, Kd), device="cuda", generator=g, dtype=torch.int32).to(torch.int8)
        w = torch.randint(-128, 128, (N, Kd), device="cuda", generator=g, dtype=torch.int32).to(torch.int8)
        b = torch.randint(-64, 65, (N,), device="cuda", generator=g, dtype=torch.int32)
    else:
        x = torch.randn(M, Kd, device="cuda", generator=g).to(dt)
        w = (torch.randn(N, Kd, device="cuda", generator=g) / math.sqrt(Kd)).to(dt)
        b = 0.02 * torch.randn(N, device="cuda", generator=g)
    return x, w, b


def _new_x(kind, M, Kd, seed):
    dt, _ = KINDS[kind]
    g = torch.Generator(device="cuda").manual_seed(seed)
    if dt == torch.int8:
        return torch.randint(-128, 128, (M, Kd), device="cuda", generator=g, dtype=torch.int32).to(torch.int8)
    return torch.randn(M, Kd, device="cuda", generator=g).to(dt)


def _faults(M, N, kind, seed):
    """Output bit flips on distinct rows: exponent and mantissa bits of the stored encoding."""
    rng = np.random.default_rng(seed)
    n = min(64, max(8, M // 8))
    rows = rng.choice(M, size=n, replace=False)
    bits = {"bf16": 16, "fp16": 16, "f32": 32, "tf32": 32, "int8": 32}[kind]
    return [K.Injection(row=int(r), col=int(rng.integers(N)), bit=int(rng.integers(bits))) for r in rows]


def _abs_terms(x, y, w_sum, bsum):
    """sum_k |x w_sum| + |bias_sum| + sum_n |y| per row (fp64): the scale of the fused d's error bound."""
    xs = x.double() if x.dtype != torch.int8 else x.to(torch.float64)
    yy = y.double()
    return (xs.abs() @ w_sum.double().abs() + abs(bsum) + yy.abs().nansum(dim=1)).cpu().numpy()


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("kind", list(KINDS))
def test_fused_flags_equal_reference_rule_at_calibrated_epsilon(kind, shape):
    M, N, Kd = shape
    dt, f32_mode = KINDS[kind]
    integer = dt == torch.int8
    prec = L.GG_P_I64 if integer else L.GG_P_F64
    x, w, b = _operands(kind, M, N, Kd, 7)
    w_sum, bsum_t = K.offline_checksum(w, b, prec)
    bsum = int(bsum_t.item()) if integer else float(bsum_t.item())
    aux = K.checksum_aux(w_sum, dt, f32_mode)
    w_split = K.split_tf32x3(w, 1) if (dt == torch.float32 and f32_mode == "3xtf32") else None
    kw = dict(w_sum=w_sum, w_aux=aux, bias_sum=bsum, f32_mode=f32_mode, w_split=w_split)

    # calibration: reference-order d of a clean launch (guard.calibrate_epsilon's statistic)
    y0, _ = K.protected_gemm(x, w, b, lo=-1e300, hi=1e300, **kw)
    ref0 = K.verify_rows(x, y0, w_sum, bsum_t, prec, lo=-1e300, hi=1e300)
    d0 = ref0.d.cpu().numpy()
    if integer:
        assert not d0.any()
        eps_list = [(0.0, 0.0, 0.0)]
    else:
        eps_list = []
        for c in CONFIDENCES:
            e = O.fit_epsilon(d0, c)
            eps_list.append((e["mu"], e["threshold_low"], e["threshold_high"]))

    # held-out input with injected output faults
    x1 = _new_x(kind, M, Kd, 11)
    faults = _faults(M, N, kind, 3)
    excused_total = 0
    for mu, lo, hi in eps_list:
        y1, fused = K.protected_gemm(x1, w, b, mu=mu, lo=lo, hi=hi, injections=faults, **kw)
        ref = K.verify_rows(x1, y1, w_sum, bsum_t, prec, mu=mu, lo=lo, hi=hi)
        fd, rd = fused.d.cpu().numpy(), ref.d.cpu().numpy()
        ff, rf = fused.flags.cpu().numpy().astype(bool), ref.flags.cpu().numpy().astype(bool)
        if integer:
            assert np.array_equal(fd, rd)
            assert np.array_equal(ff, rf)
            assert int(fused.nflag.item()) == int(ref.nflag.item()) == int(rf.sum())
            assert fused.max_disc.item() == ref.max_disc.item()
            assert int(fused.triggered.item()) == int(ref.triggered.item())
            assert rf[[f.row for f in faults]].all()  # int32 outputs: every flip changes the row sum
            continue
        tol = BOUND * _abs_terms(x1, y1, w_sum, bsum) + 1e-300
        fin = np.isfinite(rd)
        assert np.all(np.abs(fd[fin] - rd[fin]) <= tol[fin])
        assert np.array_equal(np.isnan(fd), np.isnan(rd))
        diff = np.flatnonzero(ff != rf)
        for r in diff:
            assert min(abs(rd[r] - lo), abs(rd[r] - hi)) <= tol[r], (r, rd[r], lo, hi, tol[r])
        excused_total += len(diff)
        assert abs(int(fused.nflag.item()) - int(rf.sum())) <= len(diff)
        if len(diff) == 0:
            assert int(fused.nflag.item()) == int(ref.nflag.item())
            assert int(fused.triggered.item()) == int(ref.triggered.item())
        mf, mr = fused.max_disc.item(), ref.max_disc.item()
        assert (math.isinf(mf) and math.isinf(mr)) or abs(mf - mr) <= float(tol.max())
        # the oracle itself on a slice of rows (reference-order verify is pinned to it bit for bit)
        rows = np.unique(np.concatenate([np.arange(min(M, 96)), [f.row for f in faults][:32]]))
        xs = x1[rows].float().cpu().numpy().astype(np.float64)
        ys = y1[rows].float().cpu().numpy().astype(np.float64)
        od, oflags, _, _ = O.verify(xs, ys, w_sum.cpu().numpy(), bsum, "binary64",
                                    {"mu": mu, "threshold_low": lo, "threshold_high": hi})
        assert np.array_equal(od[np.isfinite(od)], rd[rows][np.isfinite(od)])
        assert np.array_equal(oflags, rf[rows])
    print(f"{kind} {M}x{N}x{Kd}: {excused_total} flag differences inside the fused-d bound")
    assert excused_total <= 2


@pytest.mark.parametrize("kind", ["bf16", "fp16", "f32"])
def test_fused_batch_mean_is_the_reference_pairwise_mean(kind):
    """statistic=batch_mean: every row flags iff NumPy's pairwise mean of d
    (guard.py:198-201) leaves [lo, hi]; the launch re-derives the flags from
    the fused d with that exact fold."""
    dt, f32_mode = KINDS[kind]
    M, N, Kd = 50432, 768, 768
    x, w, b = _operands(kind, M, N, Kd, 5)
    w_sum, bsum_t = K.offline_checksum(w, b, L.GG_P_F64)
    bsum = float(bsum_t.item())
    kw = dict(w_sum=w_sum, bias_sum=bsum, f32_mode=f32_mode)
    y, base = K.protected_gemm(x, w, b, lo=-1e300, hi=1e300, **kw)
    d = base.d.cpu().numpy()
    dm = O.np_pairwise_sum(d) / len(d)
    assert dm == float(d.mean())  # the oracle's pairwise sum is NumPy's
    for lo, hi, want in ((dm - 1.0, dm + 1.0, 0), (dm + 1e-9, dm + 1.0, 1), (dm - 1.0, dm - 1e-9, 1),
                         (dm, dm, 0)):
        _, r = K.protected_gemm(x, w, b, mu=0.0, lo=lo, hi=hi, statistic=L.GG_BATCH_MEAN, **kw)
        flags = r.flags.cpu().numpy()
        assert np.array_equal(r.d.cpu().numpy(), d)  # d does not depend on the statistic
        assert (flags == want).all()
        assert int(r.nflag.item()) == want * M and int(r.triggered.item()) == want
        assert r.max_disc.item() == float(np.nanmax(np.abs(d)))


def test_int8_accumulator_wraps_like_the_reference():
    """SURVEY §7 hard part 9: at K = 2^17 with x = w = -128 every product is
    2^14 and the int32 accumulator reaches 2^31; the reference's int32
    accumulate wraps silently (numerics.py:262-272) and the int64-exact check
    then flags the clean row (d = 2^32).  The tcgen05 s32 accumulator does the same."""
    M, N, Kd = 3, 256, 1 << 17
    x = torch.full((M, Kd), -128, dtype=torch.int8, device="cuda")
    x[1] = 1  # a row that does not overflow
    w = torch.full((N, Kd), -128, dtype=torch.int8, device="cuda")
    b = torch.zeros(N, dtype=torch.int32, device="cuda")
    xs, ws = x.cpu().numpy(), w.cpu().numpy()
    want = O.gemm(xs, np.ascontiguousarray(ws.T), b.cpu().numpy(), "int8")
    y, _ = K.protected_gemm(x, w, b, protect=False)
    assert np.array_equal(y.cpu().numpy(), want)
    assert int(want[0, 0]) == -(2**31)
    w_sum, bs = K.offline_checksum(w, b, L.GG_P_I64)
    _, res = K.protected_gemm(x, w, b, w_sum=w_sum, bias_sum=int(bs.item()))
    d = res.d.cpu().numpy()
    assert d[0] == N * 2**32 and d[2] == N * 2**32 and d[1] == 0
    assert res.flags.cpu().numpy().tolist() == [1, 0, 1]
