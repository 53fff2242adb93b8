"""CPU ORACLE — test infrastructure only.

A NumPy restatement of the reference `gemmguard` algorithm on the
checksum-protected GEMM path (/root/reference/pkg/src/gemmguard).  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline — never as the thing measured or shipped.  The product path
(`paper_2310_03841_b200`) never imports it and fails loudly without its CUDA
library.

Parity status: PINNED.  `tests/test_oracle_golden.py` checks every function
here against (a) the reference's own known-answer vectors (lifted from
pkg/tests/*.py and SPEC.md) and (b) golden fixtures produced by importing the
reference itself (tests/golden/make_golden.py -> tests/golden/*.npz).  The
bf16 and tf32 operand kinds have no counterpart in the reference (numerics.py
:31-44 defines no such tags): the helpers for them below follow the same
rules with bf16 fields (7, 8) and are "parity unpinned".

Every reduction is np.add.accumulate, i.e. an ascending single-accumulator
fold that starts from the first element, exactly as the reference does.
"""

from __future__ import annotations

import math
from statistics import NormalDist

import numpy as np

# ----------------------------------------------------------------- encodings
# dtype tag -> (storage dtype, unsigned view, bits)      numerics.py:31-37
ENCODINGS = {
    "binary64": (np.float64, np.uint64, 64),
    "binary32": (np.float32, np.uint32, 32),
    "binary16-emulated": (np.float16, np.uint16, 16),
    "int8": (np.int8, np.uint8, 8),
    "int32": (np.int32, np.uint32, 32),
}
# (mantissa bits, exponent bits)                          numerics.py:40-44
FLOAT_FIELDS = {"binary64": (52, 11), "binary32": (23, 8), "binary16-emulated": (10, 5), "bfloat16": (7, 8)}
INT_DTYPES = ("int8", "int32")
# accumulation / checksum precision tag -> accumulator dtype  numerics.py:95-104
ACC = {
    "binary16-emulated": np.float16,
    "binary32": np.float32,
    "binary64": np.float64,
    "int64-exact": np.int64,
}
WIDTH = {"binary16-emulated": 16, "binary32": 32, "binary64": 64, "int64-exact": 64}


def fold(a: np.ndarray, axis: int) -> np.ndarray:
    """Ascending single-accumulator fold (numerics.py:211-215, guard.py:135-139)."""
    with np.errstate(over="ignore", invalid="ignore"):
        return np.take(np.add.accumulate(a, axis=axis), -1, axis=axis)


def round_to_dtype(arr: np.ndarray, dtype: str) -> np.ndarray:
    """RNE onto a dtype lattice, overflow -> +/-Inf (numerics.py:202-208)."""
    with np.errstate(over="ignore"):
        if dtype == "binary16-emulated":
            return np.asarray(arr, np.float64).astype(np.float16).astype(np.float64)
        if dtype == "binary32":
            return np.asarray(arr, np.float64).astype(np.float32)
        if dtype == "bfloat16":
            return bf16_round(np.asarray(arr, np.float64))
        return np.asarray(arr, np.float64)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Extension (parity unpinned): RNE float64 -> bfloat16, returned as float64.

    Rounds via float32 only when that is exact w.r.t. the final result: the
    value is first rounded to float32 with round-to-odd to avoid double
    rounding, then to 8 significant bits with RNE.
    """
    a = np.asarray(a, np.float64)
    f = a.astype(np.float32)
    # round-to-odd correction for the float64->float32 step
    back = f.astype(np.float64)
    bits = f.view(np.uint32).copy()
    inexact = (back != a) & np.isfinite(a)
    bits[inexact] |= 1
    lsb = (bits >> 16) & 1
    rounded = (bits + 0x7FFF + lsb) & 0xFFFF0000
    nan = np.isnan(a)
    rounded[nan] = 0x7FC00000
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


def tf32_truncate(a: np.ndarray) -> np.ndarray:
    """Extension (parity unpinned): the 19-bit tf32 operand the tensor core reads
    from an fp32 container (low 13 mantissa bits ignored)."""
    b = np.asarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


# ----------------------------------------------------------------- GEMM
PRODUCT_LIMIT = 1 << 26  # numerics.py:219


def gemm(x: np.ndarray, wt: np.ndarray, bias, dtype: str, accum: str | None = None) -> np.ndarray:
    """Y = X Wt + bias with the reference's rounding (numerics.py:237-289).

    x [B, I], wt [I, O] in the dtype's storage (float64 lattice values for
    binary16-emulated).  Products rounded in the accumulation dtype, ascending
    k single accumulator (materialised accumulate when B*I*O <= 2^26, else the
    k-loop starting from zero: numerics.py:222-234), bias added in the
    accumulation dtype, result rounded to the operand dtype.
    """
    if x.shape[1] != wt.shape[0]:
        raise ValueError(f"gemm dims mismatch: X is {x.shape}, Wt is {wt.shape}")
    if dtype in INT_DTYPES:
        if accum not in (None, "int64-exact"):
            raise ValueError("integer gemm requires the int64-exact accumulation tag")
        acc_dt = np.int32
    else:
        if accum is None:
            accum = "binary64" if dtype == "binary64" else "binary32"  # numerics.py:274-275
        if accum == "int64-exact":
            raise ValueError("float gemm requires a floating accumulation precision")
        if WIDTH[accum] < {"binary16-emulated": 16, "binary32": 32, "binary64": 64}[dtype]:
            raise ValueError(f"accumulation {accum} narrower than operand dtype {dtype}")
        if dtype == "binary16-emulated" and WIDTH[accum] < 32:
            raise ValueError("binary16-emulated gemm accumulates in binary32 or wider")
        acc_dt = ACC[accum]
    xb = x.astype(acc_dt)
    wb = wt.astype(acc_dt)
    b, i = xb.shape
    o = wb.shape[1]
    with np.errstate(over="ignore", invalid="ignore"):
        if b * i * o <= PRODUCT_LIMIT:
            prod = xb[:, :, None] * wb[None, :, :]
            y = np.ascontiguousarray(np.add.accumulate(prod, axis=1)[:, -1, :])
        else:
            y = np.zeros((b, o), dtype=acc_dt)
            for k in range(i):
                y += xb[:, k : k + 1] * wb[k : k + 1, :]
        if bias is not None:
            y = y + np.asarray(bias).astype(acc_dt)
    if dtype in INT_DTYPES:
        return y.astype(np.int32)
    return round_to_dtype(y.astype(np.float64), dtype)


# ----------------------------------------------------------------- checksum
def offline_checksum(wt: np.ndarray, bias: np.ndarray, prec: str) -> tuple[np.ndarray, float | int]:
    """w_sum[k] = fold_o Wt[k, o], bias_sum = fold bias, in `prec` (guard.py:142-160).

    wt is the reference layout [in_dim, out_dim] widened to float64 / int64."""
    integer = np.issubdtype(wt.dtype, np.integer)
    if integer and prec != "int64-exact":
        raise ValueError("integer layers require the int64-exact checksum precision")
    if not integer and prec == "int64-exact":
        raise ValueError("int64-exact checksums only apply to integer layers")
    acc = ACC[prec]
    w_sum = fold(wt.astype(np.int64 if integer else np.float64).astype(acc), axis=1)
    bias_sum = fold(np.asarray(bias).astype(acc), axis=0)
    return w_sum, (int(bias_sum) if integer else float(bias_sum))


def discrepancies(x: np.ndarray, y: np.ndarray, w_sum: np.ndarray, bias_sum, prec: str) -> np.ndarray:
    """d[b] = (fold_k x[b,k]*w_sum[k] + bias_sum) - fold_o y[b,o] in `prec`
    (guard.py:163-171); returned as float64, or int64 for int64-exact."""
    acc = np.dtype(ACC[prec])
    with np.errstate(over="ignore", invalid="ignore"):
        products = x.astype(acc) * w_sum.astype(acc)[None, :]
        predicted = fold(products, axis=1) + acc.type(bias_sum)
        observed = fold(y.astype(acc), axis=1)
        return (predicted - observed).astype(np.int64 if prec == "int64-exact" else np.float64)


def np_pairwise_sum(a: np.ndarray) -> float:
    """NumPy's pairwise summation of a contiguous float64 vector (np.add.reduce),
    used by d.mean() in the batch_mean statistic (guard.py:199)."""
    n = len(a)
    if n < 8:
        r = 0.0
        for v in a:
            r += float(v)
        return r
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return np_pairwise_sum(a[:n2]) + np_pairwise_sum(a[n2:])


def verify(x, y, w_sum, bias_sum, prec: str, eps: dict | None):
    """guard._verify_arrays (guard.py:188-215): (d, flags, max_disc, triggered).

    eps: {"mu", "threshold_low", "threshold_high", "statistic"} or None."""
    d = discrepancies(x, y, w_sum, bias_sum, prec)
    if prec == "int64-exact":
        flags = d != 0
        max_disc = float(np.abs(d).max())
    else:
        if eps is None:
            raise ValueError("floating-point verification requires an epsilon model")
        lo, hi = eps["threshold_low"], eps["threshold_high"]
        if eps.get("statistic", "per_sample") == "batch_mean":
            dm = np_pairwise_sum(d) / len(d)
            flags = np.full(d.shape, not (lo <= dm <= hi))
        else:
            flags = ~((d >= lo) & (d <= hi))
        with np.errstate(invalid="ignore"):
            gaps = np.abs(d - eps["mu"])
        max_disc = float(np.nanmax(gaps)) if np.isfinite(gaps).any() else math.inf
    return d, flags, max_disc, bool(flags.any())


# ----------------------------------------------------------------- thresholds
def threshold_from_confidence(mu: float, sigma: float, confidence: float) -> tuple[float, float]:
    """mu -/+ z*sigma, z = Phi^-1((1+c)/2) (guard.py:218-227)."""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    if not 0.5 < confidence < 1.0:
        raise ValueError("confidence must lie in (0.5, 1)")
    z = NormalDist().inv_cdf((1.0 + confidence) / 2.0)
    return (mu - z * sigma, mu + z * sigma)


def fit_epsilon(values: np.ndarray, confidence: float, integer: bool = False) -> dict:
    """Per-layer mu / sigma(ddof=1) / thresholds over clean d (guard.py:311-355)."""
    values = np.asarray(values, np.float64)
    if integer:
        if np.any(values != 0):
            raise ValueError("integer checksum discrepancies are nonzero on clean runs")
        return {"mu": 0.0, "sigma": 0.0, "threshold_low": 0.0, "threshold_high": 0.0, "n": len(values),
                "d_abs_max": 0.0}
    if len(values) < 30:
        raise ValueError(f"{len(values)} discrepancy samples < 30")
    mu = float(values.mean())
    sigma = float(values.std(ddof=1))
    if sigma == 0.0 and np.any(values != 0.0):
        raise ValueError("constant nonzero discrepancy (precision saturation)")
    lo, hi = threshold_from_confidence(mu, sigma, confidence)
    return {"mu": mu, "sigma": sigma, "threshold_low": lo, "threshold_high": hi, "n": len(values),
            "d_abs_max": float(np.abs(values).max())}


# ----------------------------------------------------------------- bit flips
def flip_bit(value, bit_index: int, dtype: str):
    """XOR one bit of the storage encoding (numerics.py:308-321); involution."""
    if dtype == "bfloat16":
        enc = np.array([value], dtype=np.float32).view(np.uint32) >> 16
        if not 0 <= bit_index < 16:
            raise ValueError(f"bit index {bit_index} out of range for {dtype} (16 bits)")
        enc = (enc ^ (1 << bit_index)) << 16
        return enc.astype(np.uint32).view(np.float32)[0]
    sdt, udt, bits = ENCODINGS[dtype]
    if not 0 <= bit_index < bits:
        raise ValueError(f"bit index {bit_index} out of range for {dtype} ({bits} bits)")
    with np.errstate(over="ignore"):
        enc = np.array([value], dtype=sdt).view(udt)
    enc ^= udt(1) << udt(bit_index)
    return enc.view(sdt)[0]


def bit_range(dtype: str, mode: str) -> tuple[int, int]:
    """Flip-mode bit ranges (injector.py:99-111)."""
    if dtype in INT_DTYPES:
        if mode != "int_bit":
            raise ValueError(f"mode {mode!r} invalid for integer dtype {dtype}")
        return (0, 8 if dtype == "int8" else 32)
    mant, exp = FLOAT_FIELDS[dtype]
    if mode == "fp_mantissa_bit":
        return (0, mant)
    if mode == "fp_exponent_bit":
        return (mant, mant + exp)
    if mode == "fp_sign_bit":
        return (mant + exp, mant + exp + 1)
    raise ValueError(f"mode {mode!r} invalid for floating dtype {dtype}")


def injection_rng(seed: int, layer_index: int, k: int) -> np.random.Generator:
    """Per-trial stream (injector.py:451-452)."""
    return np.random.default_rng(np.random.SeedSequence((seed, layer_index, k)))


def sample_output_flip(rng, target: np.ndarray, lo: float, hi: float, modes, dtype: str, max_retries: int = 64):
    """Draw order of injector.sample_injection for one output-location trial
    whose layer and sample are already fixed (injector.py:160-210): location
    (one choice: consumes no state), then per retry element, mode, bit;
    rejects no-ops and out-of-range corruptions.  Returns (element, mode, bit,
    original, corrupted) or None when the retry budget is exhausted."""
    _ = rng.integers(1)  # location choice among ("output",): integers(1) consumes nothing
    flat = target.ravel()
    for _ in range(max_retries):
        element = int(rng.integers(flat.size))
        mode = modes[int(rng.integers(len(modes)))]
        original = flat[element]
        original = int(original) if dtype in INT_DTYPES else float(original)
        b0, b1 = bit_range(dtype, mode)
        bit = int(rng.integers(b0, b1))
        out = flip_bit(original, bit, dtype)
        corrupted = int(out) if dtype in INT_DTYPES else float(out)
        if corrupted == original:
            continue
        if not (lo <= corrupted <= hi):
            continue
        return element, mode, bit, original, corrupted
    return None


def reduce_rows(a: np.ndarray) -> np.ndarray:
    """numerics.reduce_rows (numerics.py:292-297)."""
    acc = np.int64 if np.issubdtype(a.dtype, np.integer) else np.float64
    return fold(a.astype(acc), axis=1)


def reduce_cols(a: np.ndarray) -> np.ndarray:
    """numerics.reduce_cols (numerics.py:300-305)."""
    acc = np.int64 if np.issubdtype(a.dtype, np.integer) else np.float64
    return fold(a.astype(acc), axis=0)
