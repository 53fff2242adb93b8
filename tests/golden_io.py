"""Loading of the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the reference itself) and the seeded input
generator shared with that script."""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@lru_cache(None)
def npz(name: str) -> dict:
    with np.load(GOLDEN / name) as f:
        return {k: f[k] for k in f.files}


@lru_cache(None)
def doc(name: str):
    return json.loads((GOLDEN / name).read_text())


def rand_values(rng, rows, cols, dtype) -> np.ndarray:
    """Host values exactly as make_golden.rand_matrix draws them."""
    if dtype == "int8":
        return rng.integers(-128, 128, (rows, cols))
    if dtype == "int32":
        return rng.integers(-(2**20), 2**20, (rows, cols))
    v = rng.standard_normal((rows, cols))
    if dtype == "binary16-emulated":
        return v.astype(np.float16).astype(np.float64)
    if dtype == "binary32":
        return v.astype(np.float32)
    return v


def gemm_case_inputs(case):
    """(X, Wt, bias) host arrays of one GEMM fixture case, regenerated from its seed."""
    name, dt, acc, B, I, O, seed = case
    rng = np.random.default_rng(seed)
    x = rand_values(rng, B, I, dt)
    wt = rand_values(rng, I, O, dt)
    if dt in ("int8", "int32"):
        bias = rng.integers(-50, 50, O).astype(np.int32)
        if dt == "int32":
            bias = rng.integers(-(2**31), 2**31 - 1, O).astype(np.int64)
    else:
        bias = rand_values(rng, 1, O, dt)[0].astype(np.float64)
    return x, wt, bias


def cfg1_inputs(n: int = 1024, seed: int = 2310):
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    x = rng.standard_normal((n, n)).astype(np.float32)
    wt = (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32)
    bias = (0.02 * rng.standard_normal(n)).astype(np.float32).astype(np.float64)
    return x, wt, bias
