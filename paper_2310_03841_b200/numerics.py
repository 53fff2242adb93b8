"""Matrix type, precisions and the GEMM entry point of the protected path.

Drop-in for ``gemmguard.numerics`` (/root/reference/pkg/src/gemmguard/
numerics.py).  Host-side types (`Matrix2D`, `Precision`, dtype tags, bit
fields) keep the reference's names, storage conventions, validation and error
messages.  The arithmetic runs on the B200:

* `gemm` launches the tcgen05 GEMM of libgemmguard_b200.so (engine
  ``"tensor"``: kind::i8 for int8, kind::f16 for binary16-emulated, and
  3xTF32 on kind::tf32 for binary32 — x*w = hi*lo + lo*hi + hi*hi, ~2^-21 per
  product) or the reference-order CUDA-core fold (engine ``"exact"``,
  bit-identical to numerics.py:222-289 for every dtype/accum pair, and the
  only engine for binary64 and int32 operands).  Engine ``"tf32"`` is the
  explicit opt-in for single-pass TF32 on binary32 operands (10-bit mantissa
  products: about 2^-11 relative error; other dtypes run as ``"tensor"``).
  The default engine ``"auto"`` is ``"tensor"`` for int8 (bit-exact) and
  binary16-emulated (exact fp32 products, fp32 accumulation like the
  reference) and ``"exact"`` for binary32: the tensor core's fp32 accumulator
  truncates on every step, which leaves 3xTF32's row sums about 4x noisier
  than the reference's binary32 fold (cfg1: 7.7e-5 against 1.8e-5), so the
  reference's epsilon and detection parity for binary32 models come from the
  bit-exact engine unless a caller opts into the tensor pipe;
* `reduce_rows` / `reduce_cols` are ascending device folds (numerics.py:292-305).

`flip_bit` and `round_to` are scalar encodings helpers of the API
(numerics.py:308-336); the device fault injector is K3 (gg_flip_bits) and
the in-epilogue injection of the protected GEMM.
"""

from __future__ import annotations

import enum
import os
from typing import Sequence

import numpy as np
import torch

from . import _device as D
from . import _lib as L
from . import kernels as K

__all__ = [
    "Matrix2D",
    "Precision",
    "gemm",
    "reduce_rows",
    "reduce_cols",
    "flip_bit",
    "round_to",
    "FLOAT_DTYPES",
    "INT_DTYPES",
    "DTYPE_TAGS",
    "encoding_of",
    "float_fields",
    "ENGINES",
    "default_engine",
]

# tag -> (host storage dtype, unsigned encoding view, bit width)   numerics.py:31-37
_ENC = {
    "binary64": (np.float64, np.uint64, 64),
    "binary32": (np.float32, np.uint32, 32),
    "binary16-emulated": (np.float16, np.uint16, 16),
    "int8": (np.int8, np.uint8, 8),
    "int32": (np.int32, np.uint32, 32),
}
# (mantissa, exponent) bits                                        numerics.py:40-44
_FIELDS = {"binary64": (52, 11), "binary32": (23, 8), "binary16-emulated": (10, 5)}
_FLOAT_WIDTH = {"binary16-emulated": 16, "binary32": 32, "binary64": 64}

FLOAT_DTYPES = frozenset(_FIELDS)
INT_DTYPES = frozenset(("int8", "int32"))
DTYPE_TAGS = tuple(_ENC)

ENGINES = ("auto", "tensor", "exact", "tf32")


def default_engine() -> str:
    """GEMM engine used when a call does not name one ($GEMMGUARD_ENGINE, default "auto")."""
    e = os.environ.get("GEMMGUARD_ENGINE", "auto")
    if e not in ENGINES:
        raise ValueError(f"GEMMGUARD_ENGINE must be one of {ENGINES}, got {e!r}")
    return e


def encoding_of(dtype: str) -> tuple[np.dtype, np.dtype, int]:
    """(storage dtype, unsigned view dtype, bit width) of a dtype tag (numerics.py:61-67)."""
    if dtype not in _ENC:
        raise ValueError(f"unknown dtype tag {dtype!r}")
    s, u, bits = _ENC[dtype]
    return np.dtype(s), np.dtype(u), bits


def float_fields(dtype: str) -> tuple[int, int]:
    """(mantissa bits, exponent bits) of a floating tag (numerics.py:70-74)."""
    if dtype not in _FIELDS:
        raise ValueError(f"{dtype!r} is not a floating dtype")
    return _FIELDS[dtype]


class Precision(enum.Enum):
    """Accumulation / checksum precision (numerics.py:77-111)."""

    BINARY16 = "binary16-emulated"
    BINARY32 = "binary32"
    BINARY64 = "binary64"
    INT64 = "int64-exact"

    @property
    def is_float(self) -> bool:
        return self is not Precision.INT64

    @property
    def width(self) -> int:
        return 64 if self in (Precision.BINARY64, Precision.INT64) else (32 if self is Precision.BINARY32 else 16)

    @property
    def accumulator_dtype(self) -> np.dtype:
        return np.dtype({"binary16-emulated": np.float16, "binary32": np.float32,
                         "binary64": np.float64, "int64-exact": np.int64}[self.value])

    @property
    def gg_code(self) -> int:
        """enum gg_precision of include/gemmguard_b200.h."""
        return {"binary16-emulated": L.GG_P_F16, "binary32": L.GG_P_F32,
                "binary64": L.GG_P_F64, "int64-exact": L.GG_P_I64}[self.value]

    @classmethod
    def from_tag(cls, tag: str) -> "Precision":
        for p in cls:
            if p.value == tag:
                return p
        raise ValueError(f"unknown precision tag {tag!r}")


# host storage: binary16-emulated keeps float64 lattice values (numerics.py:52-58)
_HOST = {"binary64": np.float64, "binary32": np.float32, "binary16-emulated": np.float64,
         "int8": np.int8, "int32": np.int32}


def _on_b16_lattice(a: np.ndarray) -> bool:
    w = np.asarray(a, dtype=np.float64)
    with np.errstate(over="ignore"):
        rt = w.astype(np.float16).astype(np.float64)
    return bool(((rt == w) | (np.isnan(rt) & np.isnan(w))).all())


class Matrix2D:
    """Row-major matrix with a dtype tag (numerics.py:127-199).

    Construction copies; binary16-emulated data must lie on the binary16
    lattice; integer data must fit the tag; equality is bytewise.
    """

    __slots__ = ("rows", "cols", "dtype", "data", "__weakref__")

    def __init__(self, data, dtype: str = "binary64", *, _trusted: bool = False):
        if dtype not in _ENC:
            raise ValueError(f"unknown dtype tag {dtype!r}")
        src = np.asarray(data)
        if src.ndim != 2:
            raise ValueError(f"Matrix2D requires 2-D data, got shape {src.shape}")
        if min(src.shape) < 1:
            raise ValueError(f"Matrix2D requires positive dims, got shape {src.shape}")
        host = _HOST[dtype]
        if dtype in INT_DTYPES:
            if not np.issubdtype(src.dtype, np.integer):
                raise ValueError(f"{dtype} matrix requires integer data")
            out = src.astype(host)
            if not _trusted and not np.array_equal(out.astype(np.int64), src.astype(np.int64)):
                raise ValueError(f"element out of range for {dtype}")
        else:
            out = src.astype(host, copy=True)
            if not _trusted and dtype == "binary16-emulated" and not _on_b16_lattice(out):
                raise ValueError("element not representable on the binary16 lattice")
        self.rows, self.cols = int(out.shape[0]), int(out.shape[1])
        self.dtype = dtype
        self.data = np.ascontiguousarray(out)

    @classmethod
    def zeros(cls, rows: int, cols: int, dtype: str = "binary64") -> "Matrix2D":
        return cls(np.zeros((rows, cols), dtype=_HOST[dtype]), dtype, _trusted=True)

    @classmethod
    def identity(cls, n: int, dtype: str = "binary64") -> "Matrix2D":
        return cls(np.eye(n, dtype=_HOST[dtype]), dtype, _trusted=True)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def copy(self) -> "Matrix2D":
        return Matrix2D(self.data.copy(), self.dtype, _trusted=True)

    def widened(self) -> np.ndarray:
        """Exact widening: float64 for floats, int64 for ints."""
        return self.data.astype(np.int64 if self.dtype in INT_DTYPES else np.float64)

    def tolist(self):
        return self.data.tolist()

    def to_device(self) -> torch.Tensor:
        """Device copy in the device storage type (fp16 for binary16-emulated)."""
        return D.to_device(self.data, self.dtype)

    def __eq__(self, other) -> bool:
        if not isinstance(other, Matrix2D):
            return NotImplemented
        return (self.dtype, self.shape) == (other.dtype, other.shape) and \
            self.data.tobytes() == other.data.tobytes()

    def __hash__(self):
        raise TypeError("Matrix2D is unhashable")

    def __repr__(self) -> str:
        return f"Matrix2D({self.rows}x{self.cols}, {self.dtype})"


# ----------------------------------------------------------------------- GEMM
def _check_gemm_args(X: Matrix2D, Wt: Matrix2D, bias, accum):
    """Validation and defaulting exactly as numerics.gemm (numerics.py:251-281)."""
    if X.cols != Wt.rows:
        raise ValueError(f"gemm dims mismatch: X is {X.shape}, Wt is {Wt.shape}")
    if X.dtype != Wt.dtype:
        raise ValueError(f"gemm operand dtypes differ: {X.dtype} vs {Wt.dtype}")
    if bias is not None:
        bias = np.asarray(bias)
        if bias.ndim != 1 or bias.shape[0] != Wt.cols:
            raise ValueError(f"bias length {bias.shape} does not match out dim {Wt.cols}")
    dtype = X.dtype
    if dtype in INT_DTYPES:
        accum = Precision.INT64 if accum is None else accum
        if accum is not Precision.INT64:
            raise ValueError("integer gemm requires the int64-exact accumulation tag")
        return bias, accum
    if accum is None:
        accum = Precision.BINARY64 if dtype == "binary64" else Precision.BINARY32
    if not accum.is_float:
        raise ValueError("float gemm requires a floating accumulation precision")
    if accum.width < _FLOAT_WIDTH[dtype]:
        raise ValueError(f"accumulation {accum.value} narrower than operand dtype {dtype}")
    if dtype == "binary16-emulated" and accum.width < 32:
        raise ValueError("binary16-emulated gemm accumulates in binary32 or wider")
    return bias, accum


def tensor_engine_applies(dtype: str, accum: Precision) -> bool:
    """The tcgen05 path covers int8 (int32 accumulate) and binary16/binary32
    operands with binary32 accumulation (3xTF32, or opt-in tf32, for binary32)."""
    if dtype == "int8":
        return True
    return dtype in ("binary16-emulated", "binary32") and accum is Precision.BINARY32


def resolve_engine(dtype: str, accum: Precision, engine: str | None) -> str:
    e = engine or default_engine()
    if e not in ENGINES:
        raise ValueError(f"engine must be one of {ENGINES}, got {e!r}")
    if e == "auto":
        e = "exact" if dtype == "binary32" else "tensor"
    if e in ("tensor", "tf32") and not tensor_engine_applies(dtype, accum):
        return "exact"
    if e == "tf32" and dtype != "binary32":
        return "tensor"
    return e


def f32_mode_of(engine: str) -> str:
    """kernels.protected_gemm f32_mode of a tensor-path engine."""
    return "tf32" if engine == "tf32" else "3xtf32"


def is_tensor_engine(engine: str) -> bool:
    return engine in ("tensor", "tf32")


def device_bias(bias, dtype: str, engine: str) -> torch.Tensor | None:
    """Bias in the type each kernel reads: i32 (int), f32 (tensor float), f64 (exact float)."""
    if bias is None:
        return None
    b = np.asarray(bias)
    dev = D.device()
    if dtype in INT_DTYPES:
        with np.errstate(over="ignore"):
            return torch.from_numpy(b.astype(np.int32)).to(dev)  # bias.astype(int32), numerics.py:271
    if is_tensor_engine(engine):
        with np.errstate(over="ignore"):
            return torch.from_numpy(b.astype(np.float32)).to(dev)  # bias.astype(acc = fp32)
    return torch.from_numpy(b.astype(np.float64)).to(dev)


def gemm_device(x: torch.Tensor, wt_nk: torch.Tensor | None, wt_kn: torch.Tensor | None, bias_dev,
                dtype: str, accum: Precision, engine: str) -> torch.Tensor:
    """Device GEMM on prepared operands: x [M,K]; weight as [N,K] (tensor) or [K,N] (exact)."""
    if is_tensor_engine(engine):
        y, _ = K.protected_gemm(x, wt_nk, bias_dev, protect=False, f32_mode=f32_mode_of(engine))
        return y
    if dtype in INT_DTYPES:
        return K.gemm_exact(x, wt_kn, bias_dev, L.GG_P_I64)
    return K.gemm_exact(x, wt_kn, bias_dev, accum.gg_code)


def gemm(
    X: Matrix2D,
    Wt: Matrix2D,
    bias: Sequence[float] | np.ndarray | None = None,
    accum: Precision | None = None,
    *,
    engine: str | None = None,
) -> Matrix2D:
    """Y[b,o] = sum_k X[b,k] Wt[k,o] + bias[o] on the B200 (numerics.py:237-289).

    Same validation, defaults, rounding to the operand dtype and int32
    result for integer operands as the reference.  engine="exact" reproduces
    the reference's bits; engine="tensor" (default) runs tcgen05 and matches
    bit-exactly for int8 and within the binary32-accumulation bound for floats
    (binary32 operands as 3xTF32); engine="tf32" opts binary32 into one tf32
    pass (about 2^-11 relative error per product).
    """
    bias, accum = _check_gemm_args(X, Wt, bias, accum)
    dtype = X.dtype
    eng = resolve_engine(dtype, accum, engine)
    x = X.to_device()
    wt = Wt.to_device()
    b = device_bias(bias, dtype, eng)
    if is_tensor_engine(eng):
        y = gemm_device(x, wt.t().contiguous(), None, b, dtype, accum, eng)
    else:
        y = gemm_device(x, None, wt, b, dtype, accum, eng)
    out_tag = "int32" if dtype in INT_DTYPES else dtype
    return Matrix2D(D.to_host(y, out_tag), out_tag, _trusted=True)


# ----------------------------------------------------------------- reductions
def _reduce(M: Matrix2D, axis: int) -> np.ndarray:
    if M.rows == 0 or M.cols == 0:
        raise ValueError("reduce of empty matrix")
    out = K.reduce(M.to_device(), axis)
    return out.cpu().numpy()


def reduce_rows(M: Matrix2D) -> np.ndarray:
    """Per-row ascending sums in binary64 (int64 for ints), numerics.py:292-297."""
    return _reduce(M, 1)


def reduce_cols(M: Matrix2D) -> np.ndarray:
    """Per-column ascending sums in binary64 (int64 for ints), numerics.py:300-305."""
    return _reduce(M, 0)


# ------------------------------------------------------------ scalar helpers
def flip_bit(value, bit_index: int, dtype: str):
    """XOR bit `bit_index` of value's storage encoding; returns a NumPy scalar.

    Pure bit manipulation (NaN payloads survive; a second flip restores the
    encoding), numerics.py:308-321.
    """
    sdt, udt, bits = encoding_of(dtype)
    if not 0 <= bit_index < bits:
        raise ValueError(f"bit index {bit_index} out of range for {dtype} ({bits} bits)")
    with np.errstate(over="ignore"):
        word = np.array([value], dtype=sdt).view(udt)
    word ^= udt.type(1) << udt.type(bit_index)
    return word.view(sdt)[0]


def round_to(value: float, p: Precision) -> float:
    """RNE into precision p, widened back to binary64 (numerics.py:324-336)."""
    if not p.is_float:
        raise ValueError("round_to requires a floating precision")
    narrow = {Precision.BINARY16: np.float16, Precision.BINARY32: np.float32}.get(p)
    if narrow is None:
        return float(value)
    with np.errstate(over="ignore"):
        return float(narrow(value))
