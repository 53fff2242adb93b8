"""ctypes binding of the C-ABI library (include/gemmguard_b200.h).

This is the reference-side binding a maintainer would add to `gemmguard`
(see INTEGRATION.md).  It loads ``libgemmguard_b200.so`` from the package
directory and FAILS LOUDLY when it is missing or unloadable: there is no CPU
fallback for the product path.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_uint8, c_void_p
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("GEMMGUARD_LIB", Path(__file__).resolve().parent / "libgemmguard_b200.so"))

# enum gg_dtype
GG_F64, GG_F32, GG_F16, GG_BF16, GG_I8, GG_I32, GG_I64, GG_TF32X3 = range(8)
# enum gg_precision
GG_P_F16, GG_P_F32, GG_P_F64, GG_P_I64 = range(4)
GG_PER_SAMPLE, GG_BATCH_MEAN = 0, 1
GG_INJ_OUTPUT, GG_INJ_ACCUMULATOR = 0, 1
GG_B_NK, GG_B_KN = 0, 1
GG_INJ_BITFLIP, GG_INJ_SET_VALUE = 0, 1
GG_ACT_NONE, GG_ACT_GELU_TANH, GG_ACT_RELU, GG_ACT_RESIDUAL = 0, 1, 2, 3
GG_OK, GG_EINVAL, GG_ECUDA, GG_EWORKSPACE, GG_EUNSUPPORTED = 0, -1, -2, -3, -4

# every symbol include/gemmguard_b200.h declares
EXPORTED_SYMBOLS = (
    "gg_last_error",
    "gg_version",
    "gg_protected_gemm_workspace_bytes",
    "gg_b_scratch_bytes",
    "gg_protected_gemm",
    "gg_replay_tiles",
    "gg_checksum_aux_bytes",
    "gg_checksum_aux",
    "gg_split_tf32x3",
    "gg_offline_checksum",
    "gg_verify_rows",
    "gg_locate_workspace_bytes",
    "gg_locate_tiles",
    "gg_flip_bits",
    "gg_gemm_exact",
    "gg_reduce",
    "gg_round_f64_to",
    "gg_running_stats",
    "gg_minmax",
    "gg_int_finish",
    "gg_add_layernorm",
    "gg_embed_layernorm",
    "gg_patchify",
)


class GGInjection(ctypes.Structure):
    _fields_ = [
        ("row", c_int64),
        ("col", c_int32),
        ("bit", c_int32),
        ("target", c_int32),
        ("mode", c_int32),
        ("value", c_double),
    ]


class GGGemmDesc(ctypes.Structure):
    _fields_ = [
        ("ab_kind", c_int32),
        ("c_dtype", c_int32),
        ("M", c_int64),
        ("N", c_int64),
        ("K", c_int64),
        ("A", c_void_p),
        ("lda", c_int64),
        ("B", c_void_p),
        ("ldb", c_int64),
        ("bias", c_void_p),
        ("C", c_void_p),
        ("ldc", c_int64),
        ("protect", c_int32),
        ("chk_prec", c_int32),
        ("w_sum", c_void_p),
        ("w_aux", c_void_p),
        ("bias_sum_f", c_double),
        ("bias_sum_i", c_int64),
        ("mu", c_double),
        ("lo", c_double),
        ("hi", c_double),
        ("statistic", c_int32),
        ("d", c_void_p),
        ("flags", c_void_p),
        ("max_disc", c_void_p),
        ("nflag", c_void_p),
        ("triggered", c_void_p),
        ("inj", c_void_p),
        ("n_inj", c_int32),
        ("workspace", c_void_p),
        ("workspace_bytes", c_size_t),
        ("replay_rows", c_void_p),
        ("changed", c_void_p),
        ("epilogue_act", c_int32),
        ("pred_in", c_void_p),
        ("b_layout", c_int32),
        ("b_scratch", c_void_p),
        ("b_scratch_bytes", c_size_t),
        ("requant_shift", c_int32),
        ("residual", c_void_p),
        ("ld_res", c_int64),
    ]


class GemmGuardLibraryError(RuntimeError):
    """The native library could not be loaded or a CUDA call failed."""


_lib = None


def load(path: Path | None = None):
    """Load (once) and return the ctypes handle, with argtypes declared."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise GemmGuardLibraryError(
            f"{p} is missing: build it with `python -m paper_2310_03841_b200.build` "
            "(the protected GEMM has no CPU fallback)"
        )
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as e:  # pragma: no cover - environment dependent
        raise GemmGuardLibraryError(f"cannot load {p}: {e}") from e
    lib.gg_last_error.restype = ctypes.c_char_p
    lib.gg_last_error.argtypes = []
    lib.gg_version.restype = c_int32
    lib.gg_protected_gemm_workspace_bytes.restype = c_size_t
    lib.gg_protected_gemm_workspace_bytes.argtypes = [c_int64, c_int64]
    lib.gg_protected_gemm.restype = c_int32
    lib.gg_protected_gemm.argtypes = [POINTER(GGGemmDesc), c_void_p]
    lib.gg_replay_tiles.restype = c_int32
    lib.gg_replay_tiles.argtypes = [POINTER(GGGemmDesc), c_void_p]
    lib.gg_checksum_aux_bytes.restype = c_size_t
    lib.gg_checksum_aux_bytes.argtypes = [c_int32, c_int64]
    lib.gg_checksum_aux.restype = c_int32
    lib.gg_checksum_aux.argtypes = [c_int32, c_void_p, c_int64, c_void_p, c_void_p]
    lib.gg_offline_checksum.restype = c_int32
    lib.gg_split_tf32x3.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p, c_int64, c_void_p]
    lib.gg_split_tf32x3.restype = c_int32
    lib.gg_offline_checksum.argtypes = [
        c_int32, c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p, c_int32, c_int32, c_void_p, c_void_p,
        c_void_p,
    ]
    lib.gg_verify_rows.restype = c_int32
    lib.gg_verify_rows.argtypes = [
        c_int32, c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p, c_int64, c_int64, c_int32, c_void_p,
        c_void_p, c_double, c_double, c_double, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
    ]
    lib.gg_b_scratch_bytes.restype = c_size_t
    lib.gg_b_scratch_bytes.argtypes = [c_int32, c_int64, c_int64]
    lib.gg_locate_workspace_bytes.restype = ctypes.c_size_t
    lib.gg_locate_workspace_bytes.argtypes = [c_int64, c_int64]
    lib.gg_locate_tiles.restype = c_int32
    lib.gg_locate_tiles.argtypes = [
        c_int32, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int32,
        c_void_p, c_int64, c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p, c_void_p, ctypes.c_size_t,
        c_void_p,
    ]
    lib.gg_flip_bits.restype = c_int32
    lib.gg_flip_bits.argtypes = [c_void_p, c_int32, c_void_p, c_void_p, c_int64, c_void_p]
    lib.gg_gemm_exact.restype = c_int32
    lib.gg_gemm_exact.argtypes = [c_int32, c_int32, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                  c_void_p, c_void_p]
    lib.gg_reduce.restype = c_int32
    lib.gg_reduce.argtypes = [c_int32, c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p]
    lib.gg_running_stats.restype = c_int32
    lib.gg_running_stats.argtypes = [c_void_p, c_int64, c_void_p, c_void_p]
    lib.gg_minmax.restype = c_int32
    lib.gg_minmax.argtypes = [c_int32, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]
    lib.gg_int_finish.restype = c_int32
    lib.gg_int_finish.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int32, c_int32, c_int32, c_void_p,
                                  c_void_p]
    lib.gg_round_f64_to.restype = c_int32
    lib.gg_add_layernorm.argtypes = [c_int32, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, ctypes.c_float,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.gg_add_layernorm.restype = c_int32
    lib.gg_embed_layernorm.argtypes = [c_int32, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                       c_void_p, ctypes.c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.gg_embed_layernorm.restype = c_int32
    lib.gg_patchify.argtypes = [c_int32, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p]
    lib.gg_patchify.restype = c_int32
    lib.gg_round_f64_to.argtypes = [c_int32, c_void_p, c_void_p, c_int64, c_void_p]
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map a GG_E* return code onto the reference's exception convention."""
    if rc == GG_OK:
        return
    msg = load().gg_last_error().decode("utf8", "replace")
    if rc in (GG_EINVAL, GG_EWORKSPACE):
        raise ValueError(msg or f"{what}: invalid argument")
    if rc == GG_EUNSUPPORTED:
        raise NotImplementedError(msg or f"{what}: unsupported")
    raise GemmGuardLibraryError(f"{what}: {msg}")
