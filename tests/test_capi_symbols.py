"""CPU: the C-ABI library builds, loads without a GPU, and exports every
symbol include/gemmguard_b200.h declares (no compute calls)."""

import ctypes
import re
from pathlib import Path

from paper_2310_03841_b200 import _lib as L

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    text = (ROOT / "include" / "gemmguard_b200.h").read_text()
    return sorted(set(re.findall(r"GG_API\s+[\w\s\*]+?\b(gg_\w+)\s*\(", text)))


def test_header_declares_the_binding_symbols():
    assert _declared_symbols() == sorted(L.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_all_symbols():
    lib = L.load()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    assert lib.gg_version() >= 10000
    assert lib.gg_last_error() == b""


def test_workspace_size_is_host_only_and_monotone():
    lib = L.load()
    a = lib.gg_protected_gemm_workspace_bytes(197, 768)
    b = lib.gg_protected_gemm_workspace_bytes(50432, 3072)
    assert 0 < a < b
    assert lib.gg_protected_gemm_workspace_bytes(0, 10) == 0


def test_argument_errors_surface_as_value_error_without_gpu():
    """Argument validation happens before any CUDA call."""
    lib = L.load()
    desc = L.GGGemmDesc()
    desc.ab_kind = 99
    desc.M = desc.N = desc.K = 4
    rc = lib.gg_protected_gemm(ctypes.byref(desc), None)
    assert rc == L.GG_EUNSUPPORTED
    assert b"ab_kind" in lib.gg_last_error()
    rc = lib.gg_flip_bits(None, 3, None, None, 1, None)
    assert rc == L.GG_EINVAL and b"element width" in lib.gg_last_error()
