"""B200-native checksum-protected GEMM path of ALBERTA (arXiv 2310.03841).

Drop-in for the reference package ``gemmguard`` on its hot path: the same
module names (``numerics``, ``model``, ``guard``, ``injector``,
``profiler``, ``errors``), signatures, dataclasses and exceptions, with the
arithmetic in hand-written sm_100a kernels (libgemmguard_b200.so).  The
top-level exports mirror gemmguard/__init__.py:3-24.
"""

from .numerics import Matrix2D, Precision, flip_bit, gemm, reduce_cols, reduce_rows, round_to

__version__ = "0.1.0"

__all__ = [
    "Matrix2D",
    "Precision",
    "flip_bit",
    "gemm",
    "reduce_cols",
    "reduce_rows",
    "round_to",
    "__version__",
]
