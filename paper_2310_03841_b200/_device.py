"""Host <-> device plumbing for the reference-compatible API.

The reference keeps every matrix as a NumPy array (``Matrix2D.data``,
numerics.py:127-160).  The B200 path computes on CUDA tensors; these helpers
move operands in the device storage type of each dtype tag and bring results
back in the reference's host storage type.  torch only owns memory and the
stream here — all arithmetic runs in libgemmguard_b200.so.

There is no CPU fallback: without a CUDA device every entry point raises
``GemmGuardLibraryError``.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import GemmGuardLibraryError

# dtype tag -> torch dtype of the DEVICE copy.  binary16-emulated values are
# float64 lattice values on the host (numerics.py:52-58) and real fp16 on the
# device (exact: every element round-trips through binary16).
DEVICE_DTYPE = {
    "binary64": torch.float64,
    "binary32": torch.float32,
    "binary16-emulated": torch.float16,
    "bfloat16": torch.bfloat16,  # extension, not a reference tag
    "int8": torch.int8,
    "int32": torch.int32,
}

# dtype tag -> NumPy dtype of the HOST copy (the reference's storage)
HOST_DTYPE = {
    "binary64": np.float64,
    "binary32": np.float32,
    "binary16-emulated": np.float64,
    "bfloat16": np.float64,
    "int8": np.int8,
    "int32": np.int32,
}


def device() -> torch.device:
    """The CUDA device of the calling thread; raises without one."""
    if not torch.cuda.is_available():
        raise GemmGuardLibraryError(
            "the protected-GEMM path runs on CUDA only (sm_100a); no CUDA device is visible"
        )
    return torch.device("cuda", torch.cuda.current_device())


def to_device(arr: np.ndarray, tag: str) -> torch.Tensor:
    """Host array holding `tag` values -> contiguous device tensor of DEVICE_DTYPE[tag]."""
    dev = device()
    a = np.ascontiguousarray(arr)
    if tag in ("binary16-emulated", "bfloat16"):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        return t.to(dev).to(DEVICE_DTYPE[tag])
    a = a.astype(HOST_DTYPE[tag], copy=False)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def to_host(t: torch.Tensor, tag: str) -> np.ndarray:
    """Device tensor -> host array in the reference storage type of `tag`."""
    if tag in ("binary16-emulated", "bfloat16"):
        return t.to(torch.float64).cpu().numpy()
    return t.cpu().numpy().astype(HOST_DTYPE[tag], copy=False)


def scalar_tensor(value, dtype: torch.dtype) -> torch.Tensor:
    return torch.tensor([value], dtype=dtype, device=device())
