"""Builds the C-ABI library ``libgemmguard_b200.so`` in-tree with nvcc.

The library is compiled for sm_100a only (``-gencode arch=compute_100a,
code=sm_100a``) with ``-lineinfo`` so ncu's source page maps to the .cu files.
Objects compile in parallel; the shared object links the CUDA runtime
statically so it loads in any process that has a driver (torch included).

    python -m paper_2310_03841_b200.build          # build if stale
    python -m paper_2310_03841_b200.build --force  # rebuild
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG / "_build"
LIB = PKG / "libgemmguard_b200.so"

SOURCES = ["gg_gemm_sm100.cu", "gg_aux.cu", "gg_calib.cu", "gg_toy.cu", "gg_vit.cu", "gg_locate.cu", "gg_capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libgemmguard_b200.so")
    return cand


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def _compile(src: str, verbose: bool) -> Path:
    obj = BUILD / (Path(src).stem + ".o")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = BUILD / (Path(src).stem + ".ptxas.log")
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr[-6000:]}")
    if verbose:
        sys.stdout.write(f"compiled {src}\n")
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source for sm_100a and link the C-ABI library."""
    if not force and not _stale():
        return LIB
    BUILD.mkdir(exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-6000:]}")
    os.replace(tmp, LIB)
    if verbose:
        sys.stdout.write(f"linked {LIB}\n")
    return LIB


def build_variant(name: str, defines: list[str]) -> Path:
    """Diagnostics / A-B build with extra preprocessor defines, linked to
    _variants/libgemmguard_b200_<name>.so; never loaded by the product (select it
    with $GEMMGUARD_LIB)."""
    BUILD.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = BUILD / f"{Path(src).stem}.{name}.o"
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *defines, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr[-6000:]}")
        objs.append(obj)
    out = PKG / "_variants" / f"libgemmguard_b200_{name}.so"
    out.parent.mkdir(exist_ok=True)
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs), "-lcuda"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-6000:]}")
    return out


def build_trace(verbose: bool = False) -> Path:
    """-DGG_TRACE: per-tile clock64 stamps of every warp role (tools/trace_tiles.py)."""
    return build_variant("trace", ["-DGG_TRACE", "-DGG_DIAGNOSTICS"])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--trace", action="store_true", help="also build the diagnostics library")
    ap.add_argument("--variant", nargs="+", metavar=("NAME", "DEFINE"),
                    help="also build _variants/libgemmguard_b200_NAME.so with -DDEFINE for each DEFINE")
    a = ap.parse_args()
    print(build(force=a.force, verbose=True))
    if a.trace:
        print(build_trace(verbose=True))
    if a.variant:
        print(build_variant(a.variant[0], [f"-D{d}" for d in a.variant[1:]]))
