"""In-tree build of the CUDA library (libbo_cuda.so) for sm_100a.

The .so is built next to this file so it travels with the repo snapshot to
the GPU box (a JIT cache under ~/.cache would not).  nvcc cross-compiles
without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libbo_cuda.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["bo_capi.cu", "bo_ops.cu", "bo_gmres.cu", "mt64_jump.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in SOURCES if (CSRC / s).exists()]
    deps += list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [INCLUDE / "bo_cuda.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    srcs = [str(CSRC / s) for s in SOURCES if (CSRC / s).exists()]
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", str(tmp), *srcs, "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    tmp.replace(LIB)
    return LIB


def build_examples() -> None:
    """C++ host program over the C ABI (examples/cpp_gmres.cpp)."""
    ex = PKG.parent / "examples"
    src = ex / "cpp_gmres.cpp"
    out = ex / "cpp_gmres"
    if not src.exists() or not _stale(out, [src, INCLUDE / "blkorth_gpu.hpp", INCLUDE / "bo_cuda.h", LIB]):
        return
    cuda = Path(_nvcc()).resolve().parents[1]
    cmd = ["g++", "-std=c++17", "-O2", f"-I{INCLUDE}", f"-I{cuda / 'include'}", str(src), "-o", str(out),
           f"-L{PKG}", "-lbo_cuda", f"-Wl,-rpath,{PKG}", f"-L{cuda / 'lib64'}", "-lcudart",
           f"-Wl,-rpath,{cuda / 'lib64'}"]
    subprocess.run(cmd, check=True)


def build_oracle(verbose: bool = False) -> None:
    """Build the parity checkers (oracle/ restatement and, when the reference
    sources are present, oracle/_ref).  Test infrastructure only."""
    odir = PKG.parent / "oracle"
    if not odir.exists():
        return
    subprocess.run(["make", "-s", "-C", str(odir), "all"], check=True)
    if Path("/root/reference/proj/src").exists():
        subprocess.run(["make", "-s", "-C", str(odir), "ref"], check=True)


if __name__ == "__main__":
    build_cuda(verbose=True)
    build_examples()
    build_oracle(verbose=True)
