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

SOURCES = ["bo_capi.cu", "bo_ops.cu", "bo_gmres.cu", "bo_glued.cu", "mt64_jump.cpp", "bo_io.cpp", "bo_cost.cpp",
           "bo_cache.cpp"]
# the pass-engine instantiation units: bo_pass_inst.cu compiled once per combination
INST_UNITS = [f"-DBO_INST_NT={nt} -DBO_INST_T={t}" for nt in (1, 2) for t in (256, 128, 64)] + \
             [f"-DBO_INST_KC={kc} -DBO_INST_T={t}" for kc in (6, 11, 13, 16) for t in (256, 128, 64)] + ["-DBO_INST_EXACT"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]
OBJ = PKG.parent / "build" / "obj"


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


def _units():
    """(object path, source, extra defines) for every compilation unit."""
    out = [(OBJ / (Path(s).stem + ".o"), CSRC / s, []) for s in SOURCES]
    for d in INST_UNITS:
        tag = d.replace("-DBO_INST_", "").replace("=", "").replace(" ", "_").lower()
        out.append((OBJ / f"bo_pass_inst_{tag}.o", CSRC / "bo_pass_inst.cu", d.split()))
    return out


def build_cuda(force: bool = False, verbose: bool = False, defines=(), tag: str = "") -> Path:
    """Compile every unit for sm_100a (in parallel), then link libbo_cuda.so.
    defines/tag: experiment variants (build/obj_<tag>, libbo_cuda_<tag>.so)."""
    obj_dir = OBJ if not tag else OBJ.parent / f"obj_{tag}"
    lib = LIB if not tag else PKG / f"libbo_cuda_{tag}.so"
    from concurrent.futures import ThreadPoolExecutor
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [INCLUDE / "bo_cuda.h"]
    obj_dir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    jobs = []
    units = [(obj_dir / o.name, src, defs) for o, src, defs in _units()]
    for obj, src, defs in units:
        if force or _stale(obj, [src, *headers]):
            jobs.append([nvcc, *NVCC_FLAGS, *defines, *defs, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=str(CSRC))

    if jobs:
        with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
            list(ex.map(run, jobs))
    objs = [str(o) for o, _, _ in units]
    if force or jobs or _stale(lib, objs):
        tmp = lib.with_suffix(".so.tmp")
        run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", str(tmp),
             *objs, "-ldl"])
        tmp.replace(lib)
    return lib


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
        # the reference, and the reference driver on the GPU path (needs libbo_cuda.so)
        subprocess.run(["make", "-s", "-C", str(odir), "ref"] + (["refgpu"] if LIB.exists() else []), check=True)


if __name__ == "__main__":
    build_cuda(verbose=True)
    build_examples()
    build_oracle(verbose=True)
