"""CPU: the C-ABI library (libbo_cuda.so) loads without a GPU, exports every
entry point declared in include/bo_cuda.h, fails loudly without a GPU (no CPU
fallback), and its host-side MT19937-64 jump-ahead reproduces the reference's
std::mt19937_64 stream at arbitrary offsets."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    txt = (ROOT / "include" / "bo_cuda.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bo_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import paper_2503_16717_b200 as P
    return P._lib.load()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    import paper_2503_16717_b200 as P
    bound = set(P._lib.exported_symbols())
    assert set(_declared()) - bound == set()


def test_abi_version(lib):
    assert lib.bo_abi_version() == 1


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2503_16717_b200 as P
    with pytest.raises(P.CudaError, match="no CPU fallback|no CUDA device"):
        P.Context(1000)


def _raw_stream(orc, seed, count):
    rng = orc.lib.orc_rng_new
    rng.restype = C.c_void_p
    rng.argtypes = [C.c_uint64]
    nxt = orc.lib.orc_rng_next_u64
    nxt.restype = C.c_uint64
    nxt.argtypes = [C.c_void_p]
    h = rng(seed)
    return [nxt(h) for _ in range(count)]


def _temper(y):
    m = (1 << 64) - 1
    y ^= (y >> 29) & 0x5555555555555555
    y ^= (y << 17) & 0x71D67FFFEDA60000 & m
    y ^= (y << 37) & 0xFFF7EEE000000000 & m
    y ^= y >> 43
    return y & m


@pytest.mark.parametrize("seed", [5489, 5095610196844313600, 1])
@pytest.mark.parametrize("J", [0, 1, 311, 312, 4097, 20000, 123457])
def test_mt64_jump_window_matches_stream(lib, orc, seed, J):
    out = (C.c_uint64 * 312)()
    assert lib.bo_mt64_jump_window(seed, J, out) == 0
    want = _raw_stream(orc, seed, J + 312)[J:]
    assert [_temper(x) for x in out] == want


def test_count_rows_from_jumped_window(lib, orc):
    """Shard-local regeneration: rows [a, a+156) of a Count sketch from the
    window at draw 2a equal the reference's rows."""
    n, shat, seed = 100000, 10, 77
    width = 2 * (shat + 1) ** 2
    h = orc.sketch_build(1, n, shat, seed).h
    bo, so = orc.sketch_count(h, n)
    mt_seed = orc.derive_seed(seed, 0)
    for a in (0, 1234, 49999, 99000):
        out = (C.c_uint64 * 312)()
        lib.bo_mt64_jump_window(mt_seed, 2 * a, out)
        draws = [_temper(x) for x in out]
        for t in range(156):
            u, sg = draws[2 * t], draws[2 * t + 1]
            assert (u * width) >> 64 == bo[a + t]
            assert (1.0 if sg & 1 else -1.0) == so[a + t]
