import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    from py_oracle import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from py_oracle import Oracle, have_ref
    if not have_ref():
        pytest.skip("reference build oracle/_ref unavailable (no /root/reference on this host)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def gpu():
    """the CUDA extension must load and a GPU must be present (no fallback)"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_16717_b200 as P
    P._lib.load()
    return P


@pytest.fixture(scope="session")
def ddm_host():
    """host build of the device double-double log / sincos (tests/native/ddmath_host.cpp)"""
    import ctypes as C
    src = ROOT / "tests" / "native" / "ddmath_host.cpp"
    hdrs = [ROOT / "paper_2503_16717_b200" / "csrc" / h for h in ("bo_ddmath.cuh", "bo_ddmath_tables.h")]
    so = ROOT / "tests" / "native" / "libddm_host.so"
    if not so.exists() or any(p.stat().st_mtime > so.stat().st_mtime for p in [src, *hdrs]):
        import subprocess
        subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", str(src), "-o", str(so)], check=True)
    lib = C.CDLL(str(so))
    dp = C.POINTER(C.c_double)
    for name in ("ddm_log_n", "glibc_log_n"):
        getattr(lib, name).argtypes = [dp, dp, C.c_long]
    for name in ("ddm_sincos_n", "glibc_sincos_n"):
        getattr(lib, name).argtypes = [dp, dp, dp, C.c_long]
    lib.box_muller_n.argtypes = [C.c_uint64, C.c_long, C.c_int, dp]
    lib.theta_cr.argtypes = [C.c_uint64, C.c_long, C.c_long, dp]
    return lib


def ulps(a, b):
    """|a - b| in units in the last place (same-sign finite doubles)"""
    return np.abs(np.asarray(a, dtype=np.float64).view(np.int64) - np.asarray(b, dtype=np.float64).view(np.int64))


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / den) if a.size else 0.0


def orth_err(q):
    q = np.asarray(q)
    g = q.T @ q
    return float(np.linalg.norm(np.eye(q.shape[1]) - g, 2))


def kappa_tol(kappa, floor=1e-10):
    """parity contract: max(1e-10, 10 kappa eps)"""
    return max(floor, 10.0 * kappa * 2.220446049250313e-16)


def ulp_sensitivity(run, x, draws=4, entries=50, seed=0):
    """The reference algorithm's own sensitivity at this input: the worst
    relative change of each output of run(x) (a tuple of arrays, computed by
    the CPU oracle, bit-identical to the reference) when `entries` entries of
    x move by one ulp, over `draws` draws.  A GPU result whose sums are
    merely ordered differently should stay within a small multiple of it."""
    base = [np.asarray(o) for o in run(x)]
    worst = [0.0] * len(base)
    rng = np.random.default_rng(seed)
    for t in range(draws):
        y = np.array(x, copy=True)
        flat = y.reshape(-1, order="F") if y.flags.f_contiguous else y.reshape(-1)
        idx = rng.integers(0, flat.size, entries)
        flat[idx] = np.nextafter(flat[idx], np.inf if t % 2 else -np.inf)
        for i, o in enumerate(run(y)):
            worst[i] = max(worst[i], rel_err(o, base[i]))
    return worst


def order_sensitivity(orc, run, x, chunks=(148, 1184)):
    """The reference algorithm's sensitivity to the summation order of its
    tall dot products: the worst relative change of each output of run(x)
    when the C oracle sums them in `chunks` contiguous runs instead of one
    (oracle.c tall_dot)."""
    base = [np.asarray(o) for o in run(x)]
    worst = [0.0] * len(base)
    try:
        for c in chunks:
            orc.set_sum_chunks(c)
            for i, o in enumerate(run(x)):
                worst[i] = max(worst[i], rel_err(o, base[i]))
    finally:
        orc.set_sum_chunks(0)
    return worst


def envelope(sens, factor=10.0, floor=1e-10):
    """parity tolerance from a measured sensitivity"""
    return max(floor, factor * sens)


def ref_envelopes(orc, run, x, factor=10.0):
    """per-output parity tolerances: `factor` x the worst of the reference's
    own one-ulp input sensitivity and summation-order sensitivity, floored at
    the north star's 1e-10; also returns the two sensitivities for printing"""
    su, so = ulp_sensitivity(run, x), order_sensitivity(orc, run, x)
    return [envelope(max(a, b), factor) for a, b in zip(su, so)], su, so
