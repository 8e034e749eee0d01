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


@pytest.mark.parametrize("shat,seed", [(5, 11), (60, 3), (60, 987654321)])
def test_count_gauss_dense_stage_matches_reference(lib, orc, shat, seed):
    """The replicated count_gauss dense stage (mc x mhat; 7442 x 122 at
    shat = 60) equals the reference's stream entry for entry
    (sketch.cpp:91-95)."""
    import numpy as np
    mc, mh = 2 * (shat + 1) ** 2, 2 * (shat + 1)
    n = max(mc, mh) + 500  # (the oracle's dense-stage accessor wants n >= mc)
    want = orc.sketch_dense(orc.sketch_build(2, n, shat, seed).h)
    out = np.empty(mc * mh)
    lib.bo_debug_count_gauss_stage.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
    assert lib.bo_debug_count_gauss_stage(seed, mc, mh, out.ctypes.data) == 0
    assert want.shape == (mc, mh)
    assert np.array_equal(out.reshape((mc, mh), order="F"), want)


# ------------------------------------------------------------ MatrixMarket --
MM_CASES = {
    "general": "%%MatrixMarket matrix coordinate real general\n% comment\n\n3 4 5\n1 1 2.5\n3 4 -1e-3\n2 2 7\n"
               "1 3 0.125\n3 1 1e300\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 5\n1 1 4\n2 1 -1\n3 2 -1\n4 4 4\n4 3 -0.5\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 5\n1 2 0.1\n1 2 0.2\n2 1 3\n1 2 0.3\n2 2 1\n",
    "upper_banner": "%%MatrixMarket MATRIX Coordinate REAL General\n2 2 1\n2 2 1.5\n",
    "empty_rows": "%%MatrixMarket matrix coordinate real general\n5 5 2\n5 1 1\n1 5 2\n",
    "bad_banner": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "not_mm": "hello\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n3 x 1\n",
    "bad_entry": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 two 3\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n4 1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "empty": "",
}


def _ref_mm(ref, path):
    import ctypes as C
    f = ref.lib.ref_mm_read
    f.restype, f.argtypes = C.c_void_p, [C.c_char_p, C.c_char_p, C.c_size_t]
    msg = C.create_string_buffer(512)
    h = f(str(path).encode(), msg, 512)
    if not h:
        return None, msg.value.decode()
    nr, nc = C.c_size_t(), C.c_size_t()
    ref.lib.ref_csr_info.restype = C.c_size_t
    ref.lib.ref_csr_info.argtypes = [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
    nnz = ref.lib.ref_csr_info(h, C.byref(nr), C.byref(nc))
    rp = np.zeros(nr.value + 1, dtype=np.uint64)
    ci = np.zeros(nnz, dtype=np.uint64)
    vv = np.zeros(nnz)
    ref.lib.ref_csr_arrays.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_double)]
    ref.lib.ref_csr_arrays(h, rp.ctypes.data_as(C.POINTER(C.c_uint64)), ci.ctypes.data_as(C.POINTER(C.c_uint64)),
                           vv.ctypes.data_as(C.POINTER(C.c_double)))
    ref.lib.ref_csr_free.argtypes = [C.c_void_p]
    ref.lib.ref_csr_free(h)
    return (nr.value, nc.value, rp.astype(np.int64), ci.astype(np.int64), vv), None


@pytest.mark.parametrize("case", sorted(MM_CASES))
def test_matrix_market_read_matches_reference(ref, tmp_path, case):
    """bo_mm_read == the reference's read_matrix_market (sparse.cpp:88-136):
    identical CSR (sorted, symmetric mirrored, duplicates summed) or the
    identical error text"""
    import paper_2503_16717_b200 as P
    path = tmp_path / f"{case}.mtx"
    path.write_text(MM_CASES[case])
    want, err = _ref_mm(ref, path)
    if want is None:
        with pytest.raises(P.borth.Error) as ex:
            P.borth.read_matrix_market(path)
        assert str(ex.value) == err
        assert isinstance(ex.value, P.borth.ParseError if err.startswith("parse error") else P.borth.BannerError)
        return
    got = P.borth.read_matrix_market(path)
    assert got[:2] == want[:2]
    for a, b in zip(got[2:], want[2:]):
        assert np.array_equal(a, b)


def test_matrix_market_missing_file(ref, tmp_path):
    import paper_2503_16717_b200 as P
    _, err = _ref_mm(ref, tmp_path / "nope.mtx")
    with pytest.raises(P.borth.ParseError) as ex:
        P.borth.read_matrix_market(tmp_path / "nope.mtx")
    assert str(ex.value) == err and ex.value.line == 0


def test_matrix_market_write_matches_reference(ref, orc, tmp_path):
    """bo_mm_write == write_matrix_market byte for byte, and round-trips"""
    import ctypes as C

    import paper_2503_16717_b200 as P
    rp, ci, vv = orc.stencil_csr(6, 3, P.borth.convdiff_coeffs(0.3))
    vv = vv * np.pi  # 17-digit values
    n = len(rp) - 1
    P.borth.write_matrix_market(tmp_path / "ours.mtx", n, n, rp, ci, vv)
    h, keep = ref._csr_handle(rp, ci, vv, n)
    f = ref.lib.ref_mm_write
    f.restype, f.argtypes = C.c_int, [C.c_char_p, C.c_void_p, C.c_char_p, C.c_size_t]
    msg = C.create_string_buffer(256)
    assert f(str(tmp_path / "ref.mtx").encode(), h, msg, 256) == 0
    ref._csr_free(h)
    assert (tmp_path / "ours.mtx").read_bytes() == (tmp_path / "ref.mtx").read_bytes()
    got = P.borth.read_matrix_market(tmp_path / "ours.mtx")
    assert np.array_equal(got[2], rp) and np.array_equal(got[3], ci) and np.array_equal(got[4], vv)


def test_cost_model_matches_reference(ref):
    """(f)4: bo_cost_eval restates cost_model.cpp:38-111 exactly (integers and
    InvalidScheme texts), checked against the compiled reference's eval_cost"""
    import ctypes as C
    import paper_2503_16717_b200 as P
    f = ref.lib.ref_eval_cost
    f.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int64)]
    f.restype = C.c_int
    names = ["standard", "sstep", "sketch_eq_s", "sketch_between", "sketch_eq_m"]
    checked = 0
    for sc, name in enumerate(names):
        for n in (1, 7, 10_000, 8_000_000, 64_000_000):
            for m in (1, 7, 12, 60, 120):
                for s in (1, 2, 3, 5, 10, 12, 15):
                    for shat in (1, 4, 12, 30, 60):
                        for mhat in (0, 22, 45):
                            out = (C.c_int64 * 5)()
                            rc = f(sc, n, m, s, shat, mhat, out)
                            try:
                                got = P.eval_cost(name, n, m, s, shat, mhat)
                                assert rc == 0, (name, n, m, s, shat, mhat)
                                assert list(got.values()) == list(out), (name, n, m, s, shat, mhat)
                            except P.InvalidScheme as e:
                                assert rc != 0, (name, n, m, s, shat, mhat)
                                assert str(e) == ref.status()[1], (str(e), ref.status())
                            checked += 1
    assert checked > 10000
    assert P.eval_cost("sstep", 8_000_000, 60, 10)["latency"] == 24


# ------------------------------------------------------- C2 panel cache --
def test_sha256_matches_hashlib():
    import hashlib

    import paper_2503_16717_b200 as P
    rng = np.random.default_rng(3)
    for n in (0, 1, 55, 56, 63, 64, 65, 119, 1000, 1 << 20):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert P.borth.sha256(b) == hashlib.sha256(b.tobytes()).hexdigest(), n


def test_panel_cache_roundtrip_and_digest(tmp_path):
    """raw FP64 + SHA-256; the digest is that of
    the column-major payload, reading verifies it, corruption and shape
    mismatches fail loudly"""
    import hashlib

    import paper_2503_16717_b200 as P
    rng = np.random.default_rng(4)
    a = np.asfortranarray(rng.standard_normal((1003, 22)))
    path = tmp_path / "c2.bopc"
    sha = P.borth.panel_cache_write(path, a, "gen_glued(1003, 2, 11, 100, 100, 7)")
    assert sha == hashlib.sha256(a.tobytes(order="F")).hexdigest()
    info = P.borth.panel_cache_info(path)
    assert info == {"rows": 1003, "cols": 22, "sha256": sha, "desc": "gen_glued(1003, 2, 11, 100, 100, 7)"}
    b = P.borth.panel_cache_read(path)
    assert np.array_equal(a, b) and b.flags.f_contiguous
    raw = bytearray(path.read_bytes())
    raw[312 + 8 * 500] ^= 1  # one payload bit
    bad = tmp_path / "bad.bopc"
    bad.write_bytes(bytes(raw))
    with pytest.raises(P.borth.Error, match="SHA-256 mismatch"):
        P.borth.panel_cache_read(bad)
    with pytest.raises(P.borth.Error, match="holds 1003 x 22"):
        P.borth.panel_cache_read(path, np.empty((1003, 11), order="F"))
    bad.write_bytes(b"X" * 400)
    with pytest.raises(P.borth.Error, match="bad magic"):
        P.borth.panel_cache_info(bad)
    assert not (tmp_path / "c2.bopc.tmp").exists()  # written through a temporary, renamed at the end
