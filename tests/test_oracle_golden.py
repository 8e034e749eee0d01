"""CPU: the C oracle (oracle/oracle.c) reproduces every golden value generated
from the reference itself (tests/golden/reference_kats.json, made by
tests/golden/make_golden.py over oracle/_ref) and the SPEC.md examples."""
import json
from pathlib import Path

import numpy as np
import pytest

G = json.loads((Path(__file__).parent / "golden" / "reference_kats.json").read_text())


def test_derive_seed(orc):
    for key, val in G["derive_seed"].items():
        b, s = (int(x) for x in key.split(","))
        assert orc.derive_seed(b, s) == int(val)


def test_mt19937_64_standard_check(orc):
    """[rand.predef]: the 10000th output of a default-constructed mt19937_64"""
    import ctypes as C
    rng = orc.lib.orc_rng_new
    rng.restype = C.c_void_p
    rng.argtypes = [C.c_uint64]
    nxt = orc.lib.orc_rng_next_u64
    nxt.restype = C.c_uint64
    nxt.argtypes = [C.c_void_p]
    h = rng(5489)
    v = 0
    for _ in range(10000):
        v = nxt(h)
    assert v == int(G["mt19937_64_seed5489_draw10000"]) == 9981545732273789042
    h = rng(orc.derive_seed(7960286522194355700, 0))
    assert [nxt(h) for _ in range(16)] == [int(x) for x in G["mt_draws_first16_seed_cycle0"]]


def test_count_sketch_kats(orc):
    sk = G["sketch"]
    b, s = orc.sketch_count(orc.sketch_build(1, 1000, 10, 0).h, 1000)
    assert [[int(b[i]), int(s[i])] for i in range(8)] == sk["count_n1000_s10_seed0_rows0_7"]


@pytest.mark.slow
def test_count_sketch_kats_8e6(orc):
    sk = G["sketch"]["count_n8e6_s10_seed_cycle0"]
    h = orc.sketch_build(1, 8_000_000, 10, orc.derive_seed(0, 1)).h
    b, s = orc.sketch_count(h, 8_000_000)
    for i, (bb, ss) in sk.items():
        assert (int(b[int(i)]), int(s[int(i)])) == (bb, ss)
    orc.sketch_free(h)


def test_gaussian_sketch_kats(orc):
    sk = G["sketch"]
    d = orc.sketch_dense(orc.sketch_build(0, 1000, 10, 0).h)
    assert d[:4, 0].tolist() == sk["gauss_n1000_s10_seed0_col0_rows0_3"]
    assert d[0, 1] == sk["gauss_n1000_s10_seed0_r0c1"]
    d = orc.sketch_dense(orc.sketch_build(2, 5000, 5, 11).h)
    assert d[0, :6].tolist() == sk["countgauss_n5000_s5_seed11_dense_r0"]


def test_spec_dense_examples(orc):
    sp = G["spec"]
    assert orc.gram(np.array([[1.0, 0], [0, 1], [0, 0]])).tolist() == sp["gram_e1e2"] == [[1, 0], [0, 1]]
    r, f, _ = orc.cholesky(np.array([[4.0, 2], [2, 5]]))
    assert f == 0 and r.tolist() == sp["cholesky_4_2_5"]["r"] == [[2, 1], [0, 2]]
    r, f, piv = orc.cholesky(np.array([[1.0, 1], [1, 1]]))
    assert f == sp["cholesky_rank1"]["failed_at"] == 2
    q, r = orc.householder_qr(np.array([[3.0], [4.0]]))
    assert r.tolist() == sp["hhqr_3_4"]["r"] == [[5.0]]
    assert q[:, 0].tolist() == sp["hhqr_3_4"]["q"]
    assert np.allclose(q[:, 0], [0.6, 0.8], rtol=0, atol=2e-16)
    x = orc.apply_inv_upper(np.array([[3.0], [4.0]]), np.array([[5.0]])).x
    assert x[:, 0].tolist() == sp["apply_inv_upper_3_4_5"] == [0.6, 0.8]
    assert orc.apply_inv_upper(np.ones((2, 2)), np.array([[1.0, 0], [0, 0]])).code == 2


def test_spmv_spec(orc):
    y = orc.spmv((np.array([0, 2, 5, 7]), np.array([0, 1, 0, 1, 2, 1, 2]), np.array([2.0, -1, -1, 2, -1, -1, 2])),
                 np.ones(3))
    assert y.tolist() == G["spmv_tridiag"] == [1.0, 0.0, 1.0]


def test_glued_sweep(orc):
    """SURVEY App. A glued one-stage sweep: panels done, ledger, breakdown step/message."""
    th = orc.sketch_build(0, 10000, 4, 17).h
    for kap_s, row in G["glued_sweep_n1e4_12x5_seed11"].items():
        kap = float(kap_s)
        v = orc.gen_glued(10000, 12, 5, kap, kap, 11)
        for intra, name in ((0, "cholqr2"), (1, "randcholqr")):
            bb = orc.basis_new(10000, 60)
            done, msg = 0, ""
            for p in range(12):
                res = orc.bcgs2(bb, v[:, p * 5:(p + 1) * 5], intra, th if intra else None)
                if res.code:
                    msg = res.msg
                    break
                done += 1
            want = row[name]
            assert done == want["panels"] and msg == want["msg"], (kap, name)
            assert orc.basis_ledger(bb) == want["ledger"]
            if done == 12:
                q, _, _ = orc.basis_state(bb, 10000)
                assert abs(np.linalg.norm(np.eye(60) - q.T @ q, 2) - want["orth"]) < 1e-15
            orc.basis_free(bb)


@pytest.mark.parametrize("name", ["c1_cholqr2", "c1_randcholqr", "c1_twostage_pip", "c1_twostage_randbcgs",
                                  "s10_cholqr2", "s12_cholqr2", "s15_cholqr2"])
def test_gmres_kats(orc, name):
    want = G["gmres_2d100"][name]
    scheme = {"cholqr2": 0, "randcholqr": 1, "twostage_pip": 2, "twostage_randbcgs": 3}[name.split("_", 1)[1]]
    s = {"c1": 5, "s10": 10, "s12": 12, "s15": 15}[name.split("_")[0]]
    csr = orc.laplace(100, 2)
    res = orc.sstep_gmres(csr, np.ones(10000), np.zeros(10000), m=60, s=s, shat=60, scheme=scheme,
                          diagnostics=False)
    assert res.converged == want["converged"]
    assert res.breakdown == want["breakdown"]
    assert res.breakdown_detail == want["detail"]
    assert (res.restarts, res.iterations) == (want["restarts"], want["iterations"])
    assert res.reduce == want["reduce"] and res.reduce_total == want["reduce_total"]
    assert res.relres == want["relres"]  # bit-identical histories
    assert res.final_relres == want["final_relres"]


@pytest.mark.parametrize("name,scheme", [("cholqr2", 0), ("randcholqr", 1), ("twostage_pip", 2),
                                         ("twostage_randbcgs", 3)])
def test_gmres_convdiff40_kats(orc, name, scheme):
    """config-5 proxy: the C oracle on the stencil CSR reproduces the
    reference's histories bit for bit"""
    import paper_2503_16717_b200.borth as B
    want = G["gmres_convdiff40"][name]
    csr = orc.stencil_csr(40, 3, B.convdiff_coeffs(0.3))
    n = 40 ** 3
    res = orc.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme, diagnostics=False)
    assert (res.restarts, res.iterations) == (want["restarts"], want["iterations"])
    assert res.reduce == want["reduce"]
    assert res.relres == want["relres"]


def test_stencil_csr_is_from_triplets_csr(orc):
    """the test-side stencil generator emits exactly the CSR from_triplets
    builds, and reproduces laplace_3d / laplace_2d (problems.cpp:65-113)"""
    import paper_2503_16717_b200.borth as B
    for k, dims, c in [(7, 3, B.convdiff_coeffs(0.3)), (9, 2, [-1, -2, 5, -3, -4])]:
        csr = orc.stencil_csr(k, dims, c)
        assert all(np.array_equal(a, b) for a, b in zip(csr, orc.csr_from_triplets(*csr)))
    for k, dims in [(12, 3), (15, 2)]:
        lap = orc.laplace(k, dims)
        c = [-1.0] * dims + [2.0 * dims] + [-1.0] * dims
        assert all(np.array_equal(a, b) for a, b in zip(lap, orc.stencil_csr(k, dims, c)))
