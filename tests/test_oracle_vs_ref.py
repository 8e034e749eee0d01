"""CPU: the C restatement (oracle/oracle.c) is bit-identical to the reference
compiled from its own sources (oracle/_ref) on seeded random inputs, across
every routine of the hot path.  Skipped where oracle/_ref was never built."""
import numpy as np
import pytest


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("kind,n,shat,seed", [(0, 3000, 5, 1), (1, 3000, 5, 2), (2, 3000, 5, 3), (0, 500, 10, 9),
                                              (1, 800, 3, 12345678901234567)])
def test_sketch(orc, ref, kind, n, shat, seed):
    ho, hr = orc.sketch_build(kind, n, shat, seed).h, ref.sketch_build(kind, n, shat, seed).h
    if kind != 1:
        assert _eq(orc.sketch_dense(ho), ref.sketch_dense(hr))
    if kind != 0:
        bo, so = orc.sketch_count(ho, n)
        br, sr = ref.sketch_count(hr, n)
        assert _eq(bo, br) and _eq(so, sr)
    v = np.random.default_rng(seed % 1000).standard_normal((n, 6))
    assert _eq(orc.sketch_apply(ho, v), ref.sketch_apply(hr, v))


def test_ambient_too_small(orc, ref):
    a, b = orc.sketch_build(0, 22, 10, 1), ref.sketch_build(0, 22, 10, 1)
    assert a.h is None and b.h is None and a.code == b.code == 3 and a.msg == b.msg


@pytest.mark.parametrize("kappa", [1.0, 1e4, 1e9, 1e13])
def test_intra(orc, ref, kappa):
    v = orc.gen_glued(3000, 1, 8, kappa, kappa, 5)
    assert _eq(v, ref.gen_glued(3000, 1, 8, kappa, kappa, 5))
    for name in ("cholqr", "cholqr2"):
        a, b = getattr(orc, name)(v), getattr(ref, name)(v)
        assert a.code == b.code and a.msg == b.msg and a.ledger == b.ledger
        if a.code == 0:
            assert _eq(a.q, b.q) and _eq(a.r, b.r)
    so, sr = orc.sketch_build(0, 3000, 7, 4).h, ref.sketch_build(0, 3000, 7, 4).h
    a, b = orc.rand_cholqr(v, so), ref.rand_cholqr(v, sr)
    assert a.code == b.code and a.ledger == b.ledger and _eq(a.q, b.q) and _eq(a.r, b.r)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_recursive(orc, ref, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((2000, 7))
    v[:, 3] = v[:, 0] - 2 * v[:, 1]
    if seed == 2:
        v[:, 5] = 0.0
    a, b = orc.recursive_cholqr(v), ref.recursive_cholqr(v)
    assert a.code == b.code and a.kept == b.kept and a.discarded == b.discarded and a.depth == b.depth
    assert a.ledger == b.ledger and _eq(a.q, b.q) and _eq(a.coeffs, b.coeffs) and a.discard_norm == b.discard_norm


@pytest.mark.parametrize("intra", [0, 1])
@pytest.mark.parametrize("overlap", [False, True])
def test_bcgs2_sequences(orc, ref, intra, overlap):
    n, k = 2500, 6
    v = orc.gen_glued(n, 5, k, 1e5, 1e7, 3)
    so, sr = orc.sketch_build(0, n, k - 1, 8).h, ref.sketch_build(0, n, k - 1, 8).h
    bo, br = orc.basis_new(n, 5 * k), ref.basis_new(n, 5 * k)
    for p in range(5):
        vp = v[:, p * k:(p + 1) * k]
        ra = orc.bcgs2(bo, vp, intra, so if intra else None, overlap and p > 0)
        rb = ref.bcgs2(br, vp, intra, sr if intra else None, overlap and p > 0)
        assert ra.code == rb.code and ra.msg == rb.msg
    qa, _, la = orc.basis_state(bo, n)
    qb, rb_, lb = ref.basis_state(br, n)
    assert la == lb and _eq(qa, qb)
    assert _eq(orc.basis_r(bo, 5 * k), rb_)
    for kk in range(orc.basis_cols(bo)):
        assert _eq(orc.basis_input_coeff_col(bo, kk, 5), ref.basis_input_coeff_col(br, kk, 5))


def test_pip_randbcgs_two_stage(orc, ref):
    n, k = 3000, 5
    v = orc.gen_glued(n, 12, k, 1e3, 1e8, 23)
    so, sr = orc.sketch_build(0, n, 30, 29).h, ref.sketch_build(0, n, 30, 29).h
    for pre in (0, 1):
        bo, br = orc.basis_new(n, 61), ref.basis_new(n, 61)
        for big in range(2):
            orc.basis_begin_big_panel(bo, 62 if pre else 0, 0)
            ref.basis_begin_big_panel(br, 62 if pre else 0, 0)
            for p in range(6):
                vp = v[:, (big * 6 + p) * k:(big * 6 + p + 1) * k]
                ra = orc.two_stage_panel(bo, vp, pre, so if pre else None)
                rb = ref.two_stage_panel(br, vp, pre, sr if pre else None)
                assert ra.code == rb.code and ra.msg == rb.msg
            fa, fb = orc.two_stage_finish(bo, pre, True, True), ref.two_stage_finish(br, pre, True, True)
            assert fa.code == fb.code
        qa, _, la = orc.basis_state(bo, n)
        qb, rb_, lb = ref.basis_state(br, n)
        assert la == lb and _eq(qa, qb) and _eq(orc.basis_r(bo, 61), rb_)
        if pre:
            assert _eq(orc.basis_sketched(bo), ref.basis_sketched(br))


@pytest.mark.parametrize("dims,k", [(2, 17), (3, 9)])
def test_sparse(orc, ref, dims, k):
    a, b = orc.laplace(k, dims), ref.laplace(k, dims)
    for x, y in zip(a, b):
        assert _eq(x, y)
    v0 = np.random.default_rng(k).standard_normal(len(a[0]) - 1)
    assert _eq(orc.spmv(a, v0), ref.spmv(b, v0))
    assert _eq(orc.mpk(a, v0, 6), ref.mpk(b, v0, 6))


@pytest.mark.parametrize("scheme,s", [(0, 5), (1, 5), (2, 5), (3, 5), (0, 10), (1, 10), (3, 10)])
def test_gmres(orc, ref, scheme, s):
    csr = orc.laplace(40, 2)
    n = 1600
    b = np.ones(n)
    a = orc.sstep_gmres(csr, b, np.zeros(n), m=60, s=s, shat=60, scheme=scheme, max_restarts=12, diagnostics=False)
    c = ref.sstep_gmres(csr, b, np.zeros(n), m=60, s=s, shat=60, scheme=scheme, max_restarts=12)
    assert (a.converged, a.breakdown, a.breakdown_detail) == (c.converged, c.breakdown, c.breakdown_detail)
    assert (a.restarts, a.iterations, a.reduce, a.reduce_total) == (c.restarts, c.iterations, c.reduce, c.reduce_total)
    assert a.relres == c.relres and a.lsq == c.lsq
    assert _eq(a.x, c.x)
