"""Deferred bcgs2 (bo_bcgs2_enqueue + bo_basis_sync) against the synchronous
API, and run-to-run reproducibility.

  * a whole sequence enqueued and synced once gives bit-identical Q, R, C and
    ledgers to the call-by-call API (the device work is the same);
  * a breakdown in the middle of a deferred batch is reported for the right
    call, with the message, ledger and store state the synchronous API leaves
    when that call throws; the store keeps working afterwards;
  * mark_seed between deferred overlap calls (the GMRES panel loop) is
    replayed in program order;
  * the pass engine reduces in a fixed order: repeated runs are bitwise equal
    (C2 sequence, and a GMRES solve)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _glued(orc, n, panels, k, kappa, seed=7):
    return orc.gen_glued(n, panels, k, kappa, kappa, seed)


def _state(st):
    return st.basis_copy(), st.r_copy(), st.c_copy(), st.ledger().counts, st.cols()


@pytest.mark.parametrize("intra", [0, 1])
def test_deferred_sequence_bit_identical(gpu, orc, intra):
    n, k, panels = 30000, 11, 6
    v = _glued(orc, n, panels, k, 1e6)
    ctx = gpu.Context(n)
    try:
        th = gpu.SketchOperator.build(ctx, "gaussian", n, k - 1, 1) if intra else None
        dv = [ctx.from_host(v[:, p * k:(p + 1) * k]) for p in range(panels)]
        a = gpu.BasisStore(ctx, panels * k)
        for x in dv:
            gpu.bcgs2(a, x, intra, th)
        b = gpu.BasisStore(ctx, panels * k)
        for x in dv:
            gpu.bcgs2(b, x, intra, th, defer=True)
        assert b.cols() == panels * k  # speculative count before the sync
        b.sync()
        for x, y in zip(_state(a), _state(b)):
            assert np.array_equal(np.asarray(x), np.asarray(y))
    finally:
        ctx.close()


def test_deferred_breakdown_mid_batch(gpu, orc):
    """panel 2 has an exactly zero column: CholQR2 breaks down there"""
    n, k = 20000, 5
    v = _glued(orc, n, 4, k, 1e2)
    v[:, 2 * k + 2] = 0.0
    ctx = gpu.Context(n)
    try:
        dv = [ctx.from_host(v[:, p * k:(p + 1) * k]) for p in range(4)]
        seq = gpu.BasisStore(ctx, 4 * k)
        gpu.bcgs2(seq, dv[0], 0)
        gpu.bcgs2(seq, dv[1], 0)
        with pytest.raises(gpu.CholeskyBreakdown) as e_seq:
            gpu.bcgs2(seq, dv[2], 0)
        de = gpu.BasisStore(ctx, 4 * k)
        for x in dv:
            gpu.bcgs2(de, x, 0, defer=True)
        with pytest.raises(gpu.CholeskyBreakdown) as e_def:
            de.sync()
        assert e_def.value.call == 2
        assert str(e_def.value) == str(e_seq.value)
        for x, y in zip(_state(seq), _state(de)):
            assert np.array_equal(np.asarray(x), np.asarray(y))
        de.sync()  # nothing pending, the error was consumed
        gpu.bcgs2(de, dv[3], 0, defer=True)  # the store keeps working
        gpu.bcgs2(seq, dv[3], 0)
        de.sync()
        for x, y in zip(_state(seq), _state(de)):
            assert np.array_equal(np.asarray(x), np.asarray(y))
    finally:
        ctx.close()


def test_deferred_mark_seed_overlap(gpu, orc):
    """GMRES-shaped: each panel overlaps the last basis column, which is
    marked as the matrix-powers seed before the call (gmres.cpp:405-428)"""
    n, k = 25000, 6
    v = _glued(orc, n, 5, k, 1e3)
    ctx = gpu.Context(n)
    try:
        th = gpu.SketchOperator.build(ctx, "gaussian", n, k - 1, 3)
        dv = [ctx.from_host(v[:, p * k:(p + 1) * k]) for p in range(5)]
        a = gpu.BasisStore(ctx, 5 * k)
        b = gpu.BasisStore(ctx, 5 * k)
        for j, x in enumerate(dv):
            for st, defer in ((a, False), (b, True)):
                if j > 0:
                    st.mark_seed(st.cols() - 1)
                gpu.bcgs2(st, x, 1, th, overlap=j > 0, defer=defer)
        b.sync()
        for x, y in zip(_state(a), _state(b)):
            assert np.array_equal(np.asarray(x), np.asarray(y))
        assert [a.is_seed(c) for c in range(a.cols())] == [b.is_seed(c) for c in range(b.cols())]
    finally:
        ctx.close()


def test_c2_sequence_bitwise_reproducible(gpu, orc):
    """fixed-order reductions (bo_reduce.cuh): two runs, identical bits"""
    n, k = 200000, 11
    v = _glued(orc, n, 6, k, 1e6)
    ctx = gpu.Context(n)
    try:
        th = gpu.SketchOperator.build(ctx, "gaussian", n, k - 1, 1)
        dv = [ctx.from_host(v[:, p * k:(p + 1) * k]) for p in range(6)]
        runs = []
        for _ in range(2):
            st = gpu.BasisStore(ctx, 6 * k)
            for x in dv:
                gpu.bcgs2(st, x, 1, th)
            runs.append(_state(st))
            st.close()
        for x, y in zip(*runs):
            assert np.array_equal(np.asarray(x), np.asarray(y))
    finally:
        ctx.close()


def test_gmres_bitwise_reproducible(gpu):
    n = 40 ** 3
    outs = []
    for _ in range(2):
        ctx = gpu.Context(n)
        op = gpu.Operator.laplace(ctx, 3, 40)
        x, rep = gpu.sstep_gmres_solve(op, ctx.from_host(np.ones(n)), ctx.from_host(np.zeros(n)), m=60, s=10,
                                       shat=60, scheme="bcgs2_randcholqr", max_restarts=3)
        outs.append((ctx.to_host(x), rep["restart_relres"], rep["reduce"]))
        op.close()
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]


def test_import_ordered_before_next_pass(gpu):
    """bo_basis_import (the reference driver's store re-import after every
    restart and recover_panel) must land before the next pass reads the slab.
    A pageable cudaMemcpy on the legacy stream may return before its DMA is
    done and the non-blocking ctx stream does not wait for it; with 320 MB
    per import the projection right after it saw the old slab contents."""
    import ctypes as C

    from paper_2503_16717_b200 import _lib as L
    n, cols, k = 2_000_000, 20, 4
    ctx = gpu.Context(n)
    st = gpu.BasisStore(ctx, cols + k)
    rng = np.random.default_rng(5)
    v = ctx.from_host(rng.standard_normal((n, k)))
    vh = ctx.to_host(v)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    r = np.eye(cols)
    bounds = np.array([0, cols], dtype=np.uint64)
    for trial in range(4):
        q = np.asfortranarray(rng.standard_normal((n, cols)))
        stc = L.Status()
        rc = ctx.lib.bo_basis_import(st.h, cols, dp(q), n, dp(np.asfortranarray(r)), None, None,
                                     bounds.ctypes.data_as(C.POINTER(C.c_uint64)), 2, C.byref(stc))
        assert rc == 0
        got = gpu.borth.bcgs_project(st, v).coeffs
        want = q.T @ vh
        err = np.max(np.abs(got - want)) / np.max(np.abs(want))
        assert err < 1e-12, (trial, err)
    ctx.close()
