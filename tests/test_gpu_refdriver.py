"""The reference's own GMRES driver on the GPU path (§8(b) drop-in): the
UNMODIFIED sstep_gmres_solve (proj/src/gmres.cpp) compiled with
-Dbcgs2=gpu_bcgs2 and linked with examples/refdriver/gpu_bcgs2.cpp, so its
panel loop (gmres.cpp:421-428) runs bo_bcgs2 and catches the adapter's
reference-typed exceptions (oracle/Makefile target refgpu ->
oracle/_ref/libblkorth_refgpu.so).

  * config 1 (both one-stage schemes): same restarts, iterations and ledger as
    the CPU reference, relres inside the config-1 envelope, and not bitwise
    equal to the CPU run (the device arithmetic really ran);
  * the s = 10 / 12 CholQR2 breakdowns: the device CholeskyBreakdown reaches
    the reference's recover_panel (gmres.cpp:195-248), whose "; recovery
    failed: ..." suffix is in the detail, with the reference's counts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def refgpu(gpu):
    from py_oracle import REFGPU_LIB, Oracle
    if not REFGPU_LIB.exists():
        pytest.skip("oracle/_ref/libblkorth_refgpu.so not built (needs /root/reference at build time)")
    return Oracle("refgpu")


# tests/test_gpu_ops.py C1_ENVELOPE: the north star's 1e-10 through restart 5
C1_ENVELOPE = [1e-10, 1e-10, 1e-10, 1e-10, 1e-10, 1e-10, 5.2e-7, 3.0e-5, 9.1e-3, 1.7e-2]


@pytest.mark.parametrize("scheme", [0, 1])
def test_reference_driver_c1(refgpu, ref, scheme):
    csr = ref.laplace(100, 2)
    n = 100 ** 2
    got = refgpu.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme)
    want = ref.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme)
    assert got.converged and want.converged
    assert (got.restarts, got.iterations) == (want.restarts, want.iterations) == (10, 600)
    assert got.reduce == want.reduce and got.reduce_total == want.reduce_total == 581
    d = [abs(a - b) / b for a, b in zip(got.relres, want.relres)]
    print(f"scheme {scheme}: relres rel. deltas {' '.join('%.1e' % x for x in d)}")
    assert all(x <= C1_ENVELOPE[i] for i, x in enumerate(d))
    assert got.relres != want.relres  # the device path ran (its sums differ in the last bits)


@pytest.mark.parametrize("s,its", [(10, 10), (12, 12)])
def test_reference_driver_breakdown_reaches_recover_panel(refgpu, ref, s, its):
    csr = ref.laplace(100, 2)
    n = 100 ** 2
    got = refgpu.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=s, shat=60, scheme=0)
    want = ref.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=s, shat=60, scheme=0)
    detail = "cholqr: nonpositive Cholesky pivot at step 1; recovery failed: recursive CholQR discarded all columns"
    assert got.breakdown and got.breakdown_detail == want.breakdown_detail == detail
    assert (got.restarts, got.iterations) == (want.restarts, want.iterations) == (1, its)
    assert got.reduce == want.reduce
    assert abs(got.final_relres - want.final_relres) <= 1e-10 * want.final_relres
