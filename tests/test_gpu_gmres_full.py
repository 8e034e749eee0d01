"""s-step GMRES at the benchmarked configurations against full-size reference
runs (tests/golden/reference_big.json, tests/golden/make_golden_big.py over
oracle/_ref):
  config 3   laplace_3d(64) full solve and laplace_3d(200) (n = 8e6), 4 restart
             cycles, bcgs2 + RandCholQR, Gaussian sketch (bench.py's gmres leg)
  config 5   two-stage RandBCGS, s = 5, shat = m = 60 on the 200^3
             convection-diffusion operator, Gaussian (3 cycles, bench.py's c5
             leg) and CountGauss (2 cycles)
  (f)3       the per-restart cycle diagnostics ||I - Q^T Q|| and the Arnoldi
             residual (gmres.cpp:255-266) against the reference's values on
             configs 1 and 3.

Contract: identical restart and iteration counts, ledgers
and breakdown outcomes; relres within 10x the reference's own sensitivity
(tests/golden/reference_envelopes.json: 50 entries of b moved by one ulp),
floored at the north star's 1e-10.  The diagnostics are rounding-level
quantities (1e-15 .. 1e-11) whose exact values depend on summation order:
the Arnoldi residual must agree with the reference's within a factor of 2,
and ||I - Q^T Q|| must be no larger than twice the reference's (the
reference's sequential Gram sums add their own rounding; see _check)."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


def _big():
    p = GOLD / "reference_big.json"
    return json.loads(p.read_text()) if p.exists() else {}


def _env(name):
    p = GOLD / "reference_envelopes.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    return d.get(name, {}).get("relres_rel_change")


def _solve(gpu, n, make_op, **kw):
    ctx = gpu.Context(n)
    op = make_op(ctx)
    b, x0 = ctx.from_host(np.ones(n)), ctx.from_host(np.zeros(n))
    _, rep = gpu.sstep_gmres_solve(op, b, x0, **kw)
    op.close()
    ctx.close()
    return rep


def _check(rep, want, env, name, diag=True):
    assert rep["restarts"] == want["restarts"], (rep["restarts"], want["restarts"])
    assert rep["iterations"] == want["iterations"]
    assert rep["reduce"] == want["reduce"], (rep["reduce"], want["reduce"])
    assert rep["converged"] == want["converged"] and rep["breakdown"] == want["breakdown"]
    assert rep["breakdown_detail"] == want["detail"]
    deltas, tols = [], []
    for i, (g, w) in enumerate(zip(rep["restart_relres"], want["relres"])):
        e = env[min(i, len(env) - 1)] if env else 0.0
        tols.append(max(1e-10, 10.0 * e))
        deltas.append(abs(g - w) / abs(w))
    print(f"{name}: relres rel. deltas {' '.join('%.1e' % d for d in deltas)}")
    print(f"{name}: tolerances        {' '.join('%.1e' % t for t in tols)}")
    ratios = {}
    if diag and want.get("orth"):
        for key, mine in (("orth", "restart_orth_error"), ("arnoldi", "restart_arnoldi_resid")):
            ratios[key] = [g / w for g, w in zip(rep[mine], want[key]) if w > 0]
            print(f"{name}: {key} gpu/reference {' '.join('%.2f' % x for x in ratios[key])}")
    for i, (d, t) in enumerate(zip(deltas, tols)):
        assert d <= t, (name, i, d, t)
    # Arnoldi residual: same magnitude.  ||I - Q^T Q||: the GPU may only be
    # smaller.  The reference forms Q^T Q with sequential row sums, whose own
    # rounding (up to n eps / 2 when the terms share a sign, e.g. the constant
    # first basis vector of b = 1: 1.1e-12 at n = 1e4) dominates its value at
    # restart 0 (2.4e-13 vs 5e-16 here); the device Gram sums in a tree.
    for x in ratios.get("arnoldi", []):
        assert 0.5 <= x <= 2.0, ratios["arnoldi"]
    for x in ratios.get("orth", []):
        assert x <= 2.0, ratios["orth"]


def test_c3_64_randcholqr(gpu):
    want = _big().get("c3_64") or pytest.skip("fixture missing")
    rep = _solve(gpu, 64 ** 3, lambda c: gpu.Operator.laplace(c, 3, 64), m=60, s=10, shat=60,
                 scheme="bcgs2_randcholqr", sketch="gaussian", diagnostics=True)
    assert want["converged"] and want["restarts"] == 5 and want["iterations"] == 300  # SURVEY probe
    _check(rep, want, _env("c3_64"), "c3 64^3")


def test_c3_200_randcholqr(gpu):
    """config 3 at n = 8e6, the bench's 4 restart cycles"""
    want = _big().get("c3_200") or pytest.skip("fixture missing")
    rep = _solve(gpu, 200 ** 3, lambda c: gpu.Operator.laplace(c, 3, 200), m=60, s=10, shat=60,
                 scheme="bcgs2_randcholqr", sketch="gaussian", max_restarts=4, diagnostics=True)
    _check(rep, want, _env("c3_200"), "c3 200^3")


def test_c5_200_gaussian(gpu):
    want = _big().get("c5_200") or pytest.skip("fixture missing")
    rep = _solve(gpu, 200 ** 3, lambda c: gpu.Operator.convdiff(c, 200), m=60, s=5, shat=60,
                 scheme="twostage_randbcgs", sketch="gaussian", max_restarts=3, diagnostics=True)
    _check(rep, want, _env("c5_200"), "c5 200^3 gaussian")


def test_c5_200_countgauss(gpu):
    want = _big().get("c5_200_cg") or pytest.skip("fixture missing")
    rep = _solve(gpu, 200 ** 3, lambda c: gpu.Operator.convdiff(c, 200), m=60, s=5, shat=60,
                 scheme="twostage_randbcgs", sketch="countgauss", max_restarts=2, diagnostics=False)
    _check(rep, want, _env("c5_200"), "c5 200^3 countgauss", diag=False)


@pytest.mark.parametrize("scheme", ["cholqr2", "randcholqr", "twostage_pip", "twostage_randbcgs"])
def test_c1_cycle_diagnostics(gpu, scheme):
    """(f)3: per-restart ||I - Q^T Q|| and Arnoldi residual on config 1"""
    want = (_big().get("c1_diag") or pytest.skip("fixture missing"))[scheme]
    full = {"cholqr2": "bcgs2_cholqr2", "randcholqr": "bcgs2_randcholqr"}.get(scheme, scheme)
    rep = _solve(gpu, 100 ** 2, lambda c: gpu.Operator.laplace(c, 2, 100), m=60, s=5, shat=60, scheme=full,
                 sketch="gaussian", diagnostics=True)
    # the reference's own sensitivity (tests/test_gpu_ops.py C1_ENVELOPE / 10): the
    # 1e-10 floor applies through restart 5
    env = [1e-11, 1e-11, 1e-11, 1e-11, 1e-11, 1e-11, 5.2e-8, 3.0e-6, 9.1e-4, 1.7e-3]
    _check(rep, want, env, f"c1 {scheme}")
