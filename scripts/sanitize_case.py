"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
one config-1 GMRES restart for each one-stage scheme and the two-stage
RandBCGS, a six-panel bcgs2 sequence (both intras, deferred), a Count-sketch
sequence, and the matrix powers (2-D 4-row kernel, 3-D plane-marching kernel).  Exits non-zero on any library error.
    compute-sanitizer --tool racecheck python scripts/sanitize_case.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_2503_16717_b200 as P  # noqa: E402
from py_oracle import Oracle  # noqa: E402

orc = Oracle("orc")
n = 10000
ctx = P.Context(n)
op = P.Operator.laplace(ctx, 2, 100)
b, x0 = ctx.from_host(np.ones(n)), ctx.from_host(np.zeros(n))
for scheme in ("bcgs2_cholqr2", "bcgs2_randcholqr", "twostage_randbcgs"):
    _, rep = P.sstep_gmres_solve(op, b, x0, m=60, s=5, shat=60, scheme=scheme, max_restarts=1)
    print(scheme, rep["restarts"], rep["iterations"], rep["restart_relres"])
k = 11
v = orc.gen_glued(n, 6, k, 1e6, 1e6, 7)
dv = [ctx.from_host(v[:, p * k:(p + 1) * k]) for p in range(6)]
for intra, sk in ((0, None), (1, "gaussian"), (1, "count")):
    th = P.SketchOperator.build(ctx, sk, n, k - 1, 1) if sk else None
    st = P.BasisStore(ctx, 6 * k)
    for x in dv:
        P.bcgs2(st, x, intra, th, defer=True)
    st.sync()
    q = st.basis_copy()
    print("bcgs2", intra, sk, "orth", float(np.linalg.norm(np.eye(6 * k) - q.T @ q, 2)))
vk = ctx.to_host(op.mpk(ctx.from_host(np.random.default_rng(0).standard_normal(n)), 5))
print("mpk", float(np.abs(vk).max()))
# the plane-marching 3-D stencil kernel (bulk-copy plane ring, mbarriers):
# 3-D Laplace and convection-diffusion, bit-exact against the CSR kernel
n3 = 24 ** 3
ctx3 = P.Context(n3)
x3 = ctx3.from_host(np.random.default_rng(1).standard_normal(n3))
for mk in (lambda c: P.Operator.laplace(c, 3, 24), lambda c: P.Operator.convdiff(c, 24)):
    o3 = mk(ctx3)
    y = ctx3.to_host(o3.mpk(x3, 5))
    print("mpk 3-D", float(np.abs(y).max()))
ctx3.synchronize()
ctx.synchronize()
print("sanitize case ok")
