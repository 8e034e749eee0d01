"""C3 GMRES phase timings + sketch-build timing (1 GPU).
python scripts/prof_gmres.py [--side 200] [--restarts 2]"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--side", type=int, default=200)
ap.add_argument("--s", type=int, default=10)
ap.add_argument("--restarts", type=int, default=2)
ap.add_argument("--sketch", default="gaussian")
ap.add_argument("--only-solve", action="store_true")
a = ap.parse_args()
n = a.side ** 3
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
if not a.only_solve:
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = P.SketchOperator.build(ctx, a.sketch, n, a.s, 100 + i)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        th.close()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"sketch build {a.sketch} n={n}: {1e3 * (t1 - t0):.3f} ms, destroy {1e3 * (t2 - t1):.3f} ms")
op = P.Operator.laplace(ctx, 3, a.side)
b = ctx.panel(1)
b[0, : ctx.n_local] = 1.0
x0 = ctx.panel(1)
for s in range(3):
    v = ctx.panel(a.s + 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(6):
        op.mpk(b, a.s, v)
    torch.cuda.synchronize()
    print(f"mpk s={a.s} x6: {1e3 * (time.perf_counter() - t0) / 6:.3f} ms per call")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, r = P.sstep_gmres_solve(op, b, x0, m=60, s=a.s, shat=60, scheme="bcgs2_randcholqr", sketch=a.sketch,
                               max_restarts=a.restarts, diagnostics=False)
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    print(f"solve {r['restarts']} restarts: {wall:.2f} ms wall, {wall / r['restarts']:.2f} ms/restart;",
          {k: round(v / r["restarts"], 3) for k, v in r["t_ms"].items()})
