"""Config 5 per-GPU share: two-stage s-step GMRES (s = 5, shat = m = 60) on the
3D convection-diffusion operator, n = side^3 rows (default 200^3 = 8e6, the
per-GPU share of 400^3 over 8 GPUs)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 200
n = side ** 3
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
op = P.Operator.convdiff(ctx, side, 0.3)
b = ctx.panel(1)
b[0, :n] = 1.0
x0 = ctx.panel(1)
for sk in ("gaussian", "countgauss"):
    for scheme in ("twostage_randbcgs", "twostage_pip", "bcgs2_randcholqr"):
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, r = P.sstep_gmres_solve(op, b, x0, m=60, s=5, shat=60, scheme=scheme, sketch=sk, max_restarts=2,
                                       diagnostics=False)
            torch.cuda.synchronize()
            wall = 1e3 * (time.perf_counter() - t0)
        print(f"{scheme:18s} {sk:10s} {wall / r['restarts']:.2f} ms/restart (incl. setup)",
              {k: round(v / r["restarts"], 2) for k, v in r["t_ms"].items()}, r["reduce"])
        if scheme.startswith("bcgs2") or scheme == "twostage_pip":
            if sk == "countgauss":
                break
