"""Per-launch device timings of the pass kernels inside one config-5 restart
cycle (two-stage RandBCGS, Gaussian sketch, 200^3 convection-diffusion),
grouped by (kind, p).   python scripts/prof_c5_passes.py [side] [sketch]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sk = sys.argv[2] if len(sys.argv) > 2 else "gaussian"
n = side ** 3
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
op = P.Operator.convdiff(ctx, side, 0.3)
b = ctx.panel(1)
b[0, :n] = 1.0
x0 = ctx.panel(1)
kw = dict(m=60, s=5, shat=60, scheme="twostage_randbcgs", sketch=sk, diagnostics=False)
P.sstep_gmres_solve(op, b, x0, max_restarts=1, **kw)
torch.cuda.synchronize()
ctx.profile(True)
_, r = P.sstep_gmres_solve(op, b, x0, max_restarts=1, **kw)
torch.cuda.synchronize()
recs = ctx.profile_read()
ctx.profile(False)
agg, order = {}, []
for q in recs:
    key = (q["kind"], q["p"])
    if key not in agg:
        agg[key] = [0.0, q["bytes"], 0]
        order.append(key)
    agg[key][0] += q["ms"]
    agg[key][2] += 1
tot = 0.0
for key in order:
    ms, by, c = agg[key]
    tot += ms
    print(f"{key[0]:>16s} p={key[1]:3d}  {ms / c * 1e3:8.1f} us  {by / 1e9:6.3f} GB  {by / (ms / c) / 1e6:7.0f} GB/s  x{c}")
print(f"sum of passes: {tot:.3f} ms; report t_ms {r['t_ms']}; restarts {r['restarts']}")
