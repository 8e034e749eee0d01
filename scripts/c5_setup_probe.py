"""Host wall time of a config-5 solve against its device restart-cycle time
(setup / teardown outside the cycles), for several restart counts.
    python scripts/c5_setup_probe.py"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

n = 200 ** 3
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
op = P.Operator.convdiff(ctx, 200, 0.3)
b = ctx.panel(1)
b[0, :n] = 1.0
x0 = ctx.panel(1)
kw = dict(m=60, s=5, shat=60, scheme="twostage_randbcgs", sketch="gaussian", rel_tol=1e-6, seed=0, diagnostics=False)
for r in [int(a) for a in sys.argv[1:]] or [1, 1, 2, 3, 1, 3]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = P.sstep_gmres_solve(op, b, x0, max_restarts=r, **kw)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) * 1e3
    c = rep["t_ms"]["cycles"]
    print(f"restarts={r}: wall {t:7.1f} ms, cycles {c:7.1f} ms, outside {t - c:6.1f} ms, sketch {rep['t_ms']['sketch']:.1f}")
