"""Per-pass live timings of the intra-block factorizations on one 8e6 x 11
panel (cholqr, cholqr2, rand_cholqr): isolates the single-panel passes."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000, 11
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
v = torch.randn((k, ctx.ld), device="cuda", dtype=torch.float64)
v[:, n:] = 0
q = ctx.panel(k)
th = P.SketchOperator.build(ctx, "gaussian", n, k - 1, 1)
for name, fn in [("cholqr", lambda: P.cholqr(ctx, v, q=q)), ("cholqr2", lambda: P.cholqr2(ctx, v, q=q)),
                 ("rand_cholqr", lambda: P.rand_cholqr(ctx, v, th, q=q))]:
    for _ in range(3):
        fn()
    ctx.profile(True)
    for _ in range(5):
        fn()
    recs = ctx.profile_read()
    ctx.profile(False)
    torch.cuda.nvtx.range_push(name)
    fn()
    torch.cuda.nvtx.range_pop()
    ctx.synchronize()
    agg = {}
    for r in recs:
        a = agg.setdefault(r["kind"], [0.0, r["bytes"], 0])
        a[0] += r["ms"]
        a[2] += 1
    print(name, "  ".join(f"{kk}: {1e3 * a[0] / a[2]:.1f} us {a[1] / (a[0] / a[2]) / 1e6:.0f} GB/s"
                          for kk, a in agg.items()))
