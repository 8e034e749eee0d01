"""SpMV / MPK timing on the 3D 7-point stencil (laplace_3d(200), n = 8e6)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 200
n = side ** 3
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
op = P.Operator.laplace(ctx, 3, side)
x = ctx.panel(1)
x.normal_()
v = ctx.panel(11)
for _ in range(3):
    op.mpk(x, 10, v)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream)
for _ in range(10):
    op.mpk(x, 10, v)
e1.record(ctx.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"mpk s=10 n={n}: {ms:.3f} ms per call, {ms / 10 * 1e3:.1f} us per SpMV, "
      f"{16 * n / (ms / 10 * 1e-3) / 1e9:.0f} GB/s (16 B/row)")
