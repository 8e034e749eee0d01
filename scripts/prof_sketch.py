"""Gaussian / Count sketch build timing at n = 8e6 (device MT19937-64 stream +
correctly rounded Box-Muller): python scripts/prof_sketch.py [n] [shat] [kind]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
shat = int(sys.argv[2]) if len(sys.argv) > 2 else 10
kind = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
for _ in range(2):
    P.SketchOperator.build(ctx, kind, n, shat, 1).close()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record(ctx.stream)
for r in range(reps):
    P.SketchOperator.build(ctx, kind, n, shat, 2 + r).close()
e1.record(ctx.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
mh = 2 * (shat + 1) if kind == "gaussian" else 1
print(f"{kind} sketch n={n} shat={shat}: {ms:.3f} ms per build (incl. host plan + alloc), "
      f"{n * mh / (ms * 1e-3) / 1e9:.1f} G entries/s")
