"""Time the device gen_glued (n = 8e6, 6 x 11) and the Gaussian sketch build
(8e6 x 22, 8e6 x 122) on cuda:0.    python scripts/time_gen.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2503_16717_b200 as P  # noqa: E402

n = 8_000_000
ctx = P.Context(n)
t = time.time()
v = P.gen_glued(ctx, 6, 11, 1e6, 1e6, 7)
ctx.synchronize()
print(f"gen_glued 8e6 x 66: {time.time() - t:.2f} s", flush=True)
for shat in (10, 60):
    for rep in range(3):
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        th = P.SketchOperator.build(ctx, "gaussian", n, shat, 1 + rep)
        e1.record(ctx.stream)
        ctx.synchronize()
        print(f"gaussian build 8e6 x {2 * (shat + 1)}: {e0.elapsed_time(e1):.2f} ms", flush=True)
        th.close()
