"""Per-launch live timings of the C2 sequence passes (CUDA events on the
library stream), grouped by (kind, p).  python scripts/prof_passes.py [--n N]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_16717_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8_000_000)
ap.add_argument("--s", type=int, default=10)
ap.add_argument("--intra", default="rand_cholqr")
ap.add_argument("--sketch", default="gaussian")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
k = a.s + 1
ctx = P.Context(a.n, device=0)
torch.cuda.set_stream(ctx.stream)
panels = bench.make_panels(P, ctx, argparse.Namespace(s=a.s, panels=6, kappa=1e2))
intra = P.borth.RAND_CHOLQR if a.intra == "rand_cholqr" else P.borth.CHOLQR2
theta = P.SketchOperator.build(ctx, a.sketch, a.n, a.s, 1) if intra == P.borth.RAND_CHOLQR else None
st = P.BasisStore(ctx, 6 * k)


def step():
    st.reset()
    for v in panels:
        P.bcgs2(st, v, intra, theta)


for _ in range(3):
    step()
ctx.profile(True)
for _ in range(a.reps):
    step()
recs = ctx.profile_read()
ctx.profile(False)
agg = {}
order = []
for r in recs:
    key = (r["kind"], r["p"])
    if key not in agg:
        agg[key] = [0.0, r["bytes"], 0]
        order.append(key)
    agg[key][0] += r["ms"]
    agg[key][2] += 1
tot = 0.0
for key in order:
    ms, b, c = agg[key]
    ms /= c
    tot += ms * c / a.reps
    print(f"{key[0]:>16s} p={key[1]:3d}  {ms * 1e3:8.1f} us  {b / 1e9:6.3f} GB  {b / ms / 1e6:7.0f} GB/s  x{c // a.reps}")
print(f"sum of passes per sequence: {tot:.3f} ms")
