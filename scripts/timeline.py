"""Device timeline of the C2 sequence (CUPTI activity records through
torch.profiler): every kernel and memcpy of a few deferred steps with its
start/end, so the gaps between launches (host enqueue, small copies, launch
latency) can be read off.  python scripts/timeline.py [--n N] [--steps 3] [--nccl1] [--verbose]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2503_16717_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8_000_000)
ap.add_argument("--s", type=int, default=10)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--verbose", action="store_true")
ap.add_argument("--nccl1", action="store_true",
                help="size-1 NCCL communicator: every reduction through ncclAllReduce + the unfused finalize "
                     "(the multi-rank code path on one GPU)")
a = ap.parse_args()
k = a.s + 1
ctx = P.Context(a.n, device=0, nccl_id=P.Context.nccl_unique_id() if a.nccl1 else None)
torch.cuda.set_stream(ctx.stream)
panels = bench.make_panels(P, ctx, argparse.Namespace(s=a.s, panels=6, kappa=1e2))
theta = P.SketchOperator.build(ctx, "gaussian", a.n, a.s, 1)
st = P.BasisStore(ctx, 6 * k)


def step():
    st.reset()
    for v in panels:
        P.bcgs2(st, v, P.borth.RAND_CHOLQR, theta, defer=True)
    st.sync()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(a.steps):
        step()
    torch.cuda.synchronize()

evs = []
for e in prof.events():
    if e.device_type.name == "CUDA":
        evs.append((e.time_range.start, e.time_range.end, e.name))
evs.sort()
t0 = evs[0][0]
kern = mem = gap = 0.0
prev_end = None
big_gaps = []
for s, e, nm in evs:
    d = e - s
    if "emcpy" in nm or "emset" in nm:
        mem += d
    else:
        kern += d
    if prev_end is not None:
        g = max(0.0, s - prev_end)
        gap += g
        if g > 5:
            big_gaps.append((g, nm[:60]))
    if a.verbose:
        print(f"{(s - t0):10.1f} {d:9.1f} gap {0 if prev_end is None else s - prev_end:7.1f}  {nm[:90]}")
    prev_end = max(e, prev_end or e)
span = evs[-1][1] - t0
print(f"{len(evs)} device records over {a.steps} steps: span {span / 1e3:.3f} ms, kernels {kern / 1e3:.3f} ms, "
      f"copies/sets {mem / 1e3:.3f} ms, idle gaps {gap / 1e3:.3f} ms  (per step {span / a.steps / 1e3:.3f} / "
      f"{kern / a.steps / 1e3:.3f} / {mem / a.steps / 1e3:.3f} / {gap / a.steps / 1e3:.3f})")
big_gaps.sort(reverse=True)
for g, nm in big_gaps[:25]:
    print(f"  gap {g:8.1f} us before {nm}")
