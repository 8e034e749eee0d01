"""Per-phase cycle split of the pass kernels over the C2 sequence (diagnostic
library built with -DBO_PHASE_PROF=1, loaded through BO_LIB).
    BO_LIB=.../libbo_cuda_phase.so python scripts/prof_phases.py"""
import argparse
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_16717_b200 as P  # noqa: E402
from paper_2503_16717_b200 import _lib  # noqa: E402

n, k = 8_000_000, 11
ctx = P.Context(n, device=0)
torch.cuda.set_stream(ctx.stream)
panels = bench.make_panels(P, ctx, argparse.Namespace(s=k - 1, panels=6, kappa=1e2))
theta = P.SketchOperator.build(ctx, "gaussian", n, 10, 1)
st = P.BasisStore(ctx, 6 * k)
lib = ctx.lib
lib.bo_debug_phase_prof.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong)]
buf = (C.c_ulonglong * 256)()


ONLY = int(sys.argv[1]) if len(sys.argv) > 1 else -1  # record only panel ONLY (p = 11 * ONLY)


def step(rec=False):
    st.reset()
    for j, v in enumerate(panels):
        if rec and j == ONLY:
            torch.cuda.synchronize()
            lib.bo_debug_phase_prof(ctx.h, None)
        P.bcgs2(st, v, P.borth.RAND_CHOLQR, theta)
        if rec and j == ONLY:
            torch.cuda.synchronize()
            assert lib.bo_debug_phase_prof(ctx.h, buf) == 0


for _ in range(2):
    step()
torch.cuda.synchronize()
assert lib.bo_debug_phase_prof(ctx.h, None) == 0
lib.bo_debug_phase_prof(ctx.h, None)
if ONLY < 0:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    assert lib.bo_debug_phase_prof(ctx.h, buf) == 0
else:
    step(True)
names = {9: "P2_QTX", 10: "P2_UPD(_GRAM)_ST", 8: "P2_ST", 4: "P1_ST/P1_GRAM", 1: "QTX", 2: "UPD_*"}
ph = ["wfull", "wsolved", "upd", "updbar", "post+st", "contract", "wstore", "release", "S:wfull", "S:solve", "S:release"]
for shape in range(16):
    v = buf[shape * 16:(shape + 1) * 16]
    if not any(v):
        continue
    print(f"shape {shape} {names.get(shape, '?')}: cycles per tile per warp")
    for i, nm in enumerate(ph):
        cnt = v[12] if i >= 8 else v[11]
        if v[i] and cnt:
            print(f"   {nm:10s} {v[i] / cnt:8.0f}")
    if v[14]:
        print(f"   storer: store issue {v[13] / v[14]:8.0f}, upd+contract {v[15] / v[14]:8.0f}")
