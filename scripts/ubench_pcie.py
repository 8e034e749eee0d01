"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone and
both directions at once (the e2e leg of bench.py is bound by these)."""
import time

import torch

nbytes = 704_000_000  # one 8e6 x 11 FP64 panel
h_in = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return reps * nbytes * (h2d + d2h) / dt / 1e9


for _ in range(2):
    run(1, 1, 2)
print(f"H2D {run(1, 0):.1f} GB/s, D2H {run(0, 1):.1f} GB/s, both {run(1, 1):.1f} GB/s aggregate")
