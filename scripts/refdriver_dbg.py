"""Reference GMRES driver on the GPU path (oracle/_ref/libblkorth_refgpu.so):
relres history next to the CPU reference, for several solves in one process.
    python scripts/refdriver_dbg.py [scheme ...]   (default: 0 1 1 0)"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))
import paper_2503_16717_b200 as P  # noqa: E402
from py_oracle import Oracle  # noqa: E402

P._lib.load()
ref, refgpu = Oracle("ref"), Oracle("refgpu")
csr = ref.laplace(100, 2)
n = 100 ** 2
for scheme in [int(a) for a in sys.argv[1:]] or [0, 1, 1, 0]:
    got = refgpu.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme)
    want = ref.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme)
    print("scheme", scheme, "restarts", got.restarts, want.restarts, "reduce", got.reduce, want.reduce)
    print(" got ", " ".join("%.6e" % x for x in got.relres))
    print(" want", " ".join("%.6e" % x for x in want.relres))
