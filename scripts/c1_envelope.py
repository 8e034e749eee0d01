"""The reference algorithm's own sensitivity on config 1 (2D Laplace 100^2,
s=5, m=60): per-restart relres change when 50 entries of b move by one ulp
(the C oracle, bit-identical to the reference), worst over D draws, per scheme.
    python scripts/c1_envelope.py [--draws D] [s ...]   (default D = 4, s = 5)
The GPU tests allow 10x max(this, the reorder / libm envelopes of SURVEY App. B)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
from py_oracle import Oracle  # noqa: E402

o = Oracle("orc")
csr = o.laplace(100, 2)
n = 100 ** 2
rng = np.random.default_rng(0)
args = sys.argv[1:]
draws = 4
if args[:1] == ["--draws"]:
    draws, args = int(args[1]), args[2:]
svals = [int(a) for a in args] or [5]
for s in svals:
    for scheme in ((0, 1, 2, 3) if s == 5 else (0, 1)):
        base = np.array(o.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=s, shat=60, scheme=scheme,
                                      diagnostics=False).relres)
        worst = np.zeros(len(base))
        for t in range(draws):
            b = np.ones(n)
            b[rng.integers(0, n, 50)] = np.nextafter(1.0, 2.0 if t % 2 else 0.0)
            r = np.array(o.sstep_gmres(csr, b, np.zeros(n), m=60, s=s, shat=60, scheme=scheme,
                                       diagnostics=False).relres)
            m = min(len(r), len(base))
            worst[:m] = np.maximum(worst[:m], np.abs(r[:m] - base[:m]) / base[:m])
        print(f"s={s} scheme={scheme}", " ".join("%.1e" % w for w in worst))
