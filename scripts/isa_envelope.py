"""The reference's own run-to-run envelope on config 1 (2D Laplace 100^2,
s=5, m=60): the same oracle/_ref binary with glibc's FMA vs non-FMA libm
variants (the Gaussian sketch changes by <= 1 ulp in ~0.06% of entries).
Prints per-restart relative relres differences per scheme; the GPU tests
allow 10x these (tests/test_gpu_ops.py).
    python scripts/isa_envelope.py ref > a.json
    GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA,-AVX512F python scripts/isa_envelope.py ref > b.json
Measured here (Xeon model 207, glibc 2.39): randbcgs 2.9e-13 7.8e-12 2.7e-11
4.2e-11 6.5e-11 5.7e-11 6.1e-09 3.6e-07 7.7e-04 1.3e-03."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / 'oracle'))
from py_oracle import Oracle
import numpy as np
o = Oracle(sys.argv[1])
csr = o.laplace(100, 2)
n = 10000
out = {}
for name, scheme, sk in [("cholqr2",0,0),("randcholqr",1,0),("pip",2,0),("randbcgs",3,0)]:
    r = o.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme, sketch=sk)
    out[name] = r.relres
print(json.dumps(out))
