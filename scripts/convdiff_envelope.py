"""The reference algorithm's own sensitivity on the config-5 proxy
(convection-diffusion 40^3, s=5, m=60): relres change per restart when 50
entries of b move by one ulp (the C oracle, bit-identical to the reference).
Printed per scheme; the GPU test allows 10x the worst (tests/test_gpu_ops.py).
Measured: restarts 0-3 <= 5.8e-14, 2.6e-11, 1.8e-9, 5.6e-8."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / 'oracle')); sys.path.insert(0, str(ROOT))
import numpy as np
from py_oracle import Oracle
from paper_2503_16717_b200.borth import convdiff_coeffs
o=Oracle("orc")
csr=o.stencil_csr(40,3,convdiff_coeffs(0.3))
n=40**3
rng=np.random.default_rng(0)
for scheme in (0,1,2,3):
    base=o.sstep_gmres(csr,np.ones(n),np.zeros(n),m=60,s=5,shat=60,scheme=scheme,diagnostics=False).relres
    worst=np.zeros(len(base))
    for t in range(4):
        b=np.ones(n); idx=rng.integers(0,n,50); b[idx]=np.nextafter(1.0, 2.0 if t%2 else 0.0)
        r=o.sstep_gmres(csr,b,np.zeros(n),m=60,s=5,shat=60,scheme=scheme,diagnostics=False).relres
        worst=np.maximum(worst, np.abs(np.array(r)-np.array(base))/np.array(base))
    print(scheme, ["%.1e"%w for w in worst])
