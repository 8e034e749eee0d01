#!/usr/bin/env python
"""Full-size reference runs for the configurations bench.py times
(tests/golden/reference_big.json).  Generated from the UNMODIFIED reference
(oracle/_ref/libblkorth_ref.so) in the build container, where /root/reference
exists; the GPU tests and the bench compare against the committed JSON.

    python tests/golden/make_golden_big.py [section ...]

Sections (each is merged into the JSON as it finishes, so they can be run
separately):
  c3_64      laplace_3d(64), s=10, m=60, bcgs2 + RandCholQR (Gaussian), full solve
             with the per-restart diagnostics (gmres.cpp:255-266)
  c3_200     config 3: laplace_3d(200) (n = 8e6), same scheme, the first 4
             restart cycles (bench.py's gmres leg runs 1 + 3)
  c5_200     config 5 at 200^3: two-stage RandBCGS, s=5, shat=m=60, Gaussian
             (mhat = 122), convection-diffusion w = 0.3, 3 restart cycles
             (bench.py's c5 leg)
  c5_200_cg  the same with the CountGauss sketch, 2 restart cycles
  c1_diag    config 1 (2D 100^2, s=5) per-restart ||I-Q^TQ|| and Arnoldi
             residual for the four schemes
  env_<section>  the reference's own sensitivity for that section: the worst
             per-restart relative relres change over `draws` runs with 50
             entries of b moved by one ulp (the method of scripts/c1_envelope.py;
             written to reference_envelopes.json).  The GPU tests allow 10x
             this, floored at the north star's 1e-10.

Gaussian-sketch histories go through glibc 2.39 log/sin/cos and so carry the
host's libm ifunc variant (this container selects the FMA variant, as the B200
box hosts do; SURVEY.md finding 1).
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))
from py_oracle import Oracle  # noqa: E402

PATH = Path(__file__).resolve().parent / "reference_big.json"


def kat(res, secs):
    return {"converged": res.converged, "breakdown": res.breakdown, "detail": res.breakdown_detail,
            "restarts": res.restarts, "iterations": res.iterations, "final_relres": res.final_relres,
            "reduce": res.reduce, "reduce_total": res.reduce_total, "relres": res.relres, "lsq": res.lsq,
            "orth": res.orth, "arnoldi": res.arnoldi, "cpu_seconds": secs}


def run(r, csr, n, secs_label=None, **kw):
    t = time.time()
    res = r.sstep_gmres(csr, np.ones(n), np.zeros(n), **kw)
    return kat(res, time.time() - t)


def section(r, name):
    from paper_2503_16717_b200.borth import convdiff_coeffs
    if name == "c3_64":
        return run(r, r.laplace(64, 3), 64 ** 3, m=60, s=10, shat=60, scheme=1, sketch=0, diagnostics=True)
    if name == "c3_200":
        return run(r, r.laplace(200, 3), 200 ** 3, m=60, s=10, shat=60, scheme=1, sketch=0, max_restarts=4,
                   diagnostics=True)
    if name == "c5_200":
        return run(r, r.stencil_csr(200, 3, convdiff_coeffs(0.3)), 200 ** 3, m=60, s=5, shat=60, scheme=3,
                   sketch=0, max_restarts=3, diagnostics=True)
    if name == "c5_200_cg":
        return run(r, r.stencil_csr(200, 3, convdiff_coeffs(0.3)), 200 ** 3, m=60, s=5, shat=60, scheme=3,
                   sketch=2, max_restarts=2, diagnostics=False)
    if name == "c1_diag":
        csr = r.laplace(100, 2)
        return {nm: run(r, csr, 10000, m=60, s=5, shat=60, scheme=sc, diagnostics=True)
                for nm, sc in [("cholqr2", 0), ("randcholqr", 1), ("twostage_pip", 2), ("twostage_randbcgs", 3)]}
    raise SystemExit(f"unknown section {name}")


ENV_PATH = Path(__file__).resolve().parent / "reference_envelopes.json"
ENV_CASES = {  # section: (problem, n, draws, kwargs)
    "c3_64": ("lap3d", 64, 4, dict(m=60, s=10, shat=60, scheme=1, sketch=0)),
    "c3_200": ("lap3d", 200, 2, dict(m=60, s=10, shat=60, scheme=1, sketch=0, max_restarts=4)),
    "c5_200": ("convdiff", 200, 2, dict(m=60, s=5, shat=60, scheme=3, sketch=0, max_restarts=3)),
}


def envelope(r, name):
    from paper_2503_16717_b200.borth import convdiff_coeffs
    prob, k, draws, kw = ENV_CASES[name]
    csr = r.laplace(k, 3) if prob == "lap3d" else r.stencil_csr(k, 3, convdiff_coeffs(0.3))
    n = k ** 3
    base = np.array(json.loads(PATH.read_text())[name]["relres"])
    rng = np.random.default_rng(0)
    worst = np.zeros(len(base))
    for t in range(draws):
        b = np.ones(n)
        b[rng.integers(0, n, 50)] = np.nextafter(1.0, 2.0 if t % 2 else 0.0)
        rr = np.array(r.sstep_gmres(csr, b, np.zeros(n), diagnostics=False, **kw).relres)
        m = min(len(rr), len(base))
        worst[:m] = np.maximum(worst[:m], np.abs(rr[:m] - base[:m]) / base[:m])
    return {"relres_rel_change": worst.tolist(), "draws": draws,
            "method": "50 entries of b moved by one ulp, worst over draws (oracle/_ref)"}


def main():
    names = sys.argv[1:] or ["c1_diag", "c3_64", "c3_200", "c5_200", "c5_200_cg"]
    r = Oracle("ref")
    for nm in names:
        t = time.time()
        path = ENV_PATH if nm.startswith("env_") else PATH
        val = envelope(r, nm[4:]) if nm.startswith("env_") else section(r, nm)
        out = json.loads(path.read_text()) if path.exists() else {
            "generator": "tests/golden/make_golden_big.py over oracle/_ref (reference sources, g++ -O3 -DNDEBUG)"}
        out[nm[4:] if nm.startswith("env_") else nm] = val
        path.write_text(json.dumps(out, indent=1))
        print(f"{nm}: {time.time() - t:.1f} s", flush=True)


if __name__ == "__main__":
    main()
