#!/usr/bin/env python
"""Generate tests/golden/reference_kats.json from the UNMODIFIED reference
(oracle/_ref/libblkorth_ref.so, built from /root/reference/proj sources by
oracle/Makefile).  Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The fixture pins the C oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_*.py) without needing /root/reference at test time.  Values
that go through glibc log/sin/cos (Gaussian sketches, gen_glued, RandCholQR
histories) are specific to this image's glibc 2.39 and its FMA ifunc variant
on the x86-64 hosts it runs on (SURVEY.md finding 1).
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
from py_oracle import Oracle  # noqa: E402


def gmres_kat(res):
    return {"converged": res.converged, "breakdown": res.breakdown, "detail": res.breakdown_detail,
            "restarts": res.restarts, "iterations": res.iterations, "final_relres": res.final_relres,
            "reduce": res.reduce, "reduce_total": res.reduce_total, "relres": res.relres,
            "lsq": res.lsq}


def extra_sections(r):
    """Sections added after the first fixture (python make_golden.py --update):
    the config-5 proxy (3D convection-diffusion 40^3, all four schemes) and the
    full-size config-3 CholQR2 breakdown (laplace_3d(200), n = 8e6)."""
    out = {}
    sys.path.insert(0, str(ROOT))
    from paper_2503_16717_b200.borth import convdiff_coeffs
    csr = r.stencil_csr(40, 3, convdiff_coeffs(0.3))
    n = 40 ** 3
    out["gmres_convdiff40"] = {
        name: gmres_kat(r.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=5, shat=60, scheme=scheme,
                                      diagnostics=False))
        for name, scheme in [("cholqr2", 0), ("randcholqr", 1), ("twostage_pip", 2), ("twostage_randbcgs", 3)]}
    csr = r.laplace(200, 3)
    n = 200 ** 3
    out["gmres_c3_cholqr2"] = gmres_kat(r.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=10, shat=60, scheme=0,
                                                      diagnostics=False))
    return out


def main():
    r = Oracle("ref")
    path = Path(__file__).resolve().parent / "reference_kats.json"
    if "--update" in sys.argv:
        out = json.loads(path.read_text())
        out.update(extra_sections(r))
        path.write_text(json.dumps(out, indent=1))
        print("updated", path)
        return
    out = {"generator": "tests/golden/make_golden.py over oracle/_ref (reference sources, g++ -O3 -DNDEBUG)"}
    # --- rng (rng.hpp)
    out["derive_seed"] = {f"{b},{s}": str(r.derive_seed(b, s)) for b, s in [(0, 0), (0, 1), (7960286522194355700, 0),
                                                                             (7960286522194355700, 1), (12345, 7)]}
    import ctypes as C
    f = r.lib.ref_rng_draws
    f.argtypes = [C.c_uint64, C.c_size_t, C.POINTER(C.c_uint64)]
    buf = (C.c_uint64 * 10000)()
    f(5489, 10000, buf)
    out["mt19937_64_seed5489_draw10000"] = str(buf[9999])
    f(derive := r.derive_seed(7960286522194355700, 0), 16, buf)
    out["mt_draws_first16_seed_cycle0"] = [str(buf[i]) for i in range(16)]
    g = r.lib.ref_rng_normals
    g.argtypes = [C.c_uint64, C.c_size_t, C.POINTER(C.c_double)]
    nb = (C.c_double * 8)()
    g(derive, 8, nb)
    out["normals_first8_seed_cycle0"] = [float(x) for x in nb]

    # --- sketches (sketch.cpp)
    sk = {}
    h = r.sketch_build(1, 1000, 10, 0).h
    b, s = r.sketch_count(h, 1000)
    sk["count_n1000_s10_seed0_rows0_7"] = [[int(b[i]), int(s[i])] for i in range(8)]
    h = r.sketch_build(0, 1000, 10, 0).h
    d = r.sketch_dense(h)
    sk["gauss_n1000_s10_seed0_col0_rows0_3"] = [float(x) for x in d[:4, 0]]
    sk["gauss_n1000_s10_seed0_r0c1"] = float(d[0, 1])
    seed1 = r.derive_seed(0, 1)
    rows = [0, 1, 2, 3, 999999, 1000000, 1999999, 2000000, 3999999, 4000000, 7999999]
    h = r.sketch_build(1, 8_000_000, 10, seed1).h
    b, s = r.sketch_count(h, 8_000_000)
    sk["count_n8e6_s10_seed_cycle0"] = {str(i): [int(b[i]), int(s[i])] for i in rows}
    r.sketch_free(h)
    h = r.sketch_build(0, 8_000_000, 10, seed1).h
    d = r.sketch_dense(h)
    sk["gauss_n8e6_s10_seed_cycle0"] = {str(i): [float(d[i, 0]), float(d[i, 11]), float(d[i, 21])] for i in rows}
    r.sketch_free(h)
    del d
    h = r.sketch_build(2, 5000, 5, 11).h
    sk["countgauss_n5000_s5_seed11_dense_r0"] = [float(x) for x in r.sketch_dense(h)[0, :6]]
    out["sketch"] = sk

    # --- SPEC.md dense examples
    spec = {}
    g2 = r.gram(np.array([[1.0, 0], [0, 1], [0, 0]]))
    spec["gram_e1e2"] = g2.tolist()
    R, fa, _ = r.cholesky(np.array([[4.0, 2], [2, 5]]))
    spec["cholesky_4_2_5"] = {"r": R.tolist(), "failed_at": fa}
    R, fa, piv = r.cholesky(np.array([[1.0, 1], [1, 1]]))
    spec["cholesky_rank1"] = {"failed_at": fa, "pivot": piv}
    q, R = r.householder_qr(np.array([[3.0], [4.0]]))
    spec["hhqr_3_4"] = {"q": q[:, 0].tolist(), "r": R.tolist()}
    spec["apply_inv_upper_3_4_5"] = r.apply_inv_upper(np.array([[3.0], [4.0]]), np.array([[5.0]])).x[:, 0].tolist()
    out["spec"] = spec

    # --- glued one-stage sweep
    sweep = {}
    th = r.sketch_build(0, 10000, 4, 17).h
    for kap in [1e0, 1e2, 1e4, 1e6, 1e8, 1e10, 1e12, 1e14, 1e15]:
        v = r.gen_glued(10000, 12, 5, kap, kap, 11)
        row = {}
        for intra in (0, 1):
            bb = r.basis_new(10000, 60)
            done, msg = 0, ""
            for p in range(12):
                res = r.bcgs2(bb, v[:, p * 5:(p + 1) * 5], intra, th if intra else None)
                if res.code:
                    msg = res.msg
                    break
                done += 1
            q, _, led = r.basis_state(bb, 10000)
            oe = float(np.linalg.norm(np.eye(q.shape[1]) - q.T @ q, 2)) if done == 12 else None
            row["cholqr2" if intra == 0 else "randcholqr"] = {"panels": done, "ledger": led, "msg": msg,
                                                              "orth": oe}
            r.basis_free(bb)
        sweep[f"{kap:g}"] = row
    out["glued_sweep_n1e4_12x5_seed11"] = sweep

    # --- GMRES (config 1 and breakdown KATs)
    gm = {}
    csr = r.laplace(100, 2)
    n = 10000
    for name, scheme, s in [("c1_cholqr2", 0, 5), ("c1_randcholqr", 1, 5), ("c1_twostage_pip", 2, 5),
                            ("c1_twostage_randbcgs", 3, 5), ("s10_cholqr2", 0, 10), ("s12_cholqr2", 0, 12),
                            ("s15_cholqr2", 0, 15), ("s10_randcholqr", 1, 10)]:
        res = r.sstep_gmres(csr, np.ones(n), np.zeros(n), m=60, s=s, shat=60, scheme=scheme)
        gm[name] = {"converged": res.converged, "breakdown": res.breakdown, "detail": res.breakdown_detail,
                    "restarts": res.restarts, "iterations": res.iterations, "final_relres": res.final_relres,
                    "reduce": res.reduce, "reduce_total": res.reduce_total, "relres": res.relres}
    out["gmres_2d100"] = gm

    # --- spmv
    out["spmv_tridiag"] = r.spmv((np.array([0, 2, 5, 7]), np.array([0, 1, 0, 1, 2, 1, 2]),
                                  np.array([2.0, -1, -1, 2, -1, -1, 2])), np.ones(3)).tolist()
    out.update(extra_sections(r))
    path.write_text(json.dumps(out, indent=1))
    print("wrote", path)


if __name__ == "__main__":
    main()
