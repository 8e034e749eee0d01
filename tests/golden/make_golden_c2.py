#!/usr/bin/env python
"""Config-2 reference runs at the benchmarked size (tests/golden/c2_ref.npz):
the six panels of gen_glued(8e6, 6, 11, kappa, kappa, 7)
through the UNMODIFIED reference's bcgs2 sequence (p = 0, 11, ..., 55, no
overlap), oracle/_ref built from /root/reference sources.

    python tests/golden/make_golden_c2.py [n]

Stored per case (kappa in {1e2, 1e6} x {cholqr2, randcholqr}; kappa in
{1e10, 1e14} randcholqr, plus the cholqr2 breakdown message there):
  sha256 of the input panels (raw FP64, column-major; the repo's device
  gen_glued must reproduce them bit for bit), R (66 x 66), Q at 256 fixed rows,
  Q^T z for a fixed z, the column sums of Q, ||I - Q^T Q||_2, the ledger, the
  outcome message and the CPU time of the sequence.  The Gaussian sketch is
  build(gaussian, n, 10, seed=1) (m-hat = 22), as bench.py uses.
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
from py_oracle import Oracle  # noqa: E402

OUT = Path(__file__).resolve().parent / "c2_ref.npz"


def sample_rows(n, count=256):
    rng = np.random.default_rng(2503)
    rows = set([0, 1, 2, n // 2 - 1, n // 2, n - 2, n - 1])
    rows.update(int(x) for x in rng.integers(0, n, count - len(rows)))
    return np.array(sorted(rows), dtype=np.int64)


def probe(n):
    return np.random.default_rng(16717).standard_normal(n)


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 8_000_000
    k, panels = 11, 6
    r = Oracle("ref")
    rows = sample_rows(n)
    z = probe(n)
    data = {"n": np.array(n), "rows": rows}
    meta = {}
    th = r.sketch_build(0, n, k - 1, 1).h
    for kap in (1e2, 1e6, 1e10, 1e14):
        t0 = time.time()
        v = r.gen_glued(n, panels, k, kap, kap, 7)
        tg = time.time() - t0
        sha = hashlib.sha256(np.asfortranarray(v).tobytes(order="F")).hexdigest()
        for intra, name in ((0, "cholqr2"), (1, "randcholqr")):
            key = f"k{kap:g}_{name}"
            b = r.basis_new(n, panels * k)
            t0 = time.time()
            done, msg = 0, ""
            for p in range(panels):
                res = r.bcgs2(b, v[:, p * k:(p + 1) * k], intra, th if intra else None)
                if res.code:
                    msg = res.msg
                    break
                done += 1
            secs = time.time() - t0
            q, R, led = r.basis_state(b, n)
            m = {"sha256_input": sha, "panels_done": done, "msg": msg, "ledger": list(led), "cpu_seconds": secs,
                 "gen_seconds": tg}
            if done == panels:
                data[key + "_R"] = R
                data[key + "_Qrows"] = q[rows]
                data[key + "_QTz"] = q.T @ z
                data[key + "_colsum"] = q.sum(axis=0)
                m["orth"] = float(np.linalg.norm(np.eye(q.shape[1]) - q.T @ q, 2))
            meta[key] = m
            r.basis_free(b)
            del q
            print(key, m, flush=True)
        del v
    data["meta"] = np.array(json.dumps(meta))
    np.savez(OUT, **data)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
