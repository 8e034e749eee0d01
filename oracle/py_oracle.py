"""ctypes front-end for the CPU parity checkers (TEST INFRASTRUCTURE ONLY).

Two interchangeable back-ends with one Python API:
  Oracle("orc")  oracle/liboracle.so        — plain-C restatement (oracle.c)
  Oracle("ref")  oracle/_ref/libblkorth_ref.so — the unmodified reference
                  sources compiled by oracle/Makefile (absent on boxes where
                  /root/reference was never built; callers must skip then).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libblkorth_ref.so"
# the reference GMRES driver with its bcgs2 on the GPU (oracle/Makefile target refgpu)
REFGPU_LIB = HERE / "_ref" / "libblkorth_refgpu.so"

dp = C.POINTER(C.c_double)
sz = C.c_size_t
szp = C.POINTER(C.c_size_t)
u64 = C.c_uint64
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class OrcStatus(C.Structure):
    _fields_ = [("code", C.c_int), ("index", C.c_longlong), ("pivot", C.c_double), ("msg", C.c_char * 512)]


class OrcConfig(C.Structure):
    _fields_ = [("n", sz), ("m", sz), ("s", sz), ("shat", sz), ("scheme", C.c_int), ("sketch", C.c_int),
                ("rel_tol", C.c_double), ("max_restarts", sz), ("seed", u64), ("reorthogonalize", C.c_int),
                ("diagnostics", C.c_int)]


class OrcReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("breakdown", C.c_int), ("happy_breakdown", C.c_int),
                ("breakdown_detail", C.c_char * 512), ("restarts", sz), ("iterations", sz),
                ("initial_residual", C.c_double), ("final_relres", C.c_double), ("reduce", u64 * 4),
                ("reduce_total", u64), ("nhist", sz), ("relres", C.c_double * 256), ("lsq", C.c_double * 256),
                ("orth", C.c_double * 256), ("arnoldi", C.c_double * 256)]


class OrcCsr(C.Structure):
    _fields_ = [("nrows", sz), ("ncols", sz), ("nnz", sz), ("row_ptr", szp), ("col_idx", szp),
                ("values", dp)]


def ensure_built(ref: bool = False) -> None:
    if not ORC_LIB.exists() or (ref and not REF_LIB.exists() and Path("/root/reference/proj/src").exists()):
        subprocess.run(["make", "-s", "-C", str(HERE), "all"] + (["ref"] if ref and Path(
            "/root/reference/proj/src").exists() else []), check=True)


def have_ref() -> bool:
    ensure_built(ref=True)
    return REF_LIB.exists()


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(dp)


def F(a):
    """column-major float64 copy"""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class Result:
    def __init__(self, code, msg, **kw):
        self.code, self.msg = code, msg
        self.__dict__.update(kw)

    def __repr__(self):
        return f"Result(code={self.code}, msg={self.msg!r})"


class Oracle:
    """Uniform numpy API over the C restatement ('orc') or the reference ('ref')."""

    def __init__(self, which: str = "orc"):
        self.which = which
        ensure_built(ref=(which == "ref"))
        path = {"orc": ORC_LIB, "ref": REF_LIB, "refgpu": REFGPU_LIB}[which]
        if not path.exists():
            raise FileNotFoundError(path)
        self.lib = C.CDLL(str(path))
        self.p = "orc_" if which == "orc" else "ref_"
        L = self.lib
        st = getattr(L, self.p + "last_status")
        st.restype = C.POINTER(OrcStatus)
        self._status = st

    def _fn(self, name, res, args):
        f = getattr(self.lib, self.p + name)
        f.restype = res
        f.argtypes = args
        return f

    def status(self):
        s = self._status().contents
        return s.code, s.msg.decode(errors="replace"), s.index

    def set_sum_chunks(self, chunks: int):
        """test-only summation-order perturbation of the C restatement's tall
        dot products (oracle.c tall_dot); 0 restores the reference order"""
        assert self.which == "orc", "only the C restatement has a summation-order knob"
        self._fn("set_sum_chunks", None, [sz])(chunks)

    # ---------------- rng
    def derive_seed(self, base, stream):
        return int(self._fn("derive_seed", u64, [u64, u64])(base, stream))

    # ---------------- dense
    def gram(self, v):
        v = F(v)
        n, k = v.shape
        g = np.zeros((k, k), order="F")
        self._fn("gram", None, [dp, sz, sz, dp])(_d(v.T.ravel()) if False else v.ctypes.data_as(dp), n, k,
                                                 g.ctypes.data_as(dp))
        return g

    def cholesky(self, g, tol=2.220446049250313e-16):
        g = F(g)
        k = g.shape[0]
        r = np.zeros((k, k), order="F")
        piv = C.c_double()
        f = self._fn("cholesky", sz, [dp, sz, C.c_double, dp, C.POINTER(C.c_double)])(
            g.ctypes.data_as(dp), k, tol, r.ctypes.data_as(dp), C.byref(piv))
        return r, int(f), piv.value

    def householder_qr(self, v):
        v = F(v)
        n, k = v.shape
        q = np.zeros((n, k), order="F")
        r = np.zeros((k, k), order="F")
        self._fn("householder_qr", None, [dp, sz, sz, dp, dp])(v.ctypes.data_as(dp), n, k, q.ctypes.data_as(dp),
                                                                r.ctypes.data_as(dp))
        return q, r

    def apply_inv_upper(self, v, r):
        v, r = F(v), F(r)
        n, k = v.shape
        x = np.zeros((n, k), order="F")
        rc = self._fn("apply_inv_upper", C.c_int, [dp, sz, sz, dp, dp])(v.ctypes.data_as(dp), n, k,
                                                                         r.ctypes.data_as(dp), x.ctypes.data_as(dp))
        return Result(rc, self.status()[1], x=x)

    # ---------------- sketch
    def sketch_build(self, kind, n, shat, seed):
        f = self._fn("sketch_build", vp, [C.c_int, sz, sz, u64])
        h = f(kind, n, shat, seed)
        if not h:
            code, msg, _ = self.status()
            return Result(code, msg, h=None)
        return Result(0, "", h=h)

    def sketch_free(self, h):
        self._fn("sketch_free", None, [vp])(h)

    def sketch_size(self, h):
        return int(self._fn("sketch_size", sz, [vp])(h))

    def sketch_dense(self, h):
        if self.which == "orc":
            rows, cols = sz(), sz()
            ptr = self._fn("sketch_dense", dp, [vp, szp, szp])(h, C.byref(rows), C.byref(cols))
            if not ptr:
                return None
            return np.ctypeslib.as_array(ptr, shape=(cols.value * rows.value,)).reshape(
                (rows.value, cols.value), order="F").copy()
        rows, cols = sz(), sz()
        f = self._fn("sketch_dense", None, [vp, dp, szp, szp])
        f(h, None, C.byref(rows), C.byref(cols))
        out = np.zeros((rows.value, cols.value), order="F")
        if rows.value * cols.value:
            f(h, out.ctypes.data_as(dp), C.byref(rows), C.byref(cols))
        return out

    def sketch_count(self, h, n):
        if self.which == "orc":
            bp = self._fn("sketch_buckets", C.POINTER(C.c_uint32), [vp])(h)
            sp = self._fn("sketch_signs", dp, [vp])(h)
            if not bp:
                return None, None
            return (np.ctypeslib.as_array(bp, shape=(n,)).copy(), np.ctypeslib.as_array(sp, shape=(n,)).copy())
        b = np.zeros(n, dtype=np.uint32)
        s = np.zeros(n)
        self._fn("sketch_count", sz, [vp, C.POINTER(C.c_uint32), dp])(h, b.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                                      s.ctypes.data_as(dp))
        return b, s

    def sketch_apply(self, h, v):
        v = F(v)
        n, k = v.shape
        m = self.sketch_size(h)
        out = np.zeros((m, k), order="F")
        self._fn("sketch_apply", None, [vp, dp, sz, sz, dp])(h, v.ctypes.data_as(dp), n, k, out.ctypes.data_as(dp))
        return out

    # ---------------- intra
    def _intra(self, name, v, sk=None):
        v = F(v)
        n, k = v.shape
        q = np.zeros((n, k), order="F")
        r = np.zeros((k, k), order="F")
        led = (u64 * 4)()
        if sk is None:
            rc = self._fn(name, C.c_int, [dp, sz, sz, dp, dp, u64p])(v.ctypes.data_as(dp), n, k,
                                                                    q.ctypes.data_as(dp), r.ctypes.data_as(dp), led)
        else:
            rc = self._fn(name, C.c_int, [dp, sz, sz, vp, dp, dp, u64p])(v.ctypes.data_as(dp), n, k, sk,
                                                                        q.ctypes.data_as(dp), r.ctypes.data_as(dp),
                                                                        led)
        code, msg, idx = self.status()
        return Result(rc, msg if rc else "", q=q, r=r, ledger=list(led), index=idx)

    def cholqr(self, v):
        return self._intra("cholqr", v)

    def cholqr2(self, v):
        return self._intra("cholqr2", v)

    def rand_cholqr(self, v, sk):
        return self._intra("rand_cholqr", v, sk)

    def recursive_cholqr(self, v):
        v = F(v)
        n, k = v.shape
        q = np.zeros((n, k), order="F")
        co = np.zeros((k, k), order="F")
        kept = (sz * (k + 1))()
        disc = (sz * (k + 1))()
        dn = np.zeros(k + 1)
        nk, nd, depth = sz(), sz(), sz()
        led = (u64 * 4)()
        rc = self._fn("recursive_cholqr", C.c_int, [dp, sz, sz, dp, dp, szp, szp, szp, dp, szp, szp, u64p])(
            v.ctypes.data_as(dp), n, k, q.ctypes.data_as(dp), co.ctypes.data_as(dp), kept, C.byref(nk), disc,
            dn.ctypes.data_as(dp), C.byref(nd), C.byref(depth), led)
        return Result(rc, self.status()[1] if rc else "", q=q[:, : nk.value], coeffs=co[: nk.value, :],
                      kept=list(kept)[: nk.value], discarded=list(disc)[: nd.value],
                      discard_norm=list(dn[: nd.value]), depth=depth.value, ledger=list(led))

    # ---------------- basis
    def basis_new(self, n, cap):
        return self._fn("basis_new", vp, [sz, sz])(n, cap)

    def basis_free(self, b):
        self._fn("basis_free", None, [vp])(b)

    def basis_cols(self, b):
        return int(self._fn("basis_cols", sz, [vp])(b))

    def basis_state(self, b, n):
        cols = self.basis_cols(b)
        if self.which == "orc":
            qp = self._fn("basis_q", dp, [vp])(b)
            rp = self._fn("basis_r", dp, [vp])(b)
            cap = self._cap[b] if hasattr(self, "_cap") and b in self._cap else None
            led = (u64 * 4)()
            self._fn("basis_ledger", None, [vp, u64p])(b, led)
            q = np.ctypeslib.as_array(qp, shape=(n * cols,)).reshape((n, cols), order="F").copy() if cols else \
                np.zeros((n, 0))
            return q, None, list(led)
        q = np.zeros((n, cols), order="F")
        r = np.zeros((cols, cols), order="F")
        led = (u64 * 4)()
        self._fn("basis_get", None, [vp, dp, dp, u64p])(b, q.ctypes.data_as(dp), r.ctypes.data_as(dp), led)
        return q, r, list(led)

    def basis_r(self, b, cap):
        """R restricted to cols x cols (r_copy semantics)."""
        cols = self.basis_cols(b)
        if self.which == "orc":
            rp = self._fn("basis_r", dp, [vp])(b)
            full = np.ctypeslib.as_array(rp, shape=(cap * cap,)).reshape((cap, cap), order="F")
            return np.triu(full[:cols, :cols]).copy()
        r = np.zeros((cols, cols), order="F")
        n = 0
        self._fn("basis_get", None, [vp, dp, dp, u64p])(b, None, r.ctypes.data_as(dp), None)
        return r

    def basis_ledger(self, b):
        led = (u64 * 4)()
        if self.which == "orc":
            self._fn("basis_ledger", None, [vp, u64p])(b, led)
        else:
            self._fn("basis_get", None, [vp, dp, dp, u64p])(b, None, None, led)
        return list(led)

    def basis_mark_seed(self, b, col):
        self._fn("basis_mark_seed", None, [vp, sz])(b, col)

    def basis_begin_big_panel(self, b, rows, overlap):
        self._fn("basis_begin_big_panel", None, [vp, sz, C.c_int])(b, rows, int(overlap))

    def basis_input_coeff_col(self, b, k, length):
        out = np.zeros(length)
        self._fn("basis_input_coeff_col", None, [vp, sz, sz, dp])(b, k, length, out.ctypes.data_as(dp))
        return out

    def basis_sketched(self, b):
        rows = sz()
        if self.which == "orc":
            ptr = C.POINTER(C.c_double)()
            cols = self._fn("basis_sketched", sz, [vp, C.POINTER(dp), szp])(b, C.byref(ptr), C.byref(rows))
            if cols == 0:
                return np.zeros((rows.value, 0))
            return np.ctypeslib.as_array(ptr, shape=(rows.value * cols,)).reshape((rows.value, cols),
                                                                                   order="F").copy()
        f = self._fn("basis_sketched", sz, [vp, dp, szp])
        cols = f(b, None, C.byref(rows))
        out = np.zeros((rows.value, cols), order="F")
        if cols:
            f(b, out.ctypes.data_as(dp), C.byref(rows))
        return out

    def bcgs_project_range(self, b, v, lo, hi):
        v = F(v)
        n, k = v.shape
        vh = np.zeros((n, k), order="F")
        co = np.zeros((hi - lo, k), order="F")
        if self.which == "orc":
            self._fn("bcgs_project_range", None, [vp, dp, sz, sz, sz, dp, dp])(
                b, v.ctypes.data_as(dp), k, lo, hi, vh.ctypes.data_as(dp), co.ctypes.data_as(dp))
        else:
            self._fn("bcgs_project_range", None, [vp, dp, sz, sz, sz, sz, dp, dp])(
                b, v.ctypes.data_as(dp), n, k, lo, hi, vh.ctypes.data_as(dp), co.ctypes.data_as(dp))
        return vh, co

    def _vargs(self, v):
        v = F(v)
        n, k = v.shape
        return v, n, k

    def bcgs2(self, b, v, intra, sk=None, overlap=False):
        v, n, k = self._vargs(v)
        if self.which == "orc":
            rc = self._fn("bcgs2", C.c_int, [vp, dp, sz, C.c_int, vp, C.c_int])(b, v.ctypes.data_as(dp), k, intra,
                                                                             sk, int(overlap))
        else:
            rc = self._fn("bcgs2", C.c_int, [vp, dp, sz, sz, C.c_int, vp, C.c_int])(b, v.ctypes.data_as(dp), n, k,
                                                                                intra, sk, int(overlap))
        return Result(rc, self.status()[1] if rc else "", index=self.status()[2])

    def bcgs_pip(self, b, v, overlap=False):
        v, n, k = self._vargs(v)
        if self.which == "orc":
            rc = self._fn("bcgs_pip", C.c_int, [vp, dp, sz, C.c_int])(b, v.ctypes.data_as(dp), k, int(overlap))
        else:
            rc = self._fn("bcgs_pip", C.c_int, [vp, dp, sz, sz, C.c_int])(b, v.ctypes.data_as(dp), n, k,
                                                                         int(overlap))
        return Result(rc, self.status()[1] if rc else "")

    def rand_bcgs_preproc(self, b, v, sk, overlap=False):
        v, n, k = self._vargs(v)
        if self.which == "orc":
            rc = self._fn("rand_bcgs_preproc", C.c_int, [vp, dp, sz, vp, C.c_int])(b, v.ctypes.data_as(dp), k, sk,
                                                                                 int(overlap))
        else:
            rc = self._fn("rand_bcgs_preproc", C.c_int, [vp, dp, sz, sz, vp, C.c_int])(
                b, v.ctypes.data_as(dp), n, k, sk, int(overlap))
        return Result(rc, self.status()[1] if rc else "")

    def two_stage_panel(self, b, v, preproc, sk=None, overlap=False):
        v, n, k = self._vargs(v)
        if self.which == "orc":
            rc = self._fn("two_stage_panel", C.c_int, [vp, dp, sz, C.c_int, vp, C.c_int])(
                b, v.ctypes.data_as(dp), k, preproc, sk, int(overlap))
        else:
            rc = self._fn("two_stage_panel", C.c_int, [vp, dp, sz, sz, C.c_int, vp, C.c_int])(
                b, v.ctypes.data_as(dp), n, k, preproc, sk, int(overlap))
        return Result(rc, self.status()[1] if rc else "")

    def two_stage_finish(self, b, preproc, reorth=True, record=False):
        stats = np.zeros(2)
        rc = self._fn("two_stage_finish", C.c_int, [vp, C.c_int, C.c_int, C.c_int, dp])(
            b, preproc, int(reorth), int(record), stats.ctypes.data_as(dp))
        return Result(rc, self.status()[1] if rc else "", stats=stats)

    # ---------------- problems / sparse
    def gen_glued(self, n, np_, w, kp, kg, seed):
        v = np.zeros((n, np_ * w), order="F")
        self._fn("gen_glued", None, [sz, sz, sz, C.c_double, C.c_double, u64, dp])(n, np_, w, kp, kg, seed,
                                                                                  v.ctypes.data_as(dp))
        return v

    def laplace(self, k, dims):
        """CSR arrays (row_ptr, col, val) of laplace_2d / laplace_3d"""
        if self.which == "orc":
            f = self._fn("laplace_2d" if dims == 2 else "laplace_3d", C.POINTER(OrcCsr), [sz])
            a = f(k).contents
            n, nnz = a.nrows, a.nnz
            rp = np.ctypeslib.as_array(a.row_ptr, shape=(n + 1,)).astype(np.int64)
            ci = np.ctypeslib.as_array(a.col_idx, shape=(nnz,)).astype(np.int64)
            vv = np.ctypeslib.as_array(a.values, shape=(nnz,)).copy()
            self._fn("csr_free", None, [C.POINTER(OrcCsr)])(C.pointer(a))
            return rp, ci, vv
        h = self._fn("laplace", vp, [sz, C.c_int])(k, dims)
        nr, nc = sz(), sz()
        nnz = self._fn("csr_info", sz, [vp, szp, szp])(h, C.byref(nr), C.byref(nc))
        rp = np.zeros(nr.value + 1, dtype=np.uint64)
        ci = np.zeros(nnz, dtype=np.uint64)
        vv = np.zeros(nnz)
        self._fn("csr_arrays", None, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), dp])(
            h, rp.ctypes.data_as(C.POINTER(C.c_uint64)), ci.ctypes.data_as(C.POINTER(C.c_uint64)),
            vv.ctypes.data_as(dp))
        self._fn("csr_free", None, [vp])(h)
        return rp.astype(np.int64), ci.astype(np.int64), vv

    @staticmethod
    def stencil_csr(k, dims, coeffs):
        """CSR (row_ptr, col, val) of a constant-coefficient 5/7-point stencil on
        a k^dims grid, entries in ascending column order per row (what
        CsrMatrix::from_triplets, sparse.cpp:13-42, makes of the row-major
        triplet list; problems.cpp:65-113 for the Laplacian coefficients).
        Config 5's convection-diffusion operator is not in the reference
        (SURVEY finding 4): this generator is test infrastructure."""
        c = np.asarray(coeffs, dtype=np.float64)
        n = k ** dims
        me = np.arange(n, dtype=np.int64)
        if dims == 3:
            i, j, l = me // (k * k), (me // k) % k, me % k
            nb = [(i > 0, -k * k), (j > 0, -k), (l > 0, -1), (np.ones(n, bool), 0), (l + 1 < k, 1),
                  (j + 1 < k, k), (i + 1 < k, k * k)]
        else:
            i, j = me // k, me % k
            nb = [(i > 0, -k), (j > 0, -1), (np.ones(n, bool), 0), (j + 1 < k, 1), (i + 1 < k, k)]
        present = np.stack([m for m, _ in nb], axis=1)
        cols = me[:, None] + np.array([o for _, o in nb])[None, :]
        vals = np.broadcast_to(c[None, :], present.shape)
        counts = present.sum(axis=1)
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=rp[1:])
        return rp, cols[present].astype(np.int64), vals[present].astype(np.float64)

    def csr_from_triplets(self, rp, ci, vv, ncols=None):
        """round-trip through the oracle's from_triplets (sorted, duplicates summed)"""
        ncols = ncols or (len(rp) - 1)
        h, keep = self._csr_handle(rp, ci, vv, ncols)
        if self.which == "orc":
            a = h.contents
            n, nnz = a.nrows, a.nnz
            out = (np.ctypeslib.as_array(a.row_ptr, shape=(n + 1,)).astype(np.int64),
                   np.ctypeslib.as_array(a.col_idx, shape=(nnz,)).astype(np.int64),
                   np.ctypeslib.as_array(a.values, shape=(nnz,)).copy())
        else:
            nr, nc = sz(), sz()
            nnz = self._fn("csr_info", sz, [vp, szp, szp])(h, C.byref(nr), C.byref(nc))
            r = np.zeros(nr.value + 1, dtype=np.uint64)
            c = np.zeros(nnz, dtype=np.uint64)
            v = np.zeros(nnz)
            self._fn("csr_arrays", None, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), dp])(
                h, r.ctypes.data_as(C.POINTER(C.c_uint64)), c.ctypes.data_as(C.POINTER(C.c_uint64)),
                v.ctypes.data_as(dp))
            out = (r.astype(np.int64), c.astype(np.int64), v)
        self._csr_free(h)
        return out

    def _csr_handle(self, rp, ci, vv, ncols):
        n = len(rp) - 1
        rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(rp)).astype(np.uint64)
        cols = np.asarray(ci, dtype=np.uint64)
        vals = np.ascontiguousarray(vv, dtype=np.float64)
        if self.which == "orc":
            f = self._fn("csr_from_triplets", C.POINTER(OrcCsr), [sz, sz, sz, szp, szp, dp])
            h = f(n, ncols, len(vals), rows.ctypes.data_as(szp), cols.ctypes.data_as(szp), vals.ctypes.data_as(dp))
            return h, (rows, cols, vals)
        f = self._fn("csr_from_triplets", vp, [sz, sz, sz, szp, szp, dp])
        h = f(n, ncols, len(vals), rows.ctypes.data_as(szp), cols.ctypes.data_as(szp), vals.ctypes.data_as(dp))
        return h, (rows, cols, vals)

    def _csr_free(self, h):
        if self.which == "orc":
            self._fn("csr_free", None, [C.POINTER(OrcCsr)])(h)
        else:
            self._fn("csr_free", None, [vp])(h)

    def spmv(self, csr, x, ncols=None):
        rp, ci, vv = csr
        ncols = ncols or (len(rp) - 1)
        h, keep = self._csr_handle(rp, ci, vv, ncols)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(len(rp) - 1)
        if self.which == "orc":
            self._fn("spmv", None, [C.POINTER(OrcCsr), dp, dp])(h, x.ctypes.data_as(dp), y.ctypes.data_as(dp))
        else:
            self._fn("spmv", None, [vp, dp, dp])(h, x.ctypes.data_as(dp), y.ctypes.data_as(dp))
        self._csr_free(h)
        return y

    def mpk(self, csr, v0, s):
        rp, ci, vv = csr
        n = len(rp) - 1
        h, keep = self._csr_handle(rp, ci, vv, n)
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        v = np.zeros((n, s + 1), order="F")
        argt = [C.POINTER(OrcCsr) if self.which == "orc" else vp, dp, sz, dp]
        self._fn("mpk", None, argt)(h, v0.ctypes.data_as(dp), s, v.ctypes.data_as(dp))
        self._csr_free(h)
        return v

    def sstep_gmres(self, csr, b, x0, *, m=60, s=5, shat=60, scheme=0, sketch=0, rel_tol=1e-6, max_restarts=50,
                    seed=0, reorthogonalize=True, diagnostics=True):
        rp, ci, vv = csr
        n = len(rp) - 1
        h, keep = self._csr_handle(rp, ci, vv, n)
        cfg = OrcConfig(n=n, m=m, s=s, shat=shat, scheme=scheme, sketch=sketch, rel_tol=rel_tol,
                        max_restarts=max_restarts, seed=seed, reorthogonalize=int(reorthogonalize),
                        diagnostics=int(diagnostics))
        rep = OrcReport()
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        x = np.zeros(n)
        argt = [C.POINTER(OrcCsr) if self.which == "orc" else vp, dp, dp, C.POINTER(OrcConfig), dp,
                C.POINTER(OrcReport)]
        rc = self._fn("sstep_gmres", C.c_int, argt)(h, b.ctypes.data_as(dp), x0.ctypes.data_as(dp), C.byref(cfg),
                                                    x.ctypes.data_as(dp), C.byref(rep))
        self._csr_free(h)
        nh = rep.nhist
        return Result(rc, self.status()[1] if rc else "", x=x, converged=bool(rep.converged),
                      breakdown=bool(rep.breakdown), happy_breakdown=bool(rep.happy_breakdown),
                      breakdown_detail=rep.breakdown_detail.decode(errors="replace"), restarts=rep.restarts,
                      iterations=rep.iterations, initial_residual=rep.initial_residual,
                      final_relres=rep.final_relres, reduce=list(rep.reduce), reduce_total=rep.reduce_total,
                      relres=list(rep.relres)[:nh], lsq=list(rep.lsq)[:nh], orth=list(rep.orth)[:nh],
                      arnoldi=list(rep.arnoldi)[:nh])
