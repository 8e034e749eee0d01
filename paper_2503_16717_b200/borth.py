"""Python mirror of the reference blkorth interface over the C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:
  SketchOperator.build/apply  proj/include/blkorth/sketch.hpp:28-40
  cholqr/cholqr2/rand_cholqr  proj/include/blkorth/intra_orth.hpp:19-28
  recursive_cholqr            proj/include/blkorth/intra_orth.hpp:50
  BasisStore                  proj/include/blkorth/block_orth.hpp:27-102
  bcgs_project_range / bcgs2 / bcgs_pip / rand_bcgs_preproc / two_stage_*
                              proj/include/blkorth/block_orth.hpp:111-169
  mpk / spmv                  proj/include/blkorth/gmres.hpp:65, sparse.hpp:49
  sstep_gmres_solve           proj/include/blkorth/gmres.hpp:92
Exceptions mirror proj/include/blkorth/errors.hpp.

Tall ("panel") arguments live on the GPU as torch float64 tensors of shape
(k, ld) — column j is row j of the tensor, i.e. column-major n_local x k with
leading dimension ld (the reference's DenseMatrix layout,
proj/include/blkorth/dense.hpp:30-31).  torch supplies device memory and
streams only; every computation is a kernel in libbo_cuda.so.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

GAUSSIAN, COUNT, COUNT_GAUSS = 0, 1, 2
CHOLQR2, RAND_CHOLQR = 0, 1
PIP, RAND_BCGS = 0, 1
SCHEMES = {"bcgs2_cholqr2": 0, "bcgs2_randcholqr": 1, "twostage_pip": 2, "twostage_randbcgs": 3,
           "standard_cgs2": 4}
SKETCHES = {"gaussian": 0, "count": 1, "countgauss": 2, "count_gauss": 2}


# ----------------------------------------------------------------- errors --
class Error(RuntimeError):
    """blkorth::Error (errors.hpp:12)"""


class CholeskyBreakdown(Error):
    def __init__(self, msg, step):
        super().__init__(msg)
        self.step = step


class SingularTriangular(Error):
    def __init__(self, msg, index):
        super().__init__(msg)
        self.index = index


class AmbientTooSmall(Error):
    pass


class AllColumnsDiscarded(Error):
    pass


class RankDeficient(Error):
    pass


class InvalidScheme(Error):
    pass


class ZeroMatrix(Error):
    pass


class ParseError(Error):
    """errors.hpp:77 (MatrixMarket); .line = offending line number"""
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class BannerError(Error):
    """errors.hpp:88 (MatrixMarket banner)"""


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


def _raise(rc: int, st: L.Status):
    msg = st.msg.decode(errors="replace")
    if rc == 1:
        raise CholeskyBreakdown(msg, int(st.index))
    if rc == 2:
        raise SingularTriangular(msg, int(st.index))
    if rc == 3:
        raise AmbientTooSmall(msg)
    if rc == 4:
        raise AllColumnsDiscarded(msg)
    if rc == 5:
        raise RankDeficient(msg)
    if rc == 6:
        raise InvalidScheme(msg)
    if rc == 7:
        raise ZeroMatrix(msg)
    if rc == 8:
        raise CudaError(msg)
    if rc == 9:
        raise NcclError(msg)
    if rc == 10:
        raise ParseError(msg, int(st.index))
    if rc == 11:
        raise BannerError(msg)
    raise Error(f"bo error {rc}: {msg}")


def _call(fn, *args):
    st = L.Status()
    rc = fn(*args, C.byref(st))
    if rc != 0:
        _raise(rc, st)
    return rc


def _dp(a: np.ndarray):
    return a.ctypes.data_as(L.dp)


@dataclass
class ReduceLedger:
    """ReduceLedger (dense.hpp:97-119): projection / gram / sketch / norm."""
    counts: list = field(default_factory=lambda: [0, 0, 0, 0])

    @property
    def projection(self):
        return self.counts[0]

    @property
    def gram(self):
        return self.counts[1]

    @property
    def sketch(self):
        return self.counts[2]

    @property
    def norm(self):
        return self.counts[3]

    def total(self):
        return sum(self.counts)


def _ledger_in(led):
    arr = (C.c_uint64 * 4)(*(led.counts if led is not None else [0, 0, 0, 0]))
    return arr


def _ledger_out(led, arr):
    if led is not None:
        led.counts = list(arr)


# -------------------------------------------------------------- transport --
class TorchDistComm:
    """Collective transport through an initialised torch.distributed process
    group (e.g. gloo) for bo_ctx_create_comm: device buffers are staged
    through host memory.  Used to run the sharded (world > 1) path of the
    library on one GPU in tests; production multi-GPU runs use NCCL."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.ops = L.CommOps(None, L.ALLREDUCE_FN(self._allreduce), L.ALLGATHER_FN(self._allgather),
                             L.EXCHANGE_FN(self._exchange))
        self.calls = {"allreduce": 0, "allgather": 0, "exchange": 0}

    def _view(self, ptr, count, dtype):
        t = self.torch
        class _H:  # noqa: E306
            __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8" if dtype == "f8" else "<i8",
                                        "data": (int(ptr), False), "version": 3, "strides": None}
        return t.as_tensor(_H(), device="cuda")

    def _sync(self, stream):
        self.torch.cuda.ExternalStream(int(stream)).synchronize()

    def _allreduce(self, user, buf, count, stream):
        try:
            self._sync(stream)
            dev = self._view(buf, count, "f8")
            host = dev.cpu()
            self.dist.all_reduce(host, group=self.group)
            dev.copy_(host)
            self.torch.cuda.synchronize()
            self.calls["allreduce"] += 1
            return 0
        except Exception:  # pragma: no cover - reported as BO_NCCL by the library
            return 1

    def _allgather(self, user, send, count, recv, stream):
        try:
            self._sync(stream)
            mine = self._view(send, count, "i8").cpu()
            parts = [self.torch.empty_like(mine) for _ in range(self.dist.get_world_size(self.group))]
            self.dist.all_gather(parts, mine, group=self.group)
            out = self._view(recv, count * len(parts), "i8")
            out.copy_(self.torch.cat(parts).to(out.device))
            if os.environ.get("BO_DEBUG_COMM"):
                self.torch.cuda.synchronize()
                print("allgather", self.dist.get_rank(), mine.tolist(), [p_.tolist() for p_ in parts],
                      out.cpu().tolist(), flush=True)
            self.torch.cuda.synchronize()
            self.calls["allgather"] += 1
            return 0
        except Exception:  # pragma: no cover
            return 1

    def _exchange(self, user, nops, ops, stream):
        # every rank contributes its outgoing blocks to one all-gather and
        # picks its incoming ones (at most one block per peer and direction
        # per group): no point-to-point matching to go wrong
        try:
            self._sync(stream)
            me = self.dist.get_rank(self.group)
            out, recvs = {}, []
            for i in range(nops):
                o = ops[i]
                dev = self._view(o.buf, o.count, "f8")
                if o.is_send:
                    out[int(o.peer)] = dev.cpu().numpy()
                else:
                    recvs.append((int(o.peer), dev))
            allout = [None] * self.dist.get_world_size(self.group)
            self.dist.all_gather_object(allout, out, group=self.group)
            for peer, dev in recvs:
                dev.copy_(self.torch.from_numpy(allout[peer][me]))
            self.torch.cuda.synchronize()
            self.calls["exchange"] += 1
            return 0
        except Exception:  # pragma: no cover
            import traceback
            traceback.print_exc()
            return 1


# ---------------------------------------------------------------- context --
class Context:
    """One GPU: the row shard [row_begin, row_end) of an n-row problem."""

    def __init__(self, n: int, *, device: int = 0, rank: int = 0, world: int = 1,
                 row_begin: int | None = None, row_end: int | None = None,
                 nccl_id: bytes | None = None, stream=None, comm=None):
        import torch
        self.lib = L.load()
        self.torch = torch
        if row_begin is None:
            row_begin, row_end = 0, n
        self.n, self.rank, self.world = n, rank, world
        self.row_begin, self.row_end = row_begin, row_end
        if not torch.cuda.is_available():
            # let the library report it: the path has no CPU fallback
            h = C.c_void_p()
            _call(self.lib.bo_ctx_create, device, rank, world, None, n, row_begin, row_end, None, C.byref(h))
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        # the library runs on this (non-default) stream; torch work that feeds
        # it (from_host, panel) is issued on the same stream
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        h = C.c_void_p()
        self._comm = comm  # keeps the ctypes callbacks alive
        if comm is not None:
            _call(self.lib.bo_ctx_create_comm, device, rank, world, C.byref(comm.ops), n, row_begin, row_end,
                  C.c_void_p(self.stream.cuda_stream), C.byref(h))
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            _call(self.lib.bo_ctx_create, device, rank, world, idbuf, n, row_begin, row_end,
                  C.c_void_p(self.stream.cuda_stream), C.byref(h))
        self.h = h
        self.n_global = int(n)
        self.n_local = int(self.lib.bo_ctx_local_rows(h))
        self.ld = int(self.lib.bo_ctx_ld(h))
        self._children = weakref.WeakSet()

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = L.load()
        buf = C.create_string_buffer(128)
        _call(lib.bo_nccl_get_unique_id, buf)
        return buf.raw

    # tall buffers -----------------------------------------------------------
    def panel(self, k: int, zero: bool = True):
        t = self.torch
        f = t.zeros if zero else t.empty
        with t.cuda.stream(self.stream):
            return f((k, self.ld), dtype=t.float64, device=self.device)

    def from_host(self, a: np.ndarray):
        """n_local x k host array -> device panel (k, ld)."""
        a = np.asarray(a, dtype=np.float64)
        if a.ndim == 1:
            a = a[:, None]
        assert a.shape[0] == self.n_local, (a.shape, self.n_local)
        p = self.panel(a.shape[1])
        with self.torch.cuda.stream(self.stream):
            p[:, : self.n_local] = self.torch.from_numpy(np.ascontiguousarray(a.T)).to(self.device)
        return p

    def to_host(self, p, k: int | None = None) -> np.ndarray:
        k = p.shape[0] if k is None else k
        self.stream.synchronize()
        return p[:k, : self.n_local].detach().cpu().numpy().T.copy()

    def synchronize(self):
        _call(self.lib.bo_ctx_synchronize, self.h)

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.bo_ctx_kernel_launches(self.h))

    @property
    def allreduces(self) -> int:
        return int(self.lib.bo_ctx_allreduces(self.h))

    def profile(self, enable: bool = True):
        self.lib.bo_ctx_profile(self.h, int(enable))

    def profile_read(self) -> list:
        cnt = C.c_int()
        _call(self.lib.bo_ctx_profile_read, self.h, None, 0, C.byref(cnt))
        buf = (L.ProfRecord * max(cnt.value, 1))()
        _call(self.lib.bo_ctx_profile_read, self.h, buf, cnt.value, C.byref(cnt))
        out = []
        for r in list(buf)[: cnt.value]:
            out.append({"kind": self.lib.bo_pass_kind_name(r.kind).decode(), "k": r.k, "p": r.p, "mh": r.mh,
                        "rows": r.rows, "bytes": r.bytes, "ms": r.ms})
        return out

    def close(self):
        if getattr(self, "h", None):
            for ch in list(self._children):
                ch.close()
            self.lib.bo_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ld_of(p) -> int:
    return int(p.stride(0)) if p.dim() == 2 else int(p.shape[0])


def _ptr(p):
    return C.c_void_p(p.data_ptr())


# ----------------------------------------------------------------- sketch --
class SketchOperator:
    """SketchOperator (sketch.hpp:25-55), generated on the GPU."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        ctx._children.add(self)

    @classmethod
    def build(cls, ctx: Context, kind, n: int, shat: int, seed: int):
        if isinstance(kind, str):
            if kind not in SKETCHES:
                raise InvalidScheme(f"unknown sketch kind '{kind}'")
            kind = SKETCHES[kind]
        h = C.c_void_p()
        _call(ctx.lib.bo_sketch_build, ctx.h, kind, n, shat, seed, C.byref(h))
        return cls(ctx, h)

    @classmethod
    def from_dense(cls, ctx: Context, theta):
        h = C.c_void_p()
        _call(ctx.lib.bo_sketch_from_dense, ctx.h, _ptr(theta), _ld_of(theta), theta.shape[0], C.byref(h))
        return cls(ctx, h)

    def sketch_size(self) -> int:
        return int(self.ctx.lib.bo_sketch_size(self.h))

    def count_width(self) -> int:
        return int(self.ctx.lib.bo_sketch_count_width(self.h))

    def kind(self) -> int:
        return int(self.ctx.lib.bo_sketch_kind(self.h))

    def apply(self, v, ledger: ReduceLedger | None = None) -> np.ndarray:
        k = v.shape[0]
        out = np.zeros((self.sketch_size(), k), order="F")
        led = _ledger_in(ledger)
        _call(self.ctx.lib.bo_sketch_apply, self.h, _ptr(v), _ld_of(v), k, _dp(out), led)
        _ledger_out(ledger, led)
        return out

    def dense_stage(self) -> np.ndarray:
        out = np.zeros((self.ctx.n_local, self.sketch_size()), order="F")
        _call(self.ctx.lib.bo_sketch_dense_to_host, self.h, _dp(out))
        return out

    def count_stage(self):
        b = np.zeros(self.ctx.n_local, dtype=np.uint32)
        s = np.zeros(self.ctx.n_local)
        _call(self.ctx.lib.bo_sketch_count_to_host, self.h, b.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(s))
        return b, s

    def gauss_stage(self) -> np.ndarray:
        out = np.zeros((self.count_width(), self.sketch_size()), order="F")
        _call(self.ctx.lib.bo_sketch_gauss_stage_to_host, self.h, _dp(out))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.bo_sketch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ intra-orth --
@dataclass
class QrResult:
    q: object          # device panel (k, ld)
    r: np.ndarray      # k x k upper


def _intra(fn_name, ctx: Context, v, ledger, theta=None, q=None):
    k = v.shape[0]
    q = ctx.panel(k, zero=False) if q is None else q
    r = np.zeros((k, k), order="F")
    led = _ledger_in(ledger)
    fn = getattr(ctx.lib, fn_name)
    try:
        if theta is None:
            _call(fn, ctx.h, _ptr(v), _ld_of(v), k, _ptr(q), _ld_of(q), _dp(r), led)
        else:
            _call(fn, ctx.h, _ptr(v), _ld_of(v), k, theta.h, _ptr(q), _ld_of(q), _dp(r), led)
    finally:  # ledger events before a breakdown stay counted
        _ledger_out(ledger, led)
    return QrResult(q, r)


def cholqr(ctx: Context, v, ledger: ReduceLedger | None = None, q=None) -> QrResult:
    return _intra("bo_cholqr", ctx, v, ledger, q=q)


def cholqr2(ctx: Context, v, ledger: ReduceLedger | None = None, q=None) -> QrResult:
    return _intra("bo_cholqr2", ctx, v, ledger, q=q)


def rand_cholqr(ctx: Context, v, theta: SketchOperator, ledger: ReduceLedger | None = None, q=None) -> QrResult:
    return _intra("bo_rand_cholqr", ctx, v, ledger, theta=theta, q=q)


@dataclass
class RecursiveQr:
    q: object
    coeffs: np.ndarray
    kept: list
    discarded: list
    discard_norm: list
    depth: int


def recursive_cholqr(ctx: Context, v, ledger: ReduceLedger | None = None) -> RecursiveQr:
    k = v.shape[0]
    q = ctx.panel(k)
    coeffs = np.zeros((k, k), order="F")
    kept = (C.c_uint64 * k)()
    disc = (C.c_uint64 * k)()
    dn = np.zeros(k)
    nk, nd, depth = C.c_uint64(), C.c_uint64(), C.c_uint64()
    led = _ledger_in(ledger)
    try:
        _call(ctx.lib.bo_recursive_cholqr, ctx.h, _ptr(v), _ld_of(v), k, _ptr(q), _ld_of(q), _dp(coeffs), kept,
              C.byref(nk), disc, _dp(dn), C.byref(nd), C.byref(depth), led)
    finally:
        _ledger_out(ledger, led)
    return RecursiveQr(q[: nk.value], coeffs[: nk.value, :].copy(), list(kept)[: nk.value],
                       list(disc)[: nd.value], list(dn[: nd.value]), depth.value)


def gram(ctx: Context, v, ledger: ReduceLedger | None = None) -> np.ndarray:
    k = v.shape[0]
    g = np.zeros((k, k), order="F")
    led = _ledger_in(ledger)
    _call(ctx.lib.bo_gram, ctx.h, _ptr(v), _ld_of(v), k, _dp(g), led)
    _ledger_out(ledger, led)
    return g


def apply_inv_upper(ctx: Context, v, r: np.ndarray, x=None):
    k = v.shape[0]
    r = np.asfortranarray(r, dtype=np.float64)
    x = ctx.panel(k) if x is None else x
    _call(ctx.lib.bo_apply_inv_upper, ctx.h, _ptr(v), _ld_of(v), k, _dp(r), _ptr(x), _ld_of(x))
    return x


# ------------------------------------------------------------ BasisStore --
class BasisStore:
    """BasisStore (block_orth.hpp:27-102): device Q slab, host R / C mirror."""

    def __init__(self, ctx: Context, capacity: int):
        self.ctx = ctx
        h = C.c_void_p()
        _call(ctx.lib.bo_basis_create, ctx.h, capacity, C.byref(h))
        self.h = h
        self.capacity = capacity
        ctx._children.add(self)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.bo_basis_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        self.ctx.lib.bo_basis_reset(self.h)

    def sync(self):
        """complete the deferred bcgs2 calls (bo_basis_sync); raises the first
        failure with .call = the index of the failing call"""
        failed = C.c_uint64()
        st = L.Status()
        rc = self.ctx.lib.bo_basis_sync(self.h, C.byref(failed), C.byref(st))
        if rc != 0:
            try:
                _raise(rc, st)
            except Error as e:
                e.call = int(failed.value)
                raise

    def cols(self) -> int:
        return int(self.ctx.lib.bo_basis_cols(self.h))

    def ledger(self) -> ReduceLedger:
        a = (C.c_uint64 * 4)()
        self.ctx.lib.bo_basis_ledger(self.h, a)
        return ReduceLedger(list(a))

    def q_device(self):
        """torch view of the device slab, shape (capacity, ld)."""
        t = self.ctx.torch
        ld = C.c_uint64()
        ptr = self.ctx.lib.bo_basis_q_device(self.h, C.byref(ld))
        return _TorchView.make(t, ptr, self.capacity, ld.value, self.ctx.device)

    def basis_copy(self) -> np.ndarray:
        c = self.cols()
        out = np.zeros((self.ctx.n_local, c), order="F")
        if c:
            _call(self.ctx.lib.bo_basis_cols_to_host, self.h, 0, c, _dp(out))
        return out

    def basis_col(self, j: int) -> np.ndarray:
        out = np.zeros((self.ctx.n_local, 1), order="F")
        _call(self.ctx.lib.bo_basis_cols_to_host, self.h, j, j + 1, _dp(out))
        return out[:, 0]

    def r_copy(self) -> np.ndarray:
        c = self.cols()
        out = np.zeros((c, c), order="F")
        self.ctx.lib.bo_basis_r_copy(self.h, _dp(out))
        return out

    def r_entry(self, i, j) -> float:
        return float(self.ctx.lib.bo_basis_r_entry(self.h, i, j))

    def c_copy(self) -> np.ndarray:
        c = self.cols()
        out = np.zeros((c, c), order="F")
        self.ctx.lib.bo_basis_c_copy(self.h, _dp(out))
        return out

    def mark_seed(self, col: int):
        self.ctx.lib.bo_basis_mark_seed(self.h, col)

    def is_seed(self, col: int) -> bool:
        return bool(self.ctx.lib.bo_basis_is_seed(self.h, col))

    def input_coeff_col(self, k: int, length: int) -> np.ndarray:
        out = np.zeros(length)
        self.ctx.lib.bo_basis_input_coeff_col(self.h, k, length, _dp(out))
        return out

    def begin_big_panel(self, sketch_rows: int, overlap: bool = False):
        self.ctx.lib.bo_basis_begin_big_panel(self.h, sketch_rows, int(overlap))

    def big_panel_lo(self) -> int:
        return int(self.ctx.lib.bo_basis_big_panel_lo(self.h))

    def panel_boundaries(self) -> list:
        nb = int(self.ctx.lib.bo_basis_num_boundaries(self.h))
        a = (C.c_uint64 * max(nb, 1))()
        self.ctx.lib.bo_basis_boundaries(self.h, a)
        return list(a)[:nb]

    def sketched(self) -> np.ndarray:
        rows = C.c_uint64()
        cols = int(self.ctx.lib.bo_basis_sketched(self.h, None, C.byref(rows)))
        out = np.zeros((rows.value, cols), order="F")
        if rows.value * cols:
            self.ctx.lib.bo_basis_sketched(self.h, _dp(out), C.byref(rows))
        return out


class _TorchView:
    @staticmethod
    def make(torch, ptr, rows, ld, device):
        # wrap a raw device pointer as a torch tensor (no ownership)
        class _Holder:
            def __init__(self, ptr, nbytes):
                self.__cuda_array_interface__ = {
                    "shape": (rows, ld), "typestr": "<f8", "data": (ptr, False), "version": 3,
                    "strides": None,
                }
        return torch.as_tensor(_Holder(ptr, rows * ld * 8), device=device)


@dataclass
class ProjectResult:
    vhat: object
    coeffs: np.ndarray


def bcgs_project_range(store: BasisStore, v, lo: int, hi: int, vhat=None) -> ProjectResult:
    ctx = store.ctx
    k = v.shape[0]
    vhat = ctx.panel(k) if vhat is None else vhat
    coeffs = np.zeros((hi - lo, k), order="F")
    _call(ctx.lib.bo_bcgs_project_range, store.h, _ptr(v), _ld_of(v), k, lo, hi, _ptr(vhat), _ld_of(vhat),
          _dp(coeffs))
    return ProjectResult(vhat, coeffs)


def bcgs_project(store: BasisStore, v) -> ProjectResult:
    return bcgs_project_range(store, v, 0, store.cols())


def bcgs2(store: BasisStore, v, intra=CHOLQR2, theta: SketchOperator | None = None, overlap: bool = False,
          defer: bool = False):
    """bcgs2 (block_orth.hpp:123).  defer=True enqueues the call without a
    host wait (bo_bcgs2_enqueue): errors surface at store.sync(), which raises
    the first failing call's exception with .call = its index."""
    fn = store.ctx.lib.bo_bcgs2_enqueue if defer else store.ctx.lib.bo_bcgs2
    _call(fn, store.h, _ptr(v), _ld_of(v), v.shape[0], intra, theta.h if theta is not None else None, int(overlap))


def bcgs_pip(store: BasisStore, v, overlap: bool = False):
    _call(store.ctx.lib.bo_bcgs_pip, store.h, _ptr(v), _ld_of(v), v.shape[0], int(overlap))


def rand_bcgs_preproc(store: BasisStore, v, theta: SketchOperator, overlap: bool = False):
    _call(store.ctx.lib.bo_rand_bcgs_preproc, store.h, _ptr(v), _ld_of(v), v.shape[0], theta.h, int(overlap))


def two_stage_panel(store: BasisStore, v, preproc, theta: SketchOperator | None = None, overlap: bool = False):
    _call(store.ctx.lib.bo_two_stage_panel, store.h, _ptr(v), _ld_of(v), v.shape[0], preproc,
          theta.h if theta is not None else None, int(overlap))


def two_stage_finish(store: BasisStore, preproc, reorthogonalize=True, record_condition=False):
    stats = np.zeros(2)
    _call(store.ctx.lib.bo_two_stage_finish, store.h, preproc, int(reorthogonalize), int(record_condition),
          _dp(stats))
    return {"preproc_condition": stats[0], "sketched_orth_error": stats[1]}


def two_stage_cycle(store: BasisStore, panels, preproc, theta=None, reorthogonalize=True, overlap=False,
                    record_condition=False):
    """block_orth.cpp:382-389"""
    store.begin_big_panel(theta.sketch_size() if theta is not None else 0, overlap)
    for v in panels:
        two_stage_panel(store, v, preproc, theta, overlap)
    return two_stage_finish(store, preproc, reorthogonalize, record_condition)


# --------------------------------------------------------- MatrixMarket --
def read_matrix_market(path) -> tuple:
    """read_matrix_market (sparse.cpp:88-136): (nrows, ncols, row_ptr, col, val)
    of the CSR CsrMatrix::from_triplets builds; raises ParseError / BannerError
    with the reference's messages.  Host-only."""
    lib = L.load()
    h = C.c_void_p()
    _call(lib.bo_mm_read, str(path).encode(), C.byref(h))
    try:
        nr, nc, nnz = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib.bo_csr_host_info(h, C.byref(nr), C.byref(nc), C.byref(nnz))
        rp = np.zeros(nr.value + 1, dtype=np.int64)
        ci = np.zeros(nnz.value, dtype=np.int64)
        vv = np.zeros(nnz.value)
        lib.bo_csr_host_arrays(h, rp.ctypes.data_as(C.POINTER(C.c_int64)), ci.ctypes.data_as(C.POINTER(C.c_int64)),
                               _dp(vv))
    finally:
        lib.bo_csr_host_destroy(h)
    return nr.value, nc.value, rp, ci, vv


def write_matrix_market(path, nrows: int, ncols: int, row_ptr, col, val):
    """write_matrix_market (sparse.cpp:138-152)"""
    lib = L.load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col, dtype=np.int64)
    vv = np.ascontiguousarray(val, dtype=np.float64)
    _call(lib.bo_mm_write, str(path).encode(), nrows, ncols, rp.ctypes.data_as(C.POINTER(C.c_int64)),
          ci.ctypes.data_as(C.POINTER(C.c_int64)), _dp(vv))


# ------------------------------------------------------ C2 panel cache --
def panel_cache_write(path, a: np.ndarray, desc: str = "") -> str:
    """Raw FP64 panel cache (bo_panel_cache_write): a column-major host block
    (rows x cols) with its SHA-256 in the header; returns the hex digest."""
    lib = L.load()
    a = np.asfortranarray(a, dtype=np.float64)
    sha = C.create_string_buffer(65)
    _call(lib.bo_panel_cache_write, str(path).encode(), _dp(a), a.shape[0], a.shape[1], a.shape[0],
          desc.encode(), sha)
    return sha.value.decode()


def panel_cache_info(path) -> dict:
    lib = L.load()
    rows, cols = C.c_uint64(), C.c_uint64()
    sha, desc = C.create_string_buffer(65), C.create_string_buffer(257)
    _call(lib.bo_panel_cache_info, str(path).encode(), C.byref(rows), C.byref(cols), sha, desc)
    return {"rows": rows.value, "cols": cols.value, "sha256": sha.value.decode(), "desc": desc.value.decode()}


def panel_cache_read(path, out: np.ndarray | None = None) -> np.ndarray:
    """read a panel cache into a column-major host array, verifying the digest
    (raises Error on a size or SHA-256 mismatch)"""
    lib = L.load()
    info = panel_cache_info(path)
    if out is None:
        out = np.empty((info["rows"], info["cols"]), order="F")
    _call(lib.bo_panel_cache_read, str(path).encode(), _dp(out), out.shape[0], out.shape[1], out.shape[0])
    return out


def sha256(a: np.ndarray) -> str:
    """SHA-256 of an array's bytes in memory order (bo_sha256)"""
    lib = L.load()
    a = np.ascontiguousarray(a) if not a.flags.f_contiguous else a
    out = C.create_string_buffer(65)
    lib.bo_sha256(a.ctypes.data_as(C.c_void_p), a.nbytes, out)
    return out.value.decode()


def gen_glued(ctx: Context, num_panels: int, panel_width: int, kappa_panel: float, kappa_global: float,
              seed: int):
    """gen_glued (problems.cpp:21-61) over the context's n global rows,
    bit-identical to the reference; returns the rank's rows as a device panel
    (num_panels * panel_width, ld)."""
    out = ctx.panel(num_panels * panel_width, zero=False)
    ctx.stream.synchronize()
    _call(ctx.lib.bo_gen_glued, ctx.h, ctx.n, num_panels, panel_width, float(kappa_panel), float(kappa_global),
          seed, _ptr(out), ctx.ld)
    return out


COST_SCHEMES = {"standard": 0, "sstep": 1, "sketch_eq_s": 2, "sketch_between": 3, "sketch_eq_m": 4}


def eval_cost(scheme, n: int, m: int, s: int = 1, shat: int = 1, mhat: int = 0) -> dict:
    """eval_cost (cost_model.hpp:39): the per-restart-cycle cost-table entries
    as exact integers; raises InvalidScheme with the reference's messages."""
    if isinstance(scheme, str):
        if scheme not in COST_SCHEMES:
            raise InvalidScheme(f"unknown cost scheme '{scheme}'")
        scheme = COST_SCHEMES[scheme]
    out = (C.c_int64 * 5)()
    _call(L.load().bo_cost_eval, scheme, n, m, s, shat, mhat, C.cast(out, C.c_void_p))
    return dict(zip(("flops_total", "flops_second", "latency", "volume", "storage"), list(out)))


# -------------------------------------------------------------- operator --
def convdiff_coeffs(w: float = 0.3):
    """7-point coefficients (i-1, j-1, l-1, self, l+1, j+1, i+1) of the config-5
    convection-diffusion operator: -Laplace(u) + b . grad(u), constant wind b
    along (1, 1, 1), central differences, cell Peclet w = b h / 2."""
    lo, hi = -1.0 - w, -1.0 + w
    return np.array([lo, lo, lo, 6.0, hi, hi, hi])

class Operator:
    """CsrMatrix rows of this shard (or the matrix-free Laplacian) on device."""

    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        ctx._children.add(self)

    @classmethod
    def csr(cls, ctx: Context, ncols: int, row_ptr, col, val):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col, dtype=np.int64)
        vv = np.ascontiguousarray(val, dtype=np.float64)
        h = C.c_void_p()
        _call(ctx.lib.bo_op_csr, ctx.h, ncols, rp.ctypes.data_as(C.POINTER(C.c_int64)),
              ci.ctypes.data_as(C.POINTER(C.c_int64)), _dp(vv), C.byref(h))
        return cls(ctx, h)

    @classmethod
    def laplace(cls, ctx: Context, dims: int, k: int):
        h = C.c_void_p()
        _call(ctx.lib.bo_op_laplace, ctx.h, dims, k, C.byref(h))
        return cls(ctx, h)

    @classmethod
    def stencil(cls, ctx: Context, dims: int, k: int, coeffs):
        """constant-coefficient 5/7-point stencil, coeffs in ascending column order"""
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        if c.shape != (2 * dims + 1,):
            raise ValueError(f"need {2 * dims + 1} stencil coefficients")
        h = C.c_void_p()
        _call(ctx.lib.bo_op_stencil, ctx.h, dims, k, _dp(c), C.byref(h))
        return cls(ctx, h)

    @classmethod
    def convdiff(cls, ctx: Context, k: int, w: float = 0.3):
        """config 5: nonsymmetric 3D convection-diffusion, central differences
        (diagonal 6, lower neighbours -1-w, upper neighbours -1+w)"""
        return cls.stencil(ctx, 3, k, convdiff_coeffs(w))

    def spmv(self, x, y=None):
        y = self.ctx.panel(1) if y is None else y
        _call(self.ctx.lib.bo_spmv, self.h, _ptr(x), _ptr(y))
        return y

    def mpk(self, v0, s: int, v=None):
        v = self.ctx.panel(s + 1) if v is None else v
        _call(self.ctx.lib.bo_mpk, self.h, _ptr(v0), s, _ptr(v), _ld_of(v))
        return v

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.bo_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sstep_gmres_solve(op: Operator, b, x0, *, m=60, s=5, shat=60, scheme="bcgs2_cholqr2", sketch="gaussian",
                      rel_tol=1e-6, max_restarts=50, seed=0, reorthogonalize=True, diagnostics=True):
    """sstep_gmres_solve (gmres.hpp:92): returns (x device vector, report dict)."""
    ctx = op.ctx
    cfg = L.SolverConfig(n=ctx.n, m=m, s=s, shat=shat,
                         scheme=SCHEMES[scheme] if isinstance(scheme, str) else scheme,
                         sketch=SKETCHES[sketch] if isinstance(sketch, str) else sketch,
                         rel_tol=rel_tol, max_restarts=max_restarts, seed=seed,
                         reorthogonalize=int(reorthogonalize), diagnostics=int(diagnostics))
    rep = L.SolveReport()
    x = ctx.panel(1)
    _call(ctx.lib.bo_sstep_gmres, op.h, _ptr(b), _ptr(x0), C.byref(cfg), _ptr(x), C.byref(rep))
    nh = rep.nhist
    out = {
        "converged": bool(rep.converged), "breakdown": bool(rep.breakdown),
        "happy_breakdown": bool(rep.happy_breakdown),
        "breakdown_detail": rep.breakdown_detail.decode(errors="replace"),
        "restarts": rep.restarts, "iterations": rep.iterations,
        "initial_residual": rep.initial_residual, "final_relres": rep.final_relres,
        "reduce": list(rep.reduce), "reduce_total": rep.reduce_total,
        "restart_relres": list(rep.relres)[:nh], "restart_lsq_residual": list(rep.lsq)[:nh],
        "restart_orth_error": list(rep.orth)[:nh], "restart_arnoldi_resid": list(rep.arnoldi)[:nh],
        "t_ms": {"sketch": rep.t_sketch, "mpk": rep.t_mpk, "orth": rep.t_orth, "update": rep.t_update,
                 "residual": rep.t_residual, "diag": rep.t_diag, "cycles": rep.t_cycles},
    }
    return x, out
