"""ctypes binding of the C ABI in include/bo_cuda.h (libbo_cuda.so).

The library is loaded from this package directory (built in-tree by
paper_2503_16717_b200._build).  There is no fallback: if the extension is
missing or no sm_100 GPU is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libbo_cuda.so"

u64 = C.c_uint64
i64 = C.c_int64
dp = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("index", C.c_longlong), ("pivot", C.c_double), ("msg", C.c_char * 256)]


class SolverConfig(C.Structure):
    _fields_ = [
        ("n", u64), ("m", u64), ("s", u64), ("shat", u64),
        ("scheme", C.c_int), ("sketch", C.c_int),
        ("rel_tol", C.c_double), ("max_restarts", u64), ("seed", u64),
        ("reorthogonalize", C.c_int), ("diagnostics", C.c_int),
    ]


class SolveReport(C.Structure):
    _fields_ = [
        ("converged", C.c_int), ("breakdown", C.c_int), ("happy_breakdown", C.c_int),
        ("breakdown_detail", C.c_char * 256),
        ("restarts", u64), ("iterations", u64),
        ("initial_residual", C.c_double), ("final_relres", C.c_double),
        ("reduce", u64 * 4), ("reduce_total", u64), ("nhist", u64),
        ("relres", C.c_double * 256), ("lsq", C.c_double * 256),
        ("orth", C.c_double * 256), ("arnoldi", C.c_double * 256),
        ("t_sketch", C.c_double), ("t_mpk", C.c_double), ("t_orth", C.c_double),
        ("t_update", C.c_double), ("t_residual", C.c_double), ("t_diag", C.c_double),
        ("t_cycles", C.c_double),
    ]


class P2pOp(C.Structure):
    _fields_ = [("peer", C.c_int), ("is_send", C.c_int), ("buf", C.c_void_p), ("count", u64)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, u64, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, u64, C.c_void_p, C.c_void_p)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(P2pOp), C.c_void_p)


class CommOps(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum_f64", ALLREDUCE_FN), ("allgather_u64", ALLGATHER_FN),
                ("exchange_f64", EXCHANGE_FN)]


class ProfRecord(C.Structure):
    _fields_ = [("kind", C.c_int), ("k", C.c_int), ("p", C.c_int), ("mh", C.c_int), ("rows", u64),
                ("bytes", u64), ("ms", C.c_float)]


SP = C.POINTER(Status)

# name: (restype, argtypes)
_SIGS = {
    "bo_abi_version": (C.c_int, []),
    "bo_nccl_id_bytes": (C.c_int, []),
    "bo_nccl_get_unique_id": (C.c_int, [vp, SP]),
    "bo_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, u64, u64, u64, vp, C.POINTER(vp), SP]),
    "bo_ctx_create_comm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(CommOps), u64, u64, u64, vp,
                                     C.POINTER(vp), SP]),
    "bo_ctx_destroy": (C.c_int, [vp]),
    "bo_ctx_synchronize": (C.c_int, [vp, SP]),
    "bo_ctx_local_rows": (u64, [vp]),
    "bo_ctx_ld": (u64, [vp]),
    "bo_ctx_kernel_launches": (u64, [vp]),
    "bo_ctx_allreduces": (u64, [vp]),
    "bo_ctx_profile": (C.c_int, [vp, C.c_int]),
    "bo_ctx_profile_read": (C.c_int, [vp, C.POINTER(ProfRecord), C.c_int, C.POINTER(C.c_int), SP]),
    "bo_pass_kind_name": (C.c_char_p, [C.c_int]),
    "bo_sketch_build": (C.c_int, [vp, C.c_int, u64, u64, u64, C.POINTER(vp), SP]),
    "bo_sketch_from_dense": (C.c_int, [vp, vp, u64, u64, C.POINTER(vp), SP]),
    "bo_sketch_destroy": (C.c_int, [vp]),
    "bo_sketch_size": (u64, [vp]),
    "bo_sketch_count_width": (u64, [vp]),
    "bo_sketch_kind": (C.c_int, [vp]),
    "bo_sketch_dense_to_host": (C.c_int, [vp, dp, SP]),
    "bo_sketch_count_to_host": (C.c_int, [vp, C.POINTER(C.c_uint32), dp, SP]),
    "bo_sketch_gauss_stage_to_host": (C.c_int, [vp, dp, SP]),
    "bo_sketch_apply": (C.c_int, [vp, vp, u64, u64, dp, u64p, SP]),
    "bo_cholqr": (C.c_int, [vp, vp, u64, u64, vp, u64, dp, u64p, SP]),
    "bo_cholqr2": (C.c_int, [vp, vp, u64, u64, vp, u64, dp, u64p, SP]),
    "bo_rand_cholqr": (C.c_int, [vp, vp, u64, u64, vp, vp, u64, dp, u64p, SP]),
    "bo_recursive_cholqr": (C.c_int, [vp, vp, u64, u64, vp, u64, dp, u64p, u64p, u64p, dp, u64p, u64p, u64p, SP]),
    "bo_gram": (C.c_int, [vp, vp, u64, u64, dp, u64p, SP]),
    "bo_apply_inv_upper": (C.c_int, [vp, vp, u64, u64, dp, vp, u64, SP]),
    "bo_basis_create": (C.c_int, [vp, u64, C.POINTER(vp), SP]),
    "bo_basis_destroy": (C.c_int, [vp]),
    "bo_basis_reset": (C.c_int, [vp]),
    "bo_basis_cols": (u64, [vp]),
    "bo_basis_capacity": (u64, [vp]),
    "bo_basis_q_device": (vp, [vp, u64p]),
    "bo_basis_ledger": (C.c_int, [vp, u64p]),
    "bo_basis_r_copy": (C.c_int, [vp, dp]),
    "bo_basis_r_entry": (C.c_double, [vp, u64, u64]),
    "bo_basis_c_copy": (C.c_int, [vp, dp]),
    "bo_basis_mark_seed": (C.c_int, [vp, u64]),
    "bo_basis_is_seed": (C.c_int, [vp, u64]),
    "bo_basis_input_coeff_col": (C.c_int, [vp, u64, u64, dp]),
    "bo_basis_begin_big_panel": (C.c_int, [vp, u64, C.c_int]),
    "bo_basis_big_panel_lo": (u64, [vp]),
    "bo_basis_num_boundaries": (u64, [vp]),
    "bo_basis_boundaries": (C.c_int, [vp, u64p]),
    "bo_basis_sketched": (u64, [vp, dp, u64p]),
    "bo_basis_cols_to_host": (C.c_int, [vp, u64, u64, dp, SP]),
    "bo_bcgs2_enqueue": (C.c_int, [vp, vp, u64, u64, C.c_int, vp, C.c_int, SP]),
    "bo_basis_sync": (C.c_int, [vp, u64p, SP]),
    "bo_basis_last_push": (C.c_int, [vp, u64p, u64p, C.POINTER(C.c_int), dp, dp]),
    "bo_basis_import": (C.c_int, [vp, u64, dp, u64, dp, dp, C.POINTER(C.c_ubyte), u64p, u64, SP]),
    "bo_bcgs_project_range": (C.c_int, [vp, vp, u64, u64, u64, u64, vp, u64, dp, SP]),
    "bo_bcgs2": (C.c_int, [vp, vp, u64, u64, C.c_int, vp, C.c_int, SP]),
    "bo_bcgs_pip": (C.c_int, [vp, vp, u64, u64, C.c_int, SP]),
    "bo_rand_bcgs_preproc": (C.c_int, [vp, vp, u64, u64, vp, C.c_int, SP]),
    "bo_two_stage_panel": (C.c_int, [vp, vp, u64, u64, C.c_int, vp, C.c_int, SP]),
    "bo_two_stage_finish": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dp, SP]),
    "bo_op_csr": (C.c_int, [vp, u64, C.POINTER(i64), C.POINTER(i64), dp, C.POINTER(vp), SP]),
    "bo_op_laplace": (C.c_int, [vp, C.c_int, u64, C.POINTER(vp), SP]),
    "bo_cost_eval": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, SP]),
    "bo_gen_glued": (C.c_int, [vp, u64, u64, u64, C.c_double, C.c_double, u64, vp, u64, SP]),
    "bo_op_stencil": (C.c_int, [vp, C.c_int, u64, dp, C.POINTER(vp), SP]),
    "bo_op_destroy": (C.c_int, [vp]),
    "bo_mm_read": (C.c_int, [C.c_char_p, C.POINTER(vp), SP]),
    "bo_csr_host_info": (C.c_int, [vp, u64p, u64p, u64p]),
    "bo_csr_host_arrays": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), dp]),
    "bo_csr_host_destroy": (C.c_int, [vp]),
    "bo_mm_write": (C.c_int, [C.c_char_p, u64, u64, C.POINTER(C.c_int64), C.POINTER(C.c_int64), dp, SP]),
    "bo_spmv": (C.c_int, [vp, vp, vp, SP]),
    "bo_mpk": (C.c_int, [vp, vp, u64, vp, u64, SP]),
    "bo_sstep_gmres": (C.c_int, [vp, vp, vp, C.POINTER(SolverConfig), vp, C.POINTER(SolveReport), SP]),
    "bo_mt64_jump_window": (C.c_int, [u64, u64, u64p]),
    "bo_panel_cache_write": (C.c_int, [C.c_char_p, dp, u64, u64, u64, C.c_char_p, C.c_char_p, SP]),
    "bo_panel_cache_info": (C.c_int, [C.c_char_p, u64p, u64p, C.c_char_p, C.c_char_p, SP]),
    "bo_panel_cache_read": (C.c_int, [C.c_char_p, dp, u64, u64, u64, SP]),
    "bo_sha256": (C.c_int, [C.c_void_p, u64, C.c_char_p]),
}

_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libbo_cuda.so (in-tree).  Raises if it is missing — no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("BO_LIB", LIB_PATH))  # BO_LIB: experiment builds
    if not p.exists():
        raise RuntimeError(
            f"CUDA extension {p} is missing: run `python -m paper_2503_16717_b200._build` "
            "(there is no CPU fallback for the block-orthogonalization path)")
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)
