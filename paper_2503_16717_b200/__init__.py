"""B200-native (sm_100a) block-orthogonalization hot path of arXiv 2503.16717.

A drop-in for the reference blkorth library's orthogonalization/operator
interface: the CUDA kernels and their C ABI live in libbo_cuda.so
(csrc/, include/bo_cuda.h); `borth` mirrors the reference interface in
Python for tests and benchmarks.
"""
from . import _lib  # noqa: F401
from .borth import (  # noqa: F401
    AllColumnsDiscarded, AmbientTooSmall, BasisStore, CholeskyBreakdown, Context, CudaError, Error,
    InvalidScheme, NcclError, Operator, ProjectResult, QrResult, RankDeficient, RecursiveQr, ReduceLedger,
    SingularTriangular, SketchOperator, ZeroMatrix, apply_inv_upper, bcgs2, bcgs_pip, bcgs_project,
    bcgs_project_range, cholqr, cholqr2, eval_cost, gen_glued, gram, rand_bcgs_preproc, rand_cholqr, recursive_cholqr,
    sstep_gmres_solve, two_stage_cycle, two_stage_finish, two_stage_panel,
)

__all__ = [n for n in dir() if not n.startswith("_")]
