"""Multi-GPU over NCCL: row shards on world = min(4,
device_count) GPUs, one process per GPU, collectives through the library's own
NCCL communicator (bo_ctx_create with a broadcast ncclUniqueId).  Skipped
with fewer than two GPUs (the gloo / host-transport runs of
tests/test_gpu_sharded.py cover the sharded code paths on one GPU).

  * the C2-shaped bcgs2 sequence (both intras): identical ledgers, R within
    the single-GPU contract of the unsharded run;
  * config-1 GMRES (2D Laplace 100^2, s = 5, RandCholQR): identical restart /
    iteration counts and ledgers, relres within the config-1 envelope."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import torch
    import torch.distributed as dist
    import paper_2503_16717_b200 as P
    from py_oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)  # only to broadcast the NCCL id
    torch.cuda.set_device(rank)
    obj = [P.Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out = {}
    orc = Oracle("orc")
    n, k = 60000, 11
    v = orc.gen_glued(n, 6, k, 1e6, 1e6, 7)
    r0, r1 = n * rank // world, n * (rank + 1) // world
    ctx = P.Context(n, device=rank, rank=rank, world=world, row_begin=r0, row_end=r1, nccl_id=obj[0])
    for intra in (0, 1):
        th = P.SketchOperator.build(ctx, "gaussian", n, k - 1, 1) if intra else None
        st = P.BasisStore(ctx, 6 * k)
        for p in range(6):
            P.bcgs2(st, ctx.from_host(v[r0:r1, p * k:(p + 1) * k]), intra, th, defer=True)
        st.sync()
        out[f"R{intra}"] = st.r_copy()
        out[f"led{intra}"] = st.ledger().counts
    ctx.close()
    # config 1 with a sharded matrix-free Laplacian (halo exchange over NCCL)
    obj = [P.Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    n2 = 100 * 100
    a0, a1 = 100 * (100 * rank // world), 100 * (100 * (rank + 1) // world)
    ctx = P.Context(n2, device=rank, rank=rank, world=world, row_begin=a0, row_end=a1, nccl_id=obj[0])
    op = P.Operator.laplace(ctx, 2, 100)
    _, rep = P.sstep_gmres_solve(op, ctx.from_host(np.ones(a1 - a0)), ctx.from_host(np.zeros(a1 - a0)), m=60, s=5,
                                 shat=60, scheme="bcgs2_randcholqr", diagnostics=False)
    out["gmres"] = (rep["restarts"], rep["iterations"], rep["reduce"], rep["restart_relres"])
    op.close()
    ctx.close()
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs two or more GPUs")
def test_nccl_sharded_sequence_and_gmres(gpu, orc):
    import torch.multiprocessing as mp
    world = min(4, _ngpu())
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    # single-GPU references
    n, k = 60000, 11
    v = orc.gen_glued(n, 6, k, 1e6, 1e6, 7)
    ctx = gpu.Context(n)
    for intra in (0, 1):
        th = gpu.SketchOperator.build(ctx, "gaussian", n, k - 1, 1) if intra else None
        st = gpu.BasisStore(ctx, 6 * k)
        for p in range(6):
            gpu.bcgs2(st, ctx.from_host(v[:, p * k:(p + 1) * k]), intra, th)
        R = st.r_copy()
        for r in range(world):
            assert res[r][f"led{intra}"] == st.ledger().counts
            assert np.max(np.abs(res[r][f"R{intra}"] - R)) <= 2.2e-9 * np.max(np.abs(R))
        assert all(np.array_equal(res[0][f"R{intra}"], res[r][f"R{intra}"]) for r in range(world))  # replicated bits
    ctx.close()
    csr = orc.laplace(100, 2)
    want = orc.sstep_gmres(csr, np.ones(10000), np.zeros(10000), m=60, s=5, shat=60, scheme=1, diagnostics=False)
    env = [1e-10, 1.7e-10, 3.8e-10, 5.7e-10, 8.3e-10, 8.3e-10, 5.2e-7, 3.0e-5, 9.1e-3, 1.7e-2]
    for r in range(world):
        restarts, its, led, relres = res[r]["gmres"]
        assert (restarts, its, led) == (want.restarts, want.iterations, want.reduce)
        assert all(abs(g - w) <= env[i] * w for i, (g, w) in enumerate(zip(relres, want.relres)))


def test_nccl_size1_communicator(gpu, orc):
    """The library's NCCL path on ONE GPU: a context given an NCCL id with
    world = 1 creates a size-1 communicator (ncclCommInitRank, which takes the
    128-byte ncclUniqueId by value) and routes every ledger reduction through
    ncclAllReduce followed by the 1-CTA finalize kernel (the multi-rank code
    path), the GMRES norms through the same all-reduce, and a Count sketch's
    bucket sums through it too.  A sum over one rank is the identity, so the
    results must equal the fused single-GPU path bit for bit."""
    n, k = 60000, 11
    v = orc.gen_glued(n, 6, k, 1e6, 1e6, 7)
    out = {}
    for mode in ("plain", "nccl"):
        ctx = gpu.Context(n, nccl_id=gpu.Context.nccl_unique_id() if mode == "nccl" else None)
        res = {}
        for intra, kind in ((0, None), (1, "gaussian"), (1, "count")):
            th = gpu.SketchOperator.build(ctx, kind, n, k - 1, 1) if kind else None
            st = gpu.BasisStore(ctx, 6 * k)
            a0 = ctx.allreduces
            for p in range(6):
                gpu.bcgs2(st, ctx.from_host(v[:, p * k:(p + 1) * k]), intra, th, defer=True)
            st.sync()
            res[(intra, kind)] = (st.basis_copy(), st.r_copy(), st.ledger().counts, ctx.allreduces - a0)
        ctx.close()
        ctx = gpu.Context(100 * 100, nccl_id=gpu.Context.nccl_unique_id() if mode == "nccl" else None)
        op = gpu.Operator.laplace(ctx, 2, 100)
        _, rep = gpu.sstep_gmres_solve(op, ctx.from_host(np.ones(10000)), ctx.from_host(np.zeros(10000)), m=60, s=5,
                                       shat=60, scheme="bcgs2_randcholqr", diagnostics=False)
        res["gmres"] = (rep["restarts"], rep["iterations"], rep["reduce"], rep["restart_relres"])
        op.close()
        ctx.close()
        out[mode] = res
    for key in [(0, None), (1, "gaussian"), (1, "count")]:
        q0, r0, led0, ar0 = out["plain"][key]
        q1, r1, led1, ar1 = out["nccl"][key]
        assert led0 == led1
        assert ar0 == 0 and ar1 == sum(led1), (key, ar1, led1)  # one all-reduce per ledger event
        assert np.array_equal(q0, q1) and np.array_equal(r0, r1), key
    assert out["plain"]["gmres"] == out["nccl"]["gmres"]
