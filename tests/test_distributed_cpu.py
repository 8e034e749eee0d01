"""CPU, world size 2 over gloo: the row-sharded decomposition the multi-GPU
path uses (contiguous row shards, per-rank partial sums, ONE all-reduce per
reference ledger event, tiny factorizations replicated on every rank) gives
the single-process reference result, and each rank regenerates exactly its
own rows of the Count sketch from a jumped MT19937-64 window.

The numerics here are numpy stand-ins for the device kernels; what is tested
is the sharding / collective logic (which rows, which partial sums, how many
all-reduces, what is replicated)."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import ctypes as C

    import torch
    import torch.distributed as dist
    from py_oracle import Oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    orc = Oracle("orc")
    n, k, panels = 6000, 6, 4
    v = orc.gen_glued(n, panels, k, 1e4, 1e4, 13)  # every rank builds the same global input
    a, b = n * rank // world, n * (rank + 1) // world
    allreduces = 0

    def allreduce(x):
        nonlocal allreduces
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        allreduces += 1
        return t.numpy()

    def chol(g):
        r, f, _ = orc.cholesky(g)
        assert f == 0
        return r

    # sharded BCGS2 with CholQR2 intra (block_orth.cpp:207-226), local rows only
    Q = np.zeros((b - a, 0))
    R = np.zeros((panels * k, panels * k))
    for p in range(panels):
        V = v[a:b, p * k:(p + 1) * k]
        if Q.shape[1] == 0:
            G1 = allreduce(V.T @ V)                       # gram
            R1 = chol(G1)
            Y = V @ np.linalg.inv(R1)
            R2 = chol(allreduce(Y.T @ Y))                 # gram
            Qn = Y @ np.linalg.inv(R2)
            R[:k, :k] = R2 @ R1
        else:
            C1 = allreduce(Q.T @ V)                       # projection
            Vh = V - Q @ C1
            R1 = chol(allreduce(Vh.T @ Vh))               # gram
            Y = Vh @ np.linalg.inv(R1)
            R2 = chol(allreduce(Y.T @ Y))                 # gram
            Qh = Y @ np.linalg.inv(R2)
            C2 = allreduce(Q.T @ Qh)                      # projection
            Z = Qh - Q @ C2
            R3 = chol(allreduce(Z.T @ Z))                 # gram
            Qn = Z @ np.linalg.inv(R3)
            c0 = Q.shape[1]
            Rin = R2 @ R1
            R[:c0, c0:c0 + k] = C1 + C2 @ Rin
            R[c0:c0 + k, c0:c0 + k] = R3 @ Rin
        Q = np.hstack([Q, Qn])

    # shard-local Count-sketch rows from the jumped stream (bo_sketch_build)
    import paper_2503_16717_b200 as P
    lib = P._lib.load()
    seed = 4242
    width = 2 * 11 * 11
    mt_seed = orc.derive_seed(seed, 0)
    buckets = []
    for row0 in range(a, b, 156):
        out = (C.c_uint64 * 312)()
        lib.bo_mt64_jump_window(mt_seed, 2 * row0, out)
        m = (1 << 64) - 1
        for t in range(min(156, b - row0)):
            y = out[2 * t]
            y ^= (y >> 29) & 0x5555555555555555
            y ^= (y << 17) & 0x71D67FFFEDA60000 & m
            y ^= (y << 37) & 0xFFF7EEE000000000 & m
            y ^= y >> 43
            buckets.append(((y & m) * width) >> 64)
    q.put((rank, Q, R, allreduces, np.array(buckets)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    return res


def test_sharded_bcgs2_matches_single_process(sharded, orc):
    n, k, panels = 6000, 6, 4
    v = orc.gen_glued(n, panels, k, 1e4, 1e4, 13)
    ob = orc.basis_new(n, panels * k)
    for p in range(panels):
        assert orc.bcgs2(ob, v[:, p * k:(p + 1) * k], 0, None).code == 0
    qo, _, led = orc.basis_state(ob, n)
    ro = orc.basis_r(ob, panels * k)
    Q = np.vstack([sharded[0][1], sharded[1][1]])
    R0, R1 = sharded[0][2], sharded[1][2]
    assert np.array_equal(R0, R1)  # replicated tiny factorizations agree bit for bit on every rank
    assert np.max(np.abs(Q - qo)) < 1e-9
    assert np.max(np.abs(R0 - ro)) / np.max(np.abs(ro)) < 1e-10
    # one all-reduce per reference ledger event: 2 + 5 per later panel
    assert sharded[0][3] == sharded[1][3] == sum(led) == 2 + 5 * (panels - 1)


def test_count_sketch_shards_concatenate_to_reference(sharded, orc):
    n = 6000
    h = orc.sketch_build(1, n, 10, 4242).h
    bo, _ = orc.sketch_count(h, n)
    got = np.concatenate([sharded[0][4], sharded[1][4]])
    assert np.array_equal(got, bo)
