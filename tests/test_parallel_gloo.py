"""Multi-process (world_size 2, gloo on CPU) tests of the N-sharded path:
the host plumbing in paper_2106_15214_b200.parallel and the sharded
decomposition (partial W sums + one allreduce) against the single-process
oracle.  The GPU path runs the same decomposition with NCCL."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import betanmf_oracle as O
        from oracle import sharded
        from paper_2106_15214_b200 import parallel, synthetic

        F, N, K, beta = 37, 203, 4, 1.5
        v = synthetic.config4(F=F, N=N, K=K, seed=3)
        blocks = parallel.balanced_blocks(N, world, align=4)
        n0, n1 = blocks[rank]
        off, n_global = parallel.column_offsets(n1 - n0)
        assert (off, n_global) == (n0, N)
        kappa = parallel.resolve_kappa_global(v[:, n0:n1], 0.0, None)
        assert abs(kappa - 1e-9 * v.mean()) <= 1e-15 * abs(kappa) + 1e-30
        uid = parallel.broadcast_uid(lambda: b"x" * 128)
        assert uid == b"x" * 128
        w0, h0 = synthetic.uniform_init(F, N, K, seed=5)
        w0s, h0s = parallel.slice_init(w0, h0, n0, n1 - n0, N)
        mx = parallel.allreduce_scalars([float(rank)], "max")[0]
        assert mx == world - 1
        w, h, objs = sharded.run_sharded_jmm(v[:, n0:n1], beta, w0s, h0s, iters=12)
        q.put((rank, n0, n1, w, h, objs))
    finally:
        dist.destroy_process_group()


def test_sharded_jmm_matches_single_process_oracle():
    import torch.multiprocessing as mp
    from oracle import betanmf_oracle as O
    from paper_2106_15214_b200 import synthetic

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    F, N, K, beta = 37, 203, 4, 1.5
    v = synthetic.config4(F=F, N=N, K=K, seed=3)
    w0, h0 = synthetic.uniform_init(F, N, K, seed=5)
    w_ref, h_ref, obj_ref, _, _ = O.run(v, beta, K, "jmm", kappa=0.0, tol=1e-300,
                                         max_outer_iters=12, init=(w0, h0), kkt=False)
    h = np.concatenate([r[4] for r in res], axis=1)
    for r in res:
        np.testing.assert_allclose(r[3], w_ref, rtol=1e-12)     # W replicated
        np.testing.assert_allclose(r[5], obj_ref, rtol=1e-12)   # same objective everywhere
    np.testing.assert_allclose(h, h_ref, rtol=1e-12)


def test_balanced_blocks_cover_and_align():
    from paper_2106_15214_b200 import parallel
    for n, world, align in [(4194304, 8, 65536), (203, 2, 4), (10, 3, 1), (7, 8, 1)]:
        blocks = parallel.balanced_blocks(n, world, align)
        assert blocks[0][0] == 0 and blocks[-1][1] == n
        for (a, b), (c, d) in zip(blocks, blocks[1:]):
            assert b == c and a <= b
        for a, _ in blocks:
            assert a % align == 0 or a == n


def _sparse_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scipy.sparse as sp
        from oracle import sharded
        from paper_2106_15214_b200 import parallel, synthetic

        indptr, idx, vals, shape = synthetic.config5(F=300, N=80, density=0.08, seed=11)
        csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
        F, N = shape
        f0, f1 = parallel.balanced_blocks(F, world)[rank]
        off, f_global = parallel.column_offsets(f1 - f0)
        assert (off, f_global) == (f0, F)
        w0, h0 = synthetic.uniform_init(F, N, 5, seed=8)
        out = {}
        for algo in ("jmm", "bmm"):
            out[algo] = sharded.run_sharded_sparse_kl(csr[f0:f1], w0[f0:f1], h0, iters=10,
                                                      algorithm=algo)
        q.put((rank, f0, f1, out))
    finally:
        dist.destroy_process_group()


def test_row_sharded_sparse_kl_matches_single_process_oracle():
    """The row-sharded sparse decomposition (world 2, gloo) against the
    single-process sparse restatement: W rows stitched, H replicated,
    identical objective on every rank."""
    import scipy.sparse as sp
    import torch.multiprocessing as mp
    from oracle import betanmf_oracle as O
    from paper_2106_15214_b200 import synthetic

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sparse_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    indptr, idx, vals, shape = synthetic.config5(F=300, N=80, density=0.08, seed=11)
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 5, seed=8)
    for algo in ("jmm", "bmm"):
        w_ref, h_ref, obj_ref, _ = O.run_sparse_kl(csr, 5, algo, max_outer_iters=10,
                                                   init=(w0, h0))
        w = np.concatenate([r[3][algo][0] for r in res], axis=0)
        np.testing.assert_allclose(w, w_ref, rtol=1e-11)
        for r in res:
            np.testing.assert_allclose(r[3][algo][1], h_ref, rtol=1e-11)   # H replicated
            np.testing.assert_allclose(r[3][algo][2], obj_ref, rtol=1e-12)


def _agree_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_15214_b200 import parallel
        parallel.agree_on_error(None)            # nobody failed: no error anywhere
        err = ValueError("data entries must be finite") if rank == 1 else None
        try:
            parallel.agree_on_error(err)
            q.put((rank, "no error"))
        except ValueError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_input_errors_agreed_across_ranks():
    """A check that fails on one rank only raises on every rank (the failing
    rank its own message), so no rank waits in the next collective (the
    sharded entries call this before the communicator is created)."""
    import torch.multiprocessing as mp
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] == "data entries must be finite"
    assert res[0] == "input checks failed on rank(s) [1]"
