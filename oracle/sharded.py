"""CPU ORACLE -- test infrastructure only: the N-column sharded decomposition.

Restates, with numpy on each rank and torch.distributed (gloo) for the
exchange, exactly what libbnmf's multi-GPU schedule does (engine.cu /
fused_tc.cu): every rank owns a column block of V and of H, W is replicated,
and the only per-iteration exchange is one allreduce (sum) of the packed
buffer [W numerator F x K | W denominator F x K | objective] -- the same
layout as the engine's `comm` buffer.  tests/test_parallel_gloo.py runs it
with world_size 2 and checks it against the single-process oracle
(betanmf_oracle.run), which follows the reference solver.py:292-326.
"""

from __future__ import annotations

import numpy as np

from . import betanmf_oracle as O


def _allreduce(buf):
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(buf))
    dist.all_reduce(t)
    return t.numpy()


def run_sharded_jmm(v_local, beta, w0, h0_local, iters, kappa=0.0, floor=O.DEFAULT_FLOOR):
    """JMM with L = 1 over a column shard; returns (W, H_local, objectives)."""
    g = O.gamma_exponent(beta)
    vs = v_local + kappa if kappa else v_local
    wt, ht = w0.copy(), h0_local.copy()
    F, K = wt.shape
    objs = []
    for _ in range(iters):
        prod = wt @ ht + kappa
        zn, zd = O.joint_bases(vs, prod, beta)
        # W side: partial sums over the local columns, one allreduce
        num = zn @ ht.T
        den = (np.broadcast_to(ht.sum(axis=1), (F, K)) if zd is None else zd @ ht.T)
        packed = np.concatenate([num.ravel(), np.asarray(den).ravel()])
        packed = _allreduce(packed)
        num, den = packed[:F * K].reshape(F, K), packed[F * K:].reshape(F, K)
        w = wt * O.apply_exponent(O.guarded_divide(num, den, floor), g)
        # H side: column-local
        c1, c2 = O.chi1(w, wt, beta), O.chi2(w, wt, beta)
        hnum = c1.T @ zn
        hden = (np.broadcast_to(c2.sum(axis=0)[:, None], hnum.shape) if zd is None
                else c2.T @ zd)
        h = ht * O.apply_exponent(O.guarded_divide(hnum, hden, floor), g)
        obj = float(_allreduce(np.array([O.divergence_total(vs, w @ h + kappa, beta)]))[0])
        objs.append(obj)
        wt, ht = O.normalize_arrays(w, h)
    return wt, ht, np.array(objs)


def run_sharded_sparse_kl(csr_local, w0_local, h0, iters, algorithm="jmm", floor=O.DEFAULT_FLOOR):
    """Sparse KL (beta = 1) over a ROW shard of V: W rows are
    local, H is replicated.  Restates libbnmf's sparse schedule (sparse.cu):
    allreduce of [colsum W_p | sum_f W_p^2] after the W update, allreduce of
    the K x N partial H numerator, allreduce of the nonzero part of the
    objective (the dense part (1'W)(H1) is global once colsum W is).  Checked
    against the single-process restatement betanmf_oracle.run_sparse_kl."""
    import scipy.sparse as sp
    v = sp.csr_matrix(csr_local, dtype=float)
    v.sort_indices()
    rows = np.repeat(np.arange(v.shape[0]), np.diff(v.indptr))
    cols, x = v.indices, v.data
    wt, ht = np.array(w0_local, dtype=float), np.array(h0, dtype=float)
    K = wt.shape[1]

    def sddmm(wm, hm):
        return np.einsum("ik,ki->i", wm[rows], hm[:, cols])

    def zmat(vals):
        return sp.csr_matrix((vals, cols, v.indptr), shape=v.shape)

    objs = []
    for _ in range(iters):
        z = zmat(x / sddmm(wt, ht))
        w = wt * O.guarded_divide(np.asarray(z @ ht.T), ht.sum(axis=1)[None, :], floor)
        stats = _allreduce(np.concatenate([w.sum(axis=0), (w * w).sum(axis=0)]))
        colsum, sumsq = stats[:K], stats[K:]
        if algorithm == "bmm":
            z = zmat(x / sddmm(w, ht))
            hnum = _allreduce(np.asarray((z.T @ w).T))
        else:
            hnum = _allreduce(np.asarray((z.T @ wt).T))
        h = ht * O.guarded_divide(hnum, colsum[:, None], floor)
        y = sddmm(w, h)
        local = float(np.sum(x * np.log(x / y) - x))
        obj = float(_allreduce(np.array([local]))[0]) + float(colsum @ h.sum(axis=1))
        objs.append(obj)
        norms = np.sqrt(sumsq)
        wt, ht = w / norms[None, :], h * norms[:, None]
    return wt, ht, np.array(objs)
