"""The BASELINE configs at their full sizes on the device.

Configs 2 and 3 (8.4M / 16.8M entries) are small enough for the fp64 oracle to run a few dozen
iterations in seconds, so they are compared directly (north-star fp32 gate: objective within 1e-4
relative, monotone).  Config 4 (256 x 4 194 304) and config 5 (10^6 x 2 10^5 CSR, ~7 10^7
nonzeros) are checked through size-independent properties: a monotone trace, unit-norm W columns,
bitwise repeatability, and the last trace objective against an independent fp64 recomputation of
sum d_beta(V | W H) from the returned factors (core.py:89-114; for the sparse KL case the closed
form sum_nnz [v log(v / p) - v] + (1^T W)(H 1)), evaluated in chunks with torch on the device as
the checker.
"""

import numpy as np
import pytest
import torch

import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O
from paper_2106_15214_b200 import synthetic as syn

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.mark.parametrize("cfg", [2, 3])
def test_configs_2_3_full_size_match_oracle(cfg):
    F, N, K, beta = {2: (1024, 8192, 32, 2.0), 3: (1025, 16384, 20, 0.0)}[cfg]
    v = (syn.config2 if cfg == 2 else syn.config3)().astype(np.float32)
    assert v.shape == (F, N)
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    iters = 25
    for algo in ("jmm", "bmm"):
        c = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, tol=1e-300, max_outer_iters=iters)
        res = bn.fit(v, c, init=(w0, h0), dtype="fp32", kkt=False)
        got = np.array([r.objective for r in res.trace])
        _, _, ref, _, _ = O.run(v.astype(np.float64), beta, K, algo, tol=1e-300,
                                max_outer_iters=iters, init=(w0, h0), kkt=False)
        assert len(got) == len(ref) == iters
        assert _rel(got, ref) <= 1e-4, (cfg, algo, _rel(got, ref))
        assert np.all(got[1:] <= got[:-1] * (1 + 1e-6))


@pytest.mark.parametrize("cfg", [2, 3])
def test_configs_2_3_tensor_core_pair_is_bitwise_repeatable(cfg):
    """The tcgen05 pass pair (fused_tc3_kernel.cuh) at the full sizes of configs 2 and 3,
    default kkt=True: three fits give bitwise the same trace (objective and KKT) and factors."""
    F, N, K, beta = {2: (1024, 8192, 32, 2.0), 3: (1025, 16384, 20, 0.0)}[cfg]
    v = (syn.config2 if cfg == 2 else syn.config3)().astype(np.float32)
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    c = bn.SolverConfig(beta=beta, rank=K, algorithm="jmm", tol=1e-300, max_outer_iters=12)
    runs = [bn.fit(v, c, init=(w0, h0), dtype="fp32") for _ in range(3)]
    assert bn.get_context(0, "fp32").pass_info()[0] == "tcgen05"
    t0 = [(r.objective, r.kkt_w, r.kkt_h) for r in runs[0].trace]
    for other in runs[1:]:
        assert [(r.objective, r.kkt_w, r.kkt_h) for r in other.trace] == t0
        assert np.array_equal(other.factors.w, runs[0].factors.w)
        assert np.array_equal(other.factors.h, runs[0].factors.h)


def _objective_fp64(v, w, h, beta, chunk=1 << 18):
    """sum d_beta(v | w h) in fp64 on the device, column chunk by column chunk."""
    dev = torch.device("cuda:0")
    W = torch.from_numpy(np.ascontiguousarray(w)).to(dev, torch.float64)
    total = 0.0
    for a in range(0, v.shape[1], chunk):
        b = min(v.shape[1], a + chunk)
        x = torch.from_numpy(np.ascontiguousarray(v[:, a:b])).to(dev).double()
        y = W @ torch.from_numpy(np.ascontiguousarray(h[:, a:b])).to(dev, torch.float64)
        d = (x.pow(beta) / (beta * (beta - 1)) + y.pow(beta) / beta
             - x * y.pow(beta - 1) / (beta - 1))
        total += float(d.sum())
    return total


def test_config4_full_size_properties():
    F, N, K, beta = 256, 4194304, 12, 1.5
    v = syn.config4(F=F, N=N, K=K, dtype=np.float32)
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    c = bn.SolverConfig(beta=beta, rank=K, algorithm="jmm", tol=1e-300, kappa=0.0,
                        max_outer_iters=10)
    r1 = bn.fit(v, c, init=(w0, h0), dtype="fp32", kkt=False)
    obj = np.array([r.objective for r in r1.trace])
    assert len(obj) == 10
    assert np.all(obj[1:] <= obj[:-1] * (1 + 1e-6))
    np.testing.assert_allclose(np.linalg.norm(r1.factors.w, axis=0), 1.0, rtol=1e-5)
    # the trace's last objective is that of the returned iterate (normalisation keeps W H)
    check = _objective_fp64(v, r1.factors.w, r1.factors.h, beta)
    assert abs(obj[-1] - check) / check <= 1e-4, (obj[-1], check)
    r2 = bn.fit(v, c, init=(w0, h0), dtype="fp32", kkt=False)
    assert [t.objective for t in r2.trace] == list(obj)
    assert np.array_equal(r1.factors.w, r2.factors.w)
    assert np.array_equal(r1.factors.h, r2.factors.h)


def _kl_sparse_fp64(indptr, idx, vals, w, h, chunk=1 << 21):
    """sum d_1(V | W H) over a CSR V in fp64: nonzeros plus the closed-form dense term."""
    dev = torch.device("cuda:0")
    W = torch.from_numpy(w).to(dev, torch.float64)
    Ht = torch.from_numpy(np.ascontiguousarray(h.T)).to(dev, torch.float64)
    rows = np.repeat(np.arange(len(indptr) - 1, dtype=np.int64), np.diff(indptr))
    total = 0.0
    for a in range(0, len(vals), chunk):
        b = min(len(vals), a + chunk)
        r = torch.from_numpy(rows[a:b]).to(dev)
        c = torch.from_numpy(idx[a:b].astype(np.int64)).to(dev)
        x = torch.from_numpy(vals[a:b]).to(dev).double()
        p = (W[r] * Ht[c]).sum(1)
        total += float((x * torch.log(x / p) - x).sum())
    return total + float(W.sum(0) @ Ht.sum(0))


def test_config5_full_size_sparse_properties():
    import scipy.sparse as sp
    indptr, idx, vals, shape = syn.config5()
    F, N = shape
    K = 64
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    c = bn.SolverConfig(beta=1.0, rank=K, algorithm="jmm", kappa=0.0, tol=1e-300,
                        max_outer_iters=8)
    r1 = bn.fit(csr, c, init=(w0, h0), dtype="fp32")
    obj = np.array([r.objective for r in r1.trace])
    assert len(obj) == 8
    assert np.all(obj[1:] <= obj[:-1] * (1 + 1e-6))
    np.testing.assert_allclose(np.linalg.norm(r1.factors.w, axis=0), 1.0, rtol=1e-5)
    check = _kl_sparse_fp64(indptr, idx, vals, r1.factors.w, r1.factors.h)
    assert abs(obj[-1] - check) / check <= 1e-4, (obj[-1], check)
    r2 = bn.fit(csr, c, init=(w0, h0), dtype="fp32")
    assert [t.objective for t in r2.trace] == list(obj)
    assert np.array_equal(r1.factors.w, r2.factors.w)
    assert np.array_equal(r1.factors.h, r2.factors.h)
