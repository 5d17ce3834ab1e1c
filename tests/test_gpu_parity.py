"""Parity of the CUDA path (through the drop-in API and the C ABI) against the
reference, via the golden fixtures it produced (tests/golden/gen_golden.py)
and the pinned CPU oracle.

Tolerances (BASELINE.json north_star):
  fp64: W, H and every objective <= 1e-10 relative; KKT <= 1e-6 relative
  fp32: objective <= 1e-4 relative over the whole trace; trace monotone.
"""

import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from conftest import golden_fit_cases, load_golden, max_rel, parse_cfg

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-10


def _fit_case(name, **opts):
    z = load_golden("fits.npz")
    cfg = parse_cfg(str(z[f"{name}/cfg"]))
    config = bn.SolverConfig(**cfg)
    return z, bn.fit(z[f"{name}/v"], config, **opts)


@pytest.mark.parametrize("name", golden_fit_cases())
def test_fp64_fit_matches_reference(name):
    z, res = _fit_case(name, schedule="reference")
    ref_obj = z[f"{name}/obj"]
    assert res.termination.value == str(z[f"{name}/term"])
    assert res.iterations == len(ref_obj)
    obj = np.array([r.objective for r in res.trace])
    # objectives at round-off level (exact fits) are compared absolutely
    atol = 1e-14 * float(np.abs(z[f"{name}/v"]).sum())
    assert np.all(np.abs(obj - ref_obj) <= FP64_TOL * np.abs(ref_obj) + atol)
    assert max_rel(res.factors.w, z[f"{name}/w"]) <= FP64_TOL
    assert max_rel(res.factors.h, z[f"{name}/h"]) <= FP64_TOL
    kkt = np.array([[r.kkt_w, r.kkt_h] for r in res.trace])
    np.testing.assert_allclose(kkt, z[f"{name}/kkt"], rtol=1e-6, atol=1e-12)
    assert [r.iteration for r in res.trace] == list(range(1, res.iterations + 1))
    sec = [r.seconds for r in res.trace]
    assert all(b >= a for a, b in zip(sec, sec[1:]))


def test_config1_full_fp64_jmm_200_iterations():
    """PR1 gate: config 1 at full size, injected U(0,1) init."""
    from paper_2106_15214_b200 import synthetic
    z = load_golden("configs.npz")
    v = synthetic.config1()
    assert float(v.sum()) == float(z["cfg1/vsum"])
    w0, h0 = synthetic.uniform_init(361, 2429, 49, seed=149)
    for algo in ("jmm", "bmm"):
        ref_obj = z[f"cfg1_{algo}/obj"]
        cfg = bn.SolverConfig(beta=1.0, rank=49, algorithm=algo, tol=1e-300,
                              max_outer_iters=len(ref_obj))
        res = bn.fit(v, cfg, init=(w0, h0))
        obj = np.array([r.objective for r in res.trace])
        assert max_rel(obj, ref_obj) <= FP64_TOL
        assert max_rel(res.factors.w, z[f"cfg1_{algo}/w"]) <= FP64_TOL
        assert max_rel(res.factors.h, z[f"cfg1_{algo}/h"]) <= FP64_TOL
        assert all(b <= a * (1 + 1e-10) for a, b in zip(obj, obj[1:]))


@pytest.mark.parametrize("beta,algo", [(1.0, "jmm"), (0.5, "jmm"), (2.0, "bmm")])
def test_fp64_hside_cluster_row_split_matches_unsplit(monkeypatch, beta, algo):
    """The fp64 H-side pass splits the rows of a column block over a thread-block cluster when
    there are fewer column blocks than SMs (partials over DSMEM, rank 0 updates).  Every cluster
    size must reproduce the unsplit pass (same sums, added per row range), KKT pass included."""
    rng = np.random.default_rng(7)
    f, n, k = 300, 450, 21        # 15 column blocks, 10 row tiles (the last one ragged)
    v = rng.gamma(1.0, 1.0, (f, k)) @ rng.gamma(1.0, 1.0, (k, n)) + 1e-3
    w0 = rng.uniform(0.1, 1.0, (f, k))
    h0 = rng.uniform(0.1, 1.0, (k, n))
    cfg = bn.SolverConfig(beta=beta, rank=k, algorithm=algo, tol=1e-300, max_outer_iters=12)
    out = {}
    for cs in (1, 2, 3, 4):
        monkeypatch.setenv("BNMF_HSIDE_CLUSTER", str(cs))
        res = bn.fit(v, cfg, init=(w0, h0))
        out[cs] = (np.array([r.objective for r in res.trace]), res.factors.w, res.factors.h,
                   np.array([[r.kkt_w, r.kkt_h] for r in res.trace]))
    for cs in (2, 3, 4):
        assert max_rel(out[cs][0], out[1][0]) <= 1e-12
        assert max_rel(out[cs][1], out[1][1]) <= 1e-11
        assert max_rel(out[cs][2], out[1][2]) <= 1e-11
        np.testing.assert_allclose(out[cs][3], out[1][3], rtol=1e-9, atol=1e-15)


CFG = {
    "cfg2p": (lambda s: s.config2(F=1024, N=1024, K=32), 32, 2.0, None),
    "cfg3p": (lambda s: s.config3(F=1025, N=1024, K=20), 20, 0.0, None),
    "cfg4p": (lambda s: s.config4(N=4096), 12, 1.5, 0.0),
}


@pytest.mark.parametrize("schedule", ["reference", "auto"])
@pytest.mark.parametrize("name", sorted(CFG))
def test_fp32_configs_objective_within_1e4(name, schedule):
    from paper_2106_15214_b200 import synthetic
    z = load_golden("configs.npz")
    gen, K, beta, kappa = CFG[name]
    v = gen(synthetic).astype(np.float32)
    w0, h0 = synthetic.uniform_init(v.shape[0], v.shape[1], K, seed=100 + K)
    for algo in ("jmm", "bmm"):
        ref_obj = z[f"{name}_{algo}/obj"]
        cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, tol=1e-300, kappa=kappa,
                              max_outer_iters=len(ref_obj))
        res = bn.fit(v, cfg, init=(w0, h0), dtype="fp32", kkt=False, schedule=schedule)
        obj = np.array([r.objective for r in res.trace])
        assert max_rel(obj, ref_obj) <= 1e-4, (algo, max_rel(obj, ref_obj))
        assert all(b <= a * (1 + 1e-6) for a, b in zip(obj, obj[1:]))


def test_bitwise_reproducible():
    v = bn.synthetic_low_rank(150, 120, 3, noise=0.1, seed=4)
    for dtype in ("fp64", "fp32"):
        cfg = bn.SolverConfig(beta=0.0, rank=3, algorithm="jmm", seed=9,
                              max_outer_iters=30, tol=1e-300)
        r1 = bn.run_jmm(v, cfg, dtype=dtype)
        r2 = bn.run_jmm(v, cfg, dtype=dtype)
        assert np.array_equal(r1.factors.w, r2.factors.w)
        assert np.array_equal(r1.factors.h, r2.factors.h)
        assert [t.objective for t in r1.trace] == [t.objective for t in r2.trace]


def test_op_counter_semantics():
    v = bn.synthetic_low_rank(10, 8, 3, noise=0.1, seed=1)
    counter = bn.OpCounter()
    cfg = bn.SolverConfig(beta=1.5, rank=3, algorithm="jmm", seed=2, sub_iters=4,
                          max_outer_iters=5, tol=1e-300)
    bn.run_jmm(v, cfg, counter=counter)
    assert counter.anchor_products == 5 and counter.objective_products == 5
    assert counter.w_updates == 20 and counter.h_updates == 20
    counter = bn.OpCounter()
    cfg = bn.SolverConfig(beta=1.5, rank=3, algorithm="bmm", seed=2, sub_iters_w=2,
                          sub_iters_h=3, max_outer_iters=5, tol=1e-300)
    bn.run_bmm(v, cfg, counter=counter)
    assert counter.kernel_products == 25


def test_exact_fit_converges_at_second_iteration():
    init = bn.init_factors(5, 4, 2, seed=3)
    v = init.w @ init.h
    for algo in ("bmm", "jmm"):
        res = bn.fit(v, bn.SolverConfig(beta=2.0, rank=2, algorithm=algo, seed=3))
        assert res.termination == bn.Termination.CONVERGED
        assert res.iterations == 2


def test_native_library_is_what_ran():
    """The fit must have gone through libbnmf (no silent fallback)."""
    ctx = bn.get_context(0, "fp64")
    v = bn.synthetic_low_rank(20, 16, 2, noise=0.1, seed=5)
    bn.fit(v, bn.SolverConfig(beta=1.0, rank=2, algorithm="jmm", max_outer_iters=3))
    assert ctx.launches_per_iter() > 0
    assert ctx.schedule() in ("reference", "fused")


def test_sparse_kl_matches_dense_reference():
    """Config-5-like sparse KL (CSR) against the reference run on the
    densified matrix (golden cfg5p), fp32 objective <= 1e-4."""
    import scipy.sparse as sp
    from paper_2106_15214_b200 import synthetic
    z = load_golden("configs.npz")
    indptr, idx, vals, shape = synthetic.config5(F=2000, N=400, density=0.1, seed=55)
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 16, seed=116)
    for algo in ("jmm", "bmm"):
        ref = z[f"cfg5p_{algo}/obj"]
        cfg = bn.SolverConfig(beta=1.0, rank=16, algorithm=algo, kappa=0.0, tol=1e-300,
                              max_outer_iters=len(ref))
        res = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
        obj = np.array([r.objective for r in res.trace])
        assert max_rel(obj, ref) <= 1e-4, (algo, max_rel(obj, ref))
        assert res.factors.w.shape == (2000, 16) and res.factors.h.shape == (16, 400)
        # the trace carries the KKT residuals of every iterate like the reference's
        # (diagnostics.py:46-59); fp32 gradients are differences of sums
        kkt = np.array([[r.kkt_w, r.kkt_h] for r in res.trace])
        np.testing.assert_allclose(kkt, z[f"cfg5p_{algo}/kkt"], rtol=2e-3)
        # and they are outside the loop timer: kkt=False gives the same iterates
        res2 = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32", kkt=False)
        assert [r.objective for r in res2.trace] == [r.objective for r in res.trace]
        assert np.isnan(res2.trace[-1].kkt_w)


def test_sparse_matches_oracle_restatement_and_is_deterministic():
    import scipy.sparse as sp
    from oracle import betanmf_oracle as O
    from paper_2106_15214_b200 import synthetic
    indptr, idx, vals, shape = synthetic.config5(F=5000, N=3000, density=0.01, seed=7)
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 64, seed=164)
    cfg = bn.SolverConfig(beta=1.0, rank=64, algorithm="jmm", kappa=0.0, tol=1e-300,
                          max_outer_iters=10)
    r1 = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
    r2 = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
    assert np.array_equal(r1.factors.w, r2.factors.w)
    assert [t.objective for t in r1.trace] == [t.objective for t in r2.trace]
    _, _, obj, _ = O.run_sparse_kl(csr.astype(np.float64), 64, "jmm", max_outer_iters=10,
                                   init=(w0, h0))
    got = np.array([t.objective for t in r1.trace])
    assert max_rel(got, obj) <= 1e-4


def test_sparse_heavy_columns_and_row_tiles_match_oracle():
    """The sparse code paths that only exist at scale, against the oracle restatement: 300 000
    rows span three SP_TILE = 131072 row tiles, and under Zipf(1.1) over 1500 columns the
    heaviest columns hold > 100 000 nonzeros each -- far above SP_HEAVY = 2048 (row-tiled
    512-nonzero segments) and above SP_B2_HEAVY = 64 segments (pass B2h, one block per
    column).  25 iterations, JMM and BMM, north-star fp32 gate."""
    import scipy.sparse as sp
    from oracle import betanmf_oracle as O
    from paper_2106_15214_b200 import synthetic
    indptr, idx, vals, shape = synthetic.config5(F=300000, N=1500, density=0.004, seed=77)
    counts = np.bincount(idx, minlength=shape[1])
    assert counts.max() > 64 * 512 and (counts > 2048).sum() >= 20
    assert shape[0] > 2 * 131072
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 16, seed=116)
    for algo in ("jmm", "bmm"):
        cfg = bn.SolverConfig(beta=1.0, rank=16, algorithm=algo, kappa=0.0, tol=1e-300,
                              max_outer_iters=25)
        res = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
        wr, hr, obj, _ = O.run_sparse_kl(csr.astype(np.float64), 16, algo, max_outer_iters=25,
                                         init=(w0, h0))
        got = np.array([t.objective for t in res.trace])
        assert max_rel(got, obj) <= 1e-4, (algo, max_rel(got, obj))
        assert np.all(got[1:] <= got[:-1] * (1 + 1e-6))
        assert np.linalg.norm(res.factors.w - wr) / np.linalg.norm(wr) <= 1e-3
        assert np.linalg.norm(res.factors.h - hr) / np.linalg.norm(hr) <= 1e-3


def test_sparse_sharded_entry_with_one_rank_matches_unsharded():
    """The row-sharded sparse entry (sharded=True: global init sliced by row
    offsets, NCCL communicator attached) on a 1-rank process group gives the
    single-GPU result bitwise; the N > 1 decomposition is covered on CPU by
    tests/test_parallel_gloo.py."""
    import os
    import socket

    import scipy.sparse as sp
    import torch.distributed as dist
    from paper_2106_15214_b200 import synthetic
    indptr, idx, vals, shape = synthetic.config5(F=3000, N=500, density=0.02, seed=21)
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 32, seed=132)
    cfg = bn.SolverConfig(beta=1.0, rank=32, algorithm="jmm", kappa=0.0, tol=1e-300,
                          max_outer_iters=12)
    ref = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        got = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32", sharded=True)
    finally:
        dist.destroy_process_group()
    assert [t.objective for t in got.trace] == [t.objective for t in ref.trace]
    assert np.array_equal(got.factors.w, ref.factors.w)
    assert np.array_equal(got.factors.h, ref.factors.h)


@pytest.mark.parametrize("dtype,shape", [("fp32", (256, 4100, 12, 1.5)), ("fp32", (300, 2000, 20, 0.0)),
                                         ("fp64", (64, 500, 5, 1.0))])
def test_dense_sharded_entry_with_one_rank_matches_unsharded(dtype, shape):
    """Dense fit(..., sharded=True) (N-column shard) on a 1-rank process group:
    the communicator is attached (ncclCommInitRank with nranks = 1), the global checks run on
    allreduced device statistics, the init is sliced by column offsets -- and the result is
    bitwise the unsharded one (tcgen05 pass, SIMT pair and the fp64 reference schedule)."""
    import os
    import socket

    import torch.distributed as dist
    F, N, K, beta = shape
    v = bn.synthetic_low_rank(F, N, K, noise=0.05, seed=F + N)
    if dtype == "fp32":
        v = v.astype(np.float32)
    init = bn.init_factors(F, N, K, seed=K)
    cfg = bn.SolverConfig(beta=beta, rank=K, algorithm="jmm", tol=1e-300, max_outer_iters=15)
    ref = bn.fit(v, cfg, init=init, dtype=dtype, kkt=False)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        got = bn.fit(v, cfg, init=(init.w, init.h), dtype=dtype, kkt=False, sharded=True)
    finally:
        dist.destroy_process_group()
    assert [t.objective for t in got.trace] == [t.objective for t in ref.trace]
    assert np.array_equal(got.factors.w, ref.factors.w)
    assert np.array_equal(got.factors.h, ref.factors.h)
