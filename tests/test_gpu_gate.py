"""The north-star fp32 gate on the paths the bench runs: 200 iterations against
traces written by the REFERENCE package itself (tests/golden/gen_golden_gate.py).

Gate (BASELINE.json north_star / SURVEY.md §8d): objective within 1e-4 relative at
every one of the 200 iterations, trace monotone non-increasing.  The reference ran in
fp64 on the fp32-rounded V with the same injected Uniform(0,1) init.

  cfg2, cfg3   configs 2 and 3 at their full BASELINE sizes (the SIMT pair)
  cfg4s/b/k    config-4-like shapes through the tcgen05 pass with the grid capped
               (BNMF_TC_MAX_CLUSTERS): every CTA cluster walks 32..130 column blocks, so the
               steady-state schedule of the full-size pass runs against the reference --
               the cross-block H-item interleave, the FOLD = 8 TMEM -> fp64 slab folds with
               their owner reductions, the wrap of the V stage ring, a ragged last block --
               and once more with the default grid.
"""

import os

import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from conftest import load_golden, max_rel
from paper_2106_15214_b200 import synthetic as syn

pytestmark = pytest.mark.gpu

CASES = {
    "cfg2": (lambda: syn.config2(), 32, 2.0, None),
    "cfg3": (lambda: syn.config3(), 20, 0.0, None),
    "cfg4s": (lambda: syn.config4(N=16484), 12, 1.5, 0.0),
    "cfg4b": (lambda: syn.config4(F=200, N=8292, K=16, seed=41), 16, 0.5, None),
    "cfg4k": (lambda: syn.config4(N=8292, seed=42), 12, 1.0, 0.0),
}


def _run_case(name, cap=None, expect_tc=None, v1=False):
    z = load_golden("gate.npz")
    gen, K, beta, kappa = CASES[name]
    v = gen().astype(np.float32)
    assert float(v.astype(np.float64).sum()) == float(z[f"{name}/vsum"])
    F, N = v.shape
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    old = os.environ.get("BNMF_TC_MAX_CLUSTERS")
    if cap is not None:
        os.environ["BNMF_TC_MAX_CLUSTERS"] = str(cap)
    if v1:
        os.environ["BNMF_TC_V2"] = "0"     # the first-generation kernel (A/B twin)
    try:
        for algo in ("jmm", "bmm"):
            ref = z[f"{name}_{algo}/obj"]
            assert len(ref) == 200
            cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, tol=1e-300, kappa=kappa,
                                  max_outer_iters=len(ref))
            res = bn.fit(v, cfg, init=(w0, h0), dtype="fp32", kkt=False)
            ctx = bn.get_context(0, "fp32")
            assert ctx.schedule() == "fused"
            kind, grid, cl, f0 = ctx.pass_info()
            if expect_tc is not None:
                assert (kind == "tcgen05") == expect_tc, (name, kind)
            if cap is not None:
                assert kind == "tcgen05" and grid == cl * cap, (kind, grid, cl, cap)
                nblocks = -(-N // 128)
                assert nblocks // cap >= 32       # blocks per cluster: past FOLD and the ring wrap
            got = np.array([r.objective for r in res.trace])
            assert len(got) == len(ref)
            assert max_rel(got, ref) <= 1e-4, (name, algo, cap, max_rel(got, ref))
            assert np.all(got[1:] <= got[:-1] * (1 + 1e-6)), (name, algo, cap)
            # the factors themselves: W columns unit-norm and close to the reference's
            np.testing.assert_allclose(np.linalg.norm(res.factors.w, axis=0), 1.0, rtol=1e-5)
            wref = z[f"{name}_{algo}/w"]
            err = np.linalg.norm(res.factors.w - wref) / np.linalg.norm(wref)
            assert err <= 2e-2, (name, algo, cap, err)
    finally:
        if v1:
            del os.environ["BNMF_TC_V2"]
        if cap is not None:
            if old is None:
                del os.environ["BNMF_TC_MAX_CLUSTERS"]
            else:
                os.environ["BNMF_TC_MAX_CLUSTERS"] = old


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_configs_2_3_full_size_200_iterations(name):
    _run_case(name)


@pytest.mark.parametrize("name,cap", [("cfg4s", 2), ("cfg4s", 1), ("cfg4b", 2), ("cfg4k", 1),
                                      ("cfg4s", None), ("cfg4b", None), ("cfg4k", None)])
def test_config4_steady_state_schedule_200_iterations(name, cap):
    _run_case(name, cap=cap, expect_tc=True)


@pytest.mark.parametrize("name,cap", [("cfg4s", 2), ("cfg4b", None), ("cfg4k", 1)])
def test_first_generation_kernel_200_iterations(name, cap):
    """BNMF_TC_V2=0 (fused_tc_kernel.cuh: 16 epilogue warps in lock-step, one issuing warp), the
    A/B twin of the default second-generation kernel, holds the same gate."""
    _run_case(name, cap=cap, expect_tc=True, v1=True)


@pytest.mark.parametrize("name,cap", [("cfg4s", None), ("cfg4b", None), ("cfg4k", None),
                                      ("cfg2", None), ("cfg3", None), ("cfg4s", 1), ("cfg4b", 2)])
def test_fused_kkt_residuals_match_reference(name, cap):
    """KKT residuals of the fused schedule (kkt=True, the fit() default): res_W from the W-side
    sums the pass has reduced anyway, res_H from the H-side-only KKT pass, against the
    reference's trace (diagnostics.py:46-59) over 60 iterations.  fp32 forms the gradients as
    differences of sums (den - num) -- on config 2 (an exact rank-32 V) the two sums agree to
    three digits by iteration 60 and the tensor-core pass carries them in fp32 over 1024-column
    folds -- so the tolerance is 5e-3 relative plus 1e-6 of the first residual.  With the grid
    capped every cluster walks 32+ column blocks in the KKT pass too (its H~ rows are double
    buffered in TMEM, a barrier pair per buffer)."""
    old = os.environ.get("BNMF_TC_MAX_CLUSTERS")
    if cap is not None:
        os.environ["BNMF_TC_MAX_CLUSTERS"] = str(cap)
    try:
        _kkt_case(name)
    finally:
        if cap is not None:
            if old is None:
                del os.environ["BNMF_TC_MAX_CLUSTERS"]
            else:
                os.environ["BNMF_TC_MAX_CLUSTERS"] = old


def _kkt_case(name):
    z = load_golden("gate.npz")
    gen, K, beta, kappa = CASES[name]
    v = gen().astype(np.float32)
    F, N = v.shape
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    its = 60
    for algo in ("jmm", "bmm"):
        ref = z[f"{name}_{algo}/kkt"][:its]
        ref_obj = z[f"{name}_{algo}/obj"][:its]
        cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, tol=1e-300, kappa=kappa,
                              max_outer_iters=its)
        res = bn.fit(v, cfg, init=(w0, h0), dtype="fp32")
        assert bn.get_context(0, "fp32").schedule() == "fused"
        got = np.array([[r.kkt_w, r.kkt_h] for r in res.trace])
        obj = np.array([r.objective for r in res.trace])
        assert max_rel(obj, ref_obj) <= 1e-4
        assert np.all(np.isfinite(got))
        err = np.abs(got - ref) / (np.abs(ref) + 1e-6 * np.abs(ref[0]))
        assert err.max() <= 5e-3, (name, algo, float(err.max()), np.unravel_index(err.argmax(), err.shape))
