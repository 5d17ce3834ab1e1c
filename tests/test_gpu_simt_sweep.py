"""Parity sweep of the fused passes for the shapes outside the single-read tcgen05 kernel's
limits (F > 256 or K > 16, configs 2 and 3) against the CPU oracle: the tcgen05 pass pair
(fused_tc3_kernel.cuh, K <= 32) and the register-tiled SIMT pair (fs2::hpass + fs2::wpass,
32 < K <= 64, and every shape with BNMF_TC3=0).  The sweep covers both K-tile instances (K <= 32 and 32 < K <= 64), odd and
ragged K, F with a one-row last chunk (1025 = 16 x 64 + 1), column counts that are not a
multiple of the 32-column step, every beta class (0, 1, 2 and the generic rule at 0.5 / 1.5),
kappa > 0, JMM and BMM, and a TC-eligible shape forced onto the SIMT pair.  The gate is the
north star's fp32 one: objective within 1e-4 relative over the whole trace, monotone trace.
"""

import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O

pytestmark = pytest.mark.gpu

ITERS = 40
SHAPES = [(300, 700, 20), (1025, 515, 33), (70, 203, 49), (130, 1000, 64), (257, 96, 1),
          (520, 1100, 32), (200, 900, 27), (1025, 2100, 12)]
BETAS = [0.0, 0.5, 1.0, 1.5, 2.0]


def _data(F, N, K):
    v = bn.synthetic_low_rank(F, N, K, noise=0.05, seed=F + N + K).astype(np.float32)
    init = bn.init_factors(F, N, K, seed=K + 1)
    return v, init


def _check(v, init, beta, K, algo, kappa):
    cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, tol=1e-300, kappa=kappa,
                          max_outer_iters=ITERS)
    ctx = bn.get_context(0, "fp32")
    res = bn.fit(v, cfg, init=init, dtype="fp32", kkt=False)
    assert ctx.schedule() == "fused"
    got = np.array([r.objective for r in res.trace])
    _, _, ref, _, _ = O.run(v.astype(np.float64), beta, K, algo, kappa=kappa, tol=1e-300,
                            max_outer_iters=ITERS, init=(init.w, init.h), kkt=False)
    if len(got) != len(ref):
        # at convergence either precision can see a repeated or (by rounding) non-decreasing
        # objective, which is the stop rule (solver.py:174-180); the shorter trace must end on
        # such a step, and the common prefix is compared
        short = got if len(got) < len(ref) else ref
        assert short[-1] >= short[-2] * (1 - 1e-7), (len(got), len(ref), short[-2:])
        got, ref = got[:len(short)], ref[:len(short)]
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= 1e-4, (beta, algo, kappa, float(rel.max()))
    assert np.all(got[1:] <= got[:-1] * (1 + 1e-6)), (beta, algo, kappa)
    np.testing.assert_allclose(np.linalg.norm(res.factors.w, axis=0), 1.0, rtol=1e-5)
    return res


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("beta", BETAS)
def test_simt_pass_matches_oracle(shape, beta):
    F, N, K = shape
    v, init = _data(F, N, K)
    for algo in ("jmm", "bmm"):
        _check(v, init, beta, K, algo, 0.0)


@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_simt_pass_with_kappa(beta):
    v, init = _data(300, 700, 20)
    for algo in ("jmm", "bmm"):
        _check(v, init, beta, 20, algo, 1e-3)


def test_simt_pass_forced_on_tc_shape(monkeypatch):
    """A TC-eligible shape (F <= 256, K <= 16) run on the SIMT pair; results bitwise repeatable."""
    monkeypatch.setenv("BNMF_FUSED_SIMT", "1")
    v, init = _data(45, 77, 7)
    r1 = _check(v, init, 1.5, 7, "jmm", 0.0)
    r2 = _check(v, init, 1.5, 7, "jmm", 0.0)
    assert np.array_equal(r1.factors.w, r2.factors.w)
    assert np.array_equal(r1.factors.h, r2.factors.h)


@pytest.mark.parametrize("shape", [(300, 700, 20), (257, 96, 1), (520, 1100, 32)],
                         ids=lambda s: "x".join(map(str, s)))
def test_simt_pair_on_the_tensor_core_shapes(shape):
    """BNMF_TC3=0 keeps the K <= 32 shapes on the SIMT pair (the tcgen05 pass pair is the
    default for them); both must hold the gate."""
    import os
    F, N, K = shape
    v, init = _data(F, N, K)
    os.environ["BNMF_TC3"] = "0"
    try:
        for beta in (0.0, 1.5):
            _check(v, init, beta, K, "jmm", 0.0)
            assert bn.get_context(0, "fp32").pass_info()[0] == "simt"
    finally:
        del os.environ["BNMF_TC3"]
    _check(v, init, 1.0, K, "bmm", 0.0)
    assert bn.get_context(0, "fp32").pass_info()[0] == "tcgen05"
