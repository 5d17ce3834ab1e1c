"""Parity sweep of the tcgen05 fused pass (fp32, schedule "auto") against the CPU oracle.

Every template instance of ``fused_pass_tc`` is exercised: the beta classes (0, 1, 2, 1.5 and the
generic rule at 0.5), kappa = 0 and kappa > 0, JMM and BMM, one CTA per block (F <= 128) and the
2-CTA row split (F > 128), ranks up to the K <= 16 limit, and column counts that are not a
multiple of the 128-column block.  The oracle runs on the same fp32-rounded V and the same init
in fp64; the gate is the north star's fp32 one: objective within 1e-4 relative over the whole
trace, and a monotone trace.
"""

import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O

pytestmark = pytest.mark.gpu

ITERS = 60
SHAPES = [(20, 130, 3), (100, 1000, 8), (200, 3000, 12), (256, 4100, 16)]
BETAS = [0.0, 0.5, 1.0, 1.5, 2.0]


def _data(F, N, K):
    v = bn.synthetic_low_rank(F, N, K, noise=0.05, seed=F + N).astype(np.float32)
    init = bn.init_factors(F, N, K, seed=K)
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
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= 1e-4, (beta, algo, kappa, float(rel.max()))
    assert np.all(got[1:] <= got[:-1] * (1 + 1e-6)), (beta, algo, kappa)
    # the returned factors are the normalised ones, like the reference
    np.testing.assert_allclose(np.linalg.norm(res.factors.w, axis=0), 1.0, rtol=1e-5)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("beta", BETAS)
def test_tc_pass_matches_oracle(shape, beta):
    F, N, K = shape
    v, init = _data(F, N, K)
    for algo in ("jmm", "bmm"):
        _check(v, init, beta, K, algo, 0.0)


@pytest.mark.parametrize("beta", [0.5, 1.5])
def test_tc_pass_with_kappa(beta):
    v, init = _data(200, 3000, 12)
    for algo in ("jmm", "bmm"):
        _check(v, init, beta, 12, algo, 1e-3)
