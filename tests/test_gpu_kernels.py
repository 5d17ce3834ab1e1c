"""The reference's lower-level public kernels, device-backed (paper_2106_15214_b200/kernels.py ->
include/bnmf.h: bnmf_kernel), against the outputs the reference produced for the same inputs
(tests/golden/kernels.npz, written by gen_golden.py from updates.py:157-235, core.py:275-306,
diagnostics.py:62-90): fp64, 1e-10 relative."""

import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from conftest import load_golden, max_rel

pytestmark = pytest.mark.gpu


def _cases():
    z = load_golden("kernels.npz")
    return list(range(int(z["count"])))


@pytest.mark.parametrize("i", _cases())
def test_update_kernels_match_reference(i):
    z = load_golden("kernels.npz")
    key = f"k{i}"
    beta, kappa = float(z[f"{key}/beta"]), float(z[f"{key}/kappa"])
    v, wt, ht, hc, wc = (z[f"{key}/{n}"] for n in ("v", "wt", "ht", "hc", "wc"))
    vs = v + kappa
    anchor = bn.MajorizerAnchor.from_factors(wt, ht, kappa=kappa)
    counter = bn.OpCounter()
    assert max_rel(bn.jmm_update_w(vs, anchor, hc, beta, counter=counter), z[f"{key}/jmm_w"]) <= 1e-10
    assert max_rel(bn.jmm_update_h(vs, anchor, wc, beta, counter=counter), z[f"{key}/jmm_h"]) <= 1e-10
    assert max_rel(bn.bmm_update_w(vs, wc, hc, beta, kappa=kappa, counter=counter),
                   z[f"{key}/bmm_w"]) <= 1e-10
    assert max_rel(bn.bmm_update_h(vs, wc, hc, beta, kappa=kappa, counter=counter),
                   z[f"{key}/bmm_h"]) <= 1e-10
    assert (counter.w_updates, counter.h_updates, counter.kernel_products) == (2, 2, 2)
    data, pair = bn.DataMatrix(v, kappa), bn.FactorPair(wc, hc)
    assert abs(bn.objective(data, pair, beta) - float(z[f"{key}/obj"])) <= 1e-10 * abs(float(z[f"{key}/obj"]))
    kr = bn.kkt_residuals(data, pair, beta)
    assert isinstance(kr, bn.KktResiduals)
    np.testing.assert_allclose([kr.res_w, kr.res_h], z[f"{key}/kkt"], rtol=1e-9)


def test_kernel_argument_checks():
    v = bn.synthetic_low_rank(6, 5, 2, noise=0.1, seed=1)
    pair = bn.init_factors(6, 5, 2, seed=2)
    with pytest.raises(ValueError, match="dimension mismatch"):
        bn.objective(v[:, :4], pair, 1.0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        bn.kkt_residuals(v[:5], pair, 1.0)
    with pytest.raises(ValueError, match="strictly positive"):
        bn.MajorizerAnchor.from_factors(pair.w * 0.0, pair.h)
    with pytest.raises(bn.DivergenceDomainError):
        z = v.copy()
        z[0, 0] = 0.0
        bn.objective(z, pair, 0.0)
    # the fitted iterate's objective is the last trace row's
    res = bn.fit(v, bn.SolverConfig(beta=1.5, rank=2, algorithm="jmm", max_outer_iters=7, tol=1e-300))
    assert abs(bn.objective(v, res.factors, 1.5) - res.trace[-1].objective) <= 1e-10 * res.trace[-1].objective
    kr = bn.kkt_residuals(v, res.factors, 1.5)
    np.testing.assert_allclose([kr.res_w, kr.res_h], [res.trace[-1].kkt_w, res.trace[-1].kkt_h], rtol=1e-8)
