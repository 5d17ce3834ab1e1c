"""Pin the CPU oracle (oracle/betanmf_oracle.py) against the reference itself.

The fixtures under tests/golden/ were produced by tests/golden/gen_golden.py,
which imports the unmodified reference package.  If the restatement drifts
from the reference, these tests fail before any GPU parity claim is made.
"""

import numpy as np
import pytest

from conftest import golden_fit_cases, load_golden, max_rel, parse_cfg
from oracle import betanmf_oracle as O


@pytest.mark.parametrize("name", golden_fit_cases())
def test_oracle_matches_reference_fit(name):
    z = load_golden("fits.npz")
    cfg = parse_cfg(str(z[f"{name}/cfg"]))
    algo = str(cfg.pop("algorithm"))
    beta = cfg.pop("beta")
    rank = cfg.pop("rank")
    w, h, obj, kkt, term = O.run(z[f"{name}/v"], beta, rank, algo, **cfg)
    assert term == str(z[f"{name}/term"])
    assert obj.shape == z[f"{name}/obj"].shape
    assert max_rel(obj, z[f"{name}/obj"]) <= 1e-12
    assert max_rel(w, z[f"{name}/w"]) <= 1e-10
    assert max_rel(h, z[f"{name}/h"]) <= 1e-10
    np.testing.assert_allclose(kkt, z[f"{name}/kkt"], rtol=1e-8, atol=1e-300)


def test_oracle_update_kernels_match_reference():
    z = load_golden("kernels.npz")
    for i in range(int(z["count"])):
        k = f"k{i}"
        beta = float(z[f"{k}/beta"])
        kappa = float(z[f"{k}/kappa"])
        v, wt, ht, hc, wc = (z[f"{k}/{n}"] for n in ("v", "wt", "ht", "hc", "wc"))
        vs = v + kappa
        g = O.gamma_exponent(beta)
        prod = wt @ ht + kappa
        bases = O.joint_bases(vs, prod, beta)
        assert max_rel(O.jmm_update_w(bases, wt, ht, hc, beta, g, O.DEFAULT_FLOOR),
                       z[f"{k}/jmm_w"]) <= 1e-14
        assert max_rel(O.jmm_update_h(bases, wt, ht, wc, beta, g, O.DEFAULT_FLOOR),
                       z[f"{k}/jmm_h"]) <= 1e-14
        assert max_rel(O.bmm_update_w(vs, wc, hc, beta, kappa, g, O.DEFAULT_FLOOR),
                       z[f"{k}/bmm_w"]) <= 1e-14
        assert max_rel(O.bmm_update_h(vs, wc, hc, beta, kappa, g, O.DEFAULT_FLOOR),
                       z[f"{k}/bmm_h"]) <= 1e-14
        p = wc @ hc + kappa
        assert abs(O.divergence_total(vs, p, beta) - float(z[f"{k}/obj"])) <= \
            1e-12 * abs(float(z[f"{k}/obj"]))
        np.testing.assert_allclose(O.kkt_residuals_arrays(vs, wc, hc, beta, kappa),
                                   z[f"{k}/kkt"], rtol=1e-12)


def test_oracle_hand_examples():
    # test_updates.py:124-147 of the reference: JMM hand examples
    v = np.array([[2.0, 4.0], [6.0, 8.0]])
    wt, ht = np.array([[1.0], [1.0]]), np.array([[1.0, 1.0]])
    bases = O.joint_bases(v, wt @ ht, 2.0)
    w = O.jmm_update_w(bases, wt, ht, np.array([[2.0, 2.0]]), 2.0, 1.0, O.DEFAULT_FLOOR)
    np.testing.assert_allclose(w, [[1.5], [3.5]], rtol=1e-14)
    h = O.jmm_update_h(bases, wt, ht, np.array([[2.0], [2.0]]), 2.0, 1.0, O.DEFAULT_FLOOR)
    np.testing.assert_allclose(h, [[2.0, 3.0]], rtol=1e-14)
    v = np.array([[1.0, 2.0], [3.0, 4.0]])
    bases = O.joint_bases(v, wt @ ht, 1.0)
    h = O.jmm_update_h(bases, wt, ht, wt, 1.0, 1.0, O.DEFAULT_FLOOR)
    np.testing.assert_allclose(h, [[2.0, 3.0]], rtol=1e-14)
    # core.py scalar examples (test_core.py:22-42)
    assert abs(float(O.beta_divergence_elements(1.0, 2.0, 1.0)) - (1 - np.log(2))) < 1e-14
    assert abs(float(O.beta_divergence_elements(2.0, 1.0, 0.0)) - (1 - np.log(2))) < 1e-14
    assert O.gamma_exponent(0.0) == 0.5 and O.gamma_exponent(3.0) == 0.5
    assert O.should_stop(1.0, 1.0, 1e-5) is True


@pytest.mark.parametrize("name", ["cfg2p", "cfg3p", "cfg4p"])
def test_oracle_matches_reference_configs(name):
    """BASELINE config prefixes (fp32-rounded V), injected U(0,1) init."""
    from paper_2106_15214_b200 import synthetic
    z = load_golden("configs.npz")
    gen = {"cfg2p": lambda: synthetic.config2(F=1024, N=1024, K=32),
           "cfg3p": lambda: synthetic.config3(F=1025, N=1024, K=20),
           "cfg4p": lambda: synthetic.config4(N=4096)}[name]
    K, beta, kappa = {"cfg2p": (32, 2.0, None), "cfg3p": (20, 0.0, None),
                      "cfg4p": (12, 1.5, 0.0)}[name]
    v = gen().astype(np.float32).astype(np.float64)
    assert float(v.sum()) == float(z[f"{name}/vsum"])
    w0, h0 = synthetic.uniform_init(v.shape[0], v.shape[1], K, seed=100 + K)
    for algo in ("jmm", "bmm"):
        ref_obj = z[f"{name}_{algo}/obj"]
        w, h, obj, _, _ = O.run(v, beta, K, algo, kappa=kappa, tol=1e-300,
                                max_outer_iters=len(ref_obj), init=(w0, h0), kkt=False)
        assert max_rel(obj, ref_obj) <= 1e-11
        assert max_rel(w, z[f"{name}_{algo}/w"]) <= 1e-8


def test_oracle_sparse_restatement_matches_dense_reference():
    import scipy.sparse as sp
    from paper_2106_15214_b200 import synthetic
    z = load_golden("configs.npz")
    indptr, idx, vals, shape = synthetic.config5(F=2000, N=400, density=0.1, seed=55)
    assert idx.size == int(z["cfg5p/nnz"])
    csr = sp.csr_matrix((vals.astype(np.float64), idx, indptr), shape=shape)
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 16, seed=116)
    for algo in ("jmm", "bmm"):
        ref = z[f"cfg5p_{algo}/obj"]
        w, h, obj, _ = O.run_sparse_kl(csr, 16, algo, max_outer_iters=len(ref),
                                       init=(w0, h0))
        assert max_rel(obj, ref) <= 1e-11
        assert max_rel(w, z[f"cfg5p_{algo}/w"]) <= 1e-8
