"""Large inputs are validated from device statistics of the upload
(bnmf_data_stats) instead of host scans; the errors and the kappa rule must be
the reference's (core.py:176-228, solver.py:205-221)."""
import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import solver

pytestmark = pytest.mark.gpu

F, N = 256, 1 << 16   # 2^24 entries: the device-checked path


def _data(seed=0):
    rng = np.random.default_rng(seed)
    return (rng.random((F, N), dtype=np.float32) + 0.5).astype(np.float32)


def test_threshold_routes_to_device():
    assert F * N >= solver._DEVICE_CHECK_MIN


@pytest.mark.parametrize("bad,exc,msg", [
    (np.nan, ValueError, "finite"),
    (np.inf, ValueError, "finite"),
    (-1.0, ValueError, "nonnegative"),
])
def test_entry_errors(bad, exc, msg):
    v = _data()
    v[17, 12345] = bad
    with pytest.raises(exc, match=msg):
        bn.fit(v, bn.SolverConfig(beta=1.5, rank=4, algorithm="jmm", max_outer_iters=1),
               dtype="fp32")


def test_zero_domain_errors():
    v = _data()
    v[3, 4] = 0.0
    with pytest.raises(bn.DivergenceDomainError):
        bn.fit(v, bn.SolverConfig(beta=0.5, rank=4, algorithm="jmm", kappa=0.0,
                                  max_outer_iters=1), dtype="fp32")
    with pytest.raises(bn.DivergenceDomainError):
        bn.fit(v, bn.SolverConfig(beta=0.0, rank=4, algorithm="jmm", kappa=0.0,
                                  max_outer_iters=1), dtype="fp32")


def test_data_stats_match_numpy():
    v = _data(1)
    ctx = solver.get_context(0, "fp32")
    with ctx.lock:
        ctx.set_dense(v, 0.0)
        mn, mx, sm, nf, cnt = ctx.data_stats()
    assert mn == float(v.min()) and mx == float(v.max())
    assert nf == 0 and cnt == v.size
    assert sm == pytest.approx(float(v.sum(dtype=np.float64)), rel=1e-12)


def test_auto_kappa_matches_host_rule():
    # beta = 0 and zeros in the data: kappa = 1e-9 * mean (default_kappa)
    v = _data(2)
    v[::7, ::5] = 0.0
    init = bn.init_factors(F, N, 4, seed=3)
    cfg = bn.SolverConfig(beta=0.0, rank=4, algorithm="jmm", max_outer_iters=3, tol=1e-300)
    dev = bn.fit(v, cfg, init=init, dtype="fp32", kkt=False)                 # device checks
    host = bn.fit(bn.DataMatrix(v, bn.default_kappa(v, 0.0)), cfg, init=init, dtype="fp32",
                  kkt=False)                                                 # host checks
    a = np.array([t.objective for t in dev.trace])
    b = np.array([t.objective for t in host.trace])
    assert np.allclose(a, b, rtol=1e-6)


@pytest.mark.parametrize("where,bad,msg", [
    ("h", np.nan, "factor entries must be finite"),
    ("w", np.inf, "factor entries must be finite"),
    ("h", 0.0, "factor entries must be strictly positive"),
    ("w", -2.0, "factor entries must be strictly positive"),
])
def test_large_init_checked_on_device(where, bad, msg):
    """An injected init of >= 2^24 entries is validated on its device copy
    (Context.set_factors), with the reference FactorPair's messages."""
    Fi, Ni, K = 64, 1 << 18, 64
    assert K * Ni >= solver._DEVICE_CHECK_MIN
    rng = np.random.default_rng(2)
    v = (rng.random((Fi, Ni), dtype=np.float32) + 0.5).astype(np.float32)
    w0 = rng.random((Fi, K)) + 0.1
    h0 = rng.random((K, Ni)) + 0.1
    cfg = bn.SolverConfig(beta=1.0, rank=K, algorithm="jmm", max_outer_iters=2, tol=1e-300)
    res = bn.fit(v, cfg, init=(w0, h0), dtype="fp32", kkt=False)
    assert res.iterations == 2
    (w0 if where == "w" else h0)[5, 7] = bad
    with pytest.raises(ValueError, match=msg):
        bn.fit(v, cfg, init=(w0, h0), dtype="fp32", kkt=False)
    # the host path (small data) raises the same message
    with pytest.raises(ValueError, match=msg):
        bn.fit(v[:, :64], cfg, init=(w0, h0[:, :64]), dtype="fp32", kkt=False)
