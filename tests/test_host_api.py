"""Host-side semantics of the drop-in API that run before any device work
(solver.py:62-114 validation, solver.py:205-221 domain checks,
solver.py:137-153 init, solver.py:174-180 stop rule)."""

import numpy as np
import pytest

import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O


def test_config_validation():
    with pytest.raises(ValueError):
        bn.SolverConfig(beta=1.0, rank=0, algorithm="bmm")
    with pytest.raises(ValueError):
        bn.SolverConfig(beta=1.0, rank=2, algorithm="bmm", tol=0.0)
    with pytest.raises(ValueError):
        bn.SolverConfig(beta=1.0, rank=2, algorithm="bmm", sub_iters=0)
    with pytest.raises(ValueError):
        bn.SolverConfig(beta=1.0, rank=2, algorithm="bmm", denominator_floor=0.0)
    with pytest.raises(ValueError):
        bn.run_jmm(np.ones((2, 2)), bn.SolverConfig(beta=1.0, rank=1, algorithm="bmm"))


def test_domain_errors_raised_before_device_work():
    v = np.array([[0.0, 1.0], [2.0, 3.0]])
    with pytest.raises(bn.DivergenceDomainError):
        bn.run_bmm(v, bn.SolverConfig(beta=0.0, rank=1, algorithm="bmm", kappa=0.0))
    with pytest.raises(ValueError):
        bn.fit(np.array([[-1.0, 1.0]]), bn.SolverConfig(beta=1.0, rank=1, algorithm="jmm"))
    with pytest.raises(ValueError):
        bn.fit(np.array([[np.nan, 1.0]]), bn.SolverConfig(beta=1.0, rank=1, algorithm="jmm"))


def test_init_factors_matches_reference_rule():
    a = bn.init_factors(7, 5, 3, seed=11)
    w, h = O.init_factors(7, 5, 3, 11)
    assert np.array_equal(a.w, w) and np.array_equal(a.h, h)


def test_gamma_and_kappa_rules():
    for b in (-0.5, 0.0, 0.5, 1.0, 1.5, 2.0, 3.0):
        assert bn.gamma_exponent(b) == O.gamma_exponent(b)
    v = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert bn.default_kappa(v, 1.5) == 0.0
    assert bn.default_kappa(v, 0.0) == pytest.approx(1e-9 * 2.5)


def test_should_stop_examples():
    assert bn.should_stop(1.0, 0.999999, 1e-5) is True
    assert bn.should_stop(1.0, 0.9, 1e-5) is False
    assert bn.should_stop(1.0, 1.0, 1e-5) is True
    assert bn.should_stop(0.0, 0.0, 1e-5) is True


def test_normalize_hand_example():
    out = bn.normalize(bn.FactorPair(np.array([[3.0], [4.0]]), np.array([[1.0, 1.0]])))
    assert np.allclose(out.w, [[0.6], [0.8]], rtol=1e-15)
    assert np.allclose(out.h, [[5.0, 5.0]], rtol=1e-15)


def test_scalar_divergence_examples():
    assert abs(bn.beta_divergence(1.0, 2.0, 1.0) - (1 - np.log(2))) < 1e-14
    assert abs(bn.beta_divergence(2.0, 1.0, 0.0) - (1 - np.log(2))) < 1e-14
    assert bn.beta_divergence(3.0, 1.0, 2.0) == 2.0
    with pytest.raises(bn.DivergenceDomainError):
        bn.beta_divergence(0.0, 1.0, 0.0)


def test_sparse_layout_does_not_mutate_the_callers_matrix():
    """csr_with_csc_view sorts indices on a copy (the reference never mutates
    its inputs)."""
    import scipy.sparse as sp
    from paper_2106_15214_b200.solver import csr_with_csc_view
    indptr = np.array([0, 3, 5])
    idx = np.array([2, 0, 1, 1, 0], dtype=np.int32)
    data = np.array([1., 2., 3., 4., 5.], dtype=np.float32)
    m = sp.csr_matrix((data, idx, indptr), shape=(2, 3))
    before = (m.indices.copy(), m.data.copy())
    (ip, ix, v, cp, ri, pm), shape = csr_with_csc_view(m)
    assert np.array_equal(m.indices, before[0]) and np.array_equal(m.data, before[1])
    assert shape == (2, 3) and list(ix) == [0, 1, 2, 0, 1] and list(v) == [2, 3, 1, 5, 4]
    assert list(cp) == [0, 2, 4, 5] and list(v[pm]) == [2, 5, 3, 4, 1]


def test_reference_public_names_are_exported():
    """The solver-path names of the reference's __init__.py (betanmf/__init__.py:38-114)
    resolve against the drop-in; the CPU-only audits of the bound (verify suites, aux_value,
    finite-difference gradients, operation-count model) are out of scope."""
    import paper_2106_15214_b200 as bn
    names = ["Algorithm", "BenchReport", "BetaParam", "DataMatrix", "DivergenceDomainError",
             "FactorPair", "FitResult", "KktResiduals", "MajorizerAnchor", "OpCounter",
             "SolverConfig", "Termination", "UpdateKind", "beta_divergence", "bmm_update_h",
             "bmm_update_w", "default_kappa", "fit", "format_report", "gamma_exponent",
             "init_factors", "jmm_update_h", "jmm_update_w", "kkt_residuals", "load_matrix",
             "match_columns", "normalize", "objective", "run_bench", "run_bmm", "run_jmm",
             "save_factors", "save_trace", "should_stop", "summarize", "synthetic_low_rank"]
    missing = [n for n in names if not hasattr(bn, n) or n not in bn.__all__]
    assert not missing, missing
    # the kernels are device-backed: without a device they raise, they never fall back
    from paper_2106_15214_b200 import _native
    if _native.device_count() == 0:
        import numpy as np
        import pytest
        v = bn.synthetic_low_rank(6, 5, 2, noise=0.1, seed=1)
        with pytest.raises(_native.NativeUnavailable):
            bn.objective(v, bn.init_factors(6, 5, 2, seed=2), 1.0)
