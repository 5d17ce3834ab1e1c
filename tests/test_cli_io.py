"""Matrix IO, the multi-seed harness and the CLI.

CPU tests cover parsing, error messages, round trips, statistics and argument handling, following
the reference's own IO / CLI tests (``pkg/tests/test_matrixio.py``, ``test_cli.py``); the GPU
tests run ``fit`` and ``bench`` end to end on the device.
"""

import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.io import mmwrite

from paper_2106_15214_b200 import cli, harness, matrixio


def _write(path, text):
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)
    return str(path)


def test_csv_header_and_values(tmp_path):
    p = _write(tmp_path / "a.csv", "c1,c2,c3\n1,2,3\n\n4,5.5,6e-3\n")
    dm = matrixio.load_matrix(p)
    np.testing.assert_array_equal(dm.values, [[1, 2, 3], [4, 5.5, 6e-3]])


@pytest.mark.parametrize("text,msg", [
    ("1,2\n3,x\n", "cannot parse 'x' at line 2, column 2"),
    ("1,2\n3\n", "line 2 has 1 values, expected 2"),
    ("1,2\n3,-4\n", "negative value -4.0 at row 2, column 2"),
    ("1,nan\n", "non-finite value nan at row 1, column 2"),
    ("hdr\n", "no data rows found"),
])
def test_csv_errors(tmp_path, text, msg):
    p = _write(tmp_path / "b.csv", text)
    with pytest.raises(matrixio.MatrixParseError, match=msg):
        matrixio.load_matrix(p)


def test_mtx_dense_and_densify_guard(tmp_path):
    m = sp.random(30, 20, density=0.2, random_state=1, format="coo") * 5
    p = str(tmp_path / "m.mtx")
    mmwrite(p, m)
    dm = matrixio.load_matrix(p, "mtx")
    np.testing.assert_allclose(dm.values, m.toarray(), rtol=1e-15)
    with pytest.raises(matrixio.MatrixParseError, match="above the limit of 100"):
        matrixio.load_matrix(p, "mtx", densify_limit=100)


def test_mtx_sparse_is_never_densified(tmp_path):
    # 10^6 x 10^6 would be 10^12 dense entries: only the sparse reader can take it
    p = _write(tmp_path / "big.mtx",
               "%%MatrixMarket matrix coordinate real general\n"
               "1000000 1000000 3\n1 1 2.0\n1000000 999999 1.5\n1 1 0.5\n")
    with pytest.raises(matrixio.MatrixParseError, match="above the limit"):
        matrixio.load_matrix(p, "mtx")
    csr = matrixio.load_matrix(p, "mtx", sparse=True)
    assert sp.isspmatrix_csr(csr) and csr.shape == (10**6, 10**6)
    assert csr.nnz == 2 and csr[0, 0] == 2.5 and csr[999999, 999998] == 1.5   # duplicates summed


def test_mtx_sparse_rejects_negative(tmp_path):
    p = _write(tmp_path / "neg.mtx",
               "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 2.0\n3 2 -1\n")
    with pytest.raises(matrixio.MatrixParseError, match="negative value -1.0 at row 3, column 2"):
        matrixio.load_sparse(p)


@pytest.mark.parametrize("text,msg", [
    ("garbage\n1 1 1\n", "missing MatrixMarket header"),
    ("%%MatrixMarket matrix coordinate real general\n% c\nx y\n", "malformed size line at line 3"),
    ("%%MatrixMarket matrix coordinate real general\n", "no size line found"),
])
def test_mtx_header_errors(tmp_path, text, msg):
    p = _write(tmp_path / "h.mtx", text)
    with pytest.raises(matrixio.MatrixParseError, match=msg):
        matrixio.load_matrix(p, "mtx")


def test_sparse_requires_mtx(tmp_path):
    p = _write(tmp_path / "c.csv", "1,2\n")
    with pytest.raises(ValueError, match="MatrixMarket"):
        matrixio.load_matrix(p, "csv", sparse=True)


def test_factor_and_trace_round_trip(tmp_path):
    from paper_2106_15214_b200.solver import FactorPair, FitResult, Termination, TraceRow

    rng = np.random.default_rng(0)
    w, h = rng.random((7, 3)) / 3.0, rng.random((3, 9)) * 1e-7
    trace = [TraceRow(1, 1.0 / 3.0, 0.25, 1e-9, 2e-9), TraceRow(2, 0.1, 0.5, 0.0, 1.0)]
    res = FitResult(factors=FactorPair(w, h), trace=trace, termination=Termination.CONVERGED,
                    iterations=2, config=None)
    matrixio.save_factors(res, str(tmp_path / "o"))
    w2, h2 = matrixio.load_factors(str(tmp_path / "o"))
    assert np.array_equal(w, w2) and np.array_equal(h, h2)   # %.17g is exact for float64
    matrixio.save_trace(res, str(tmp_path / "t.csv"))
    lines = open(tmp_path / "t.csv").read().splitlines()
    assert lines[0] == matrixio.TRACE_HEADER and len(lines) == 3
    assert float(lines[1].split(",")[1]) == 1.0 / 3.0


def test_summarize():
    assert harness.summarize([2.0]) == (2.0, 0.0, 2.0, 2.0)
    m, s, lo, hi = harness.summarize([1.0, 2.0, 3.0, 4.0])
    assert m == 2.5 and abs(s - np.std([1, 2, 3, 4], ddof=1)) < 1e-15
    assert abs(hi - lo - 2 * 1.96 * s / 2.0) < 1e-12
    with pytest.raises(ValueError):
        harness.summarize([])


@pytest.mark.parametrize("rank", [4, 9])   # exhaustive and assignment branches
def test_match_columns_recovers_permutation(rank):
    rng = np.random.default_rng(rank)
    wa = rng.random((50, rank))
    perm = rng.permutation(rank)
    wb = np.empty_like(wa)
    wb[:, perm] = wa * 2.0   # column k of wa sits at perm[k] of wb, scaled
    got, mismatch = harness.match_columns(wa, wb)
    assert np.array_equal(got, perm)
    assert abs(mismatch - 0.5) < 1e-12   # |a - 2a| / |2a|
    with pytest.raises(ValueError, match="shape mismatch"):
        harness.match_columns(wa, wb[:, :-1])


def test_run_bench_argument_checks():
    with pytest.raises(ValueError, match="jobs"):
        harness.run_bench(np.ones((3, 3)), 1.0, 1, jobs=2)
    with pytest.raises(ValueError, match="at least one seed"):
        harness.run_bench(np.ones((3, 3)), 1.0, 1, n_seeds=0)


def test_cli_argument_errors(capsys, tmp_path):
    assert cli.main(["fit", "--beta", "1", "--rank", "2", "--algo", "jmm",
                     "--out", str(tmp_path)]) == 1
    assert "either --input or --synthetic" in capsys.readouterr().err
    p = _write(tmp_path / "a.csv", "1,2\n")
    assert cli.main(["fit", "--input", p, "--synthetic", "3,3,1,0", "--beta", "1", "--rank", "1",
                     "--algo", "bmm", "--out", str(tmp_path)]) == 1
    assert "mutually exclusive" in capsys.readouterr().err
    bad = _write(tmp_path / "bad.csv", "1,-2\n")
    assert cli.main(["fit", "--input", bad, "--beta", "1", "--rank", "1", "--algo", "bmm",
                     "--out", str(tmp_path)]) == 1
    assert "negative value" in capsys.readouterr().err
    for spec in ("1,2,3", "0,2,1,0.1", "a,b,c,d"):
        with pytest.raises(SystemExit):
            cli.build_parser().parse_args(["fit", "--synthetic", spec, "--beta", "1",
                                           "--rank", "1", "--algo", "jmm", "--out", "x"])
    args = cli.build_parser().parse_args(["bench", "--synthetic", "5,6,2,0.1", "--beta", "0.5",
                                          "--rank", "2", "--kappa", "auto", "--dtype", "fp32"])
    assert args.kappa is None and args.dtype == "fp32" and args.seeds == 25 and args.jobs == 1


# ---------------------------------------------------------------- GPU ----

@pytest.mark.gpu
def test_cli_fit_matches_api(tmp_path):
    import paper_2106_15214_b200 as bn

    out = str(tmp_path / "fit")
    rc = cli.main(["fit", "--synthetic", "40,60,4,0.1", "--synthetic-seed", "3", "--beta", "1.5",
                   "--rank", "4", "--algo", "jmm", "--max-iters", "30", "--tol", "1e-300",
                   "--out", out])
    assert rc == 2   # stopped at the iteration cap
    w, h = matrixio.load_factors(out)
    v = bn.synthetic_low_rank(40, 60, 4, noise=0.1, seed=3)
    ref = bn.fit(v, bn.SolverConfig(beta=1.5, rank=4, algorithm="jmm", max_outer_iters=30,
                                    tol=1e-300, kappa=0.0))
    np.testing.assert_array_equal(w, ref.factors.w)
    np.testing.assert_array_equal(h, ref.factors.h)
    rows = open(os.path.join(out, "trace.csv")).read().splitlines()[1:]
    got = np.array([float(r.split(",")[1]) for r in rows])
    np.testing.assert_array_equal(got, [t.objective for t in ref.trace])


@pytest.mark.gpu
def test_cli_bench_report(tmp_path):
    rep = str(tmp_path / "r.json")
    rc = cli.main(["bench", "--synthetic", "30,50,3,0.1", "--beta", "0", "--rank", "3",
                   "--kappa", "auto", "--seeds", "2", "--max-iters", "40", "--report", rep])
    assert rc == 0
    d = json.load(open(rep))
    assert d["seeds"] == [0, 1] and set(d["algorithms"]) == {"bmm", "jmm"}
    assert d["acceleration_pct"] is not None and len(d["agreement"]) == 2
    for algo in ("bmm", "jmm"):
        assert len(d["algorithms"][algo]["runs"]) == 2


@pytest.mark.gpu
def test_sparse_mtx_end_to_end(tmp_path):
    import paper_2106_15214_b200 as bn

    rng = np.random.default_rng(5)
    m = sp.random(300, 200, density=0.05, random_state=5, format="coo")
    m.data = np.floor(rng.geometric(0.3, size=m.nnz)).astype(float)
    p = str(tmp_path / "s.mtx")
    mmwrite(p, m)
    csr = matrixio.load_sparse(p)
    cfg = bn.SolverConfig(beta=1.0, rank=5, algorithm="jmm", kappa=0.0, max_outer_iters=20,
                          tol=1e-300)
    a = bn.fit(csr, cfg, dtype="fp32")
    b = bn.fit(sp.csr_matrix(m), cfg, dtype="fp32")
    assert [t.objective for t in a.trace] == [t.objective for t in b.trace]
    out = str(tmp_path / "o")
    assert cli.main(["fit", "--input", p, "--format", "mtx", "--sparse", "--beta", "1",
                     "--rank", "5", "--algo", "jmm", "--max-iters", "20", "--tol", "1e-300",
                     "--out", out]) == 2
    w, _ = matrixio.load_factors(out)
    np.testing.assert_allclose(w, a.factors.w, rtol=0, atol=0)
