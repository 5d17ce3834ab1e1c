"""Multi-seed comparison of the two update families on the device.

Mirrors the reference harness ``betanmf.bench`` (``/root/reference/pkg/src/betanmf/bench.py``):
for every seed both families start from identical half-normal factors (the reference's
``init_factors``, solver.py:137-153), the harness collects the solver-loop seconds, final raw and
per-entry objectives, KKT residuals and iteration counts, summarises them with mean, sample
standard deviation and a normal 95 % interval (bench.py:26-40), reports the joint-update
acceleration (bench.py:172-177) and matches the two solutions column-wise per seed
(bench.py:178-182, diagnostics.py:93-130).

Differences from the reference, all because the work runs on one GPU:
* every fit goes through :func:`paper_2106_15214_b200.fit` (libbnmf), with the ``dtype`` and
  ``device`` keywords passed through;
* ``jobs > 1`` is refused: fits on one device are serialised on its stream anyway, and the
  reference's process pool only exists to spread CPU fits over cores (bench.py:150-154).
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass, field
from itertools import permutations

import numpy as np

from .solver import SolverConfig, fit
from .updates import Algorithm

#: ranks up to this are matched exhaustively, above by optimal assignment (diagnostics.py:19)
EXHAUSTIVE_MATCH_LIMIT = 7


def summarize(values):
    """Mean, sample standard deviation (n-1) and mean +/- 1.96 std / sqrt(n)."""
    values = [float(v) for v in values]
    if not values:
        raise ValueError("cannot summarize an empty sequence")
    n = len(values)
    mean = sum(values) / n
    if n == 1:
        return mean, 0.0, mean, mean
    std = math.sqrt(sum((v - mean) ** 2 for v in values) / (n - 1))
    half = 1.96 * std / math.sqrt(n)
    return mean, std, mean - half, mean + half


def match_columns(wa, wb):
    """Column permutation of ``wb`` maximising the total cosine similarity with ``wa`` and the
    worst matched relative l2 column difference (diagnostics.py:93-130)."""
    wa = np.asarray(wa, dtype=float)
    wb = np.asarray(wb, dtype=float)
    if wa.shape != wb.shape:
        raise ValueError(f"shape mismatch: {wa.shape} vs {wb.shape}")
    rank = wa.shape[1]
    na = np.linalg.norm(wa, axis=0)
    nb = np.linalg.norm(wb, axis=0)
    sim = (wa.T @ wb) / np.outer(np.maximum(na, 1e-300), np.maximum(nb, 1e-300))
    if rank <= EXHAUSTIVE_MATCH_LIMIT:
        idx = np.arange(rank)
        perm = np.array(max(permutations(range(rank)), key=lambda p: sim[idx, list(p)].sum()))
    else:
        from scipy.optimize import linear_sum_assignment

        rows, cols = linear_sum_assignment(sim, maximize=True)
        perm = cols[np.argsort(rows)]
    diffs = np.linalg.norm(wa - wb[:, perm], axis=0)
    scales = np.maximum(np.maximum(na, nb[perm]), 1e-300)
    return perm, float(np.max(diffs / scales))


@dataclass
class SeedRun:
    seed: int
    seconds: float
    objective: float
    objective_per_entry: float
    kkt_w: float
    kkt_h: float
    iterations: int
    termination: str


@dataclass
class AlgorithmStats:
    mean_seconds: float
    std_seconds: float
    ci95_seconds: tuple
    mean_objective: float
    mean_objective_per_entry: float
    mean_kkt_w: float
    mean_kkt_h: float
    runs: list = field(default_factory=list)


@dataclass
class BenchReport:
    """``acceleration_pct`` = (mean bmm seconds - mean jmm seconds) / mean bmm seconds * 100."""

    shape: tuple
    beta: float
    rank: int
    seeds: list
    algorithms: dict
    acceleration_pct: float | None = None
    agreement: list | None = None
    dtype: str = "fp64"

    def to_dict(self):
        return dataclasses.asdict(self)


def _entries(values):
    return values.shape[0] * values.shape[1]


def run_bench(values, beta, rank, n_seeds=25, algorithms=("bmm", "jmm"), base_seed=0, jobs=1,
              dtype="fp64", device=None, **config_kwargs):
    """Seed-paired comparison (bench.py:112-192) with every fit on the device."""
    if jobs != 1:
        raise ValueError("jobs > 1 is not supported: fits on one device run back to back")
    if n_seeds < 1:
        raise ValueError("need at least one seed")
    import scipy.sparse as sp

    if not sp.issparse(values):
        values = np.asarray(values, dtype=float)
    algorithms = [Algorithm(a).value for a in algorithms]
    seeds = [base_seed + i for i in range(n_seeds)]
    runs = {a: [] for a in algorithms}
    final_w = {a: {} for a in algorithms}
    for seed in seeds:
        for algo in algorithms:
            cfg = SolverConfig(beta=beta, rank=rank, algorithm=Algorithm(algo), seed=seed,
                               **config_kwargs)
            res = fit(values, cfg, dtype=dtype, device=device)
            last = res.trace[-1]
            runs[algo].append(SeedRun(seed=seed, seconds=last.seconds, objective=last.objective,
                                      objective_per_entry=last.objective / _entries(values),
                                      kkt_w=last.kkt_w, kkt_h=last.kkt_h,
                                      iterations=res.iterations,
                                      termination=res.termination.value))
            final_w[algo][seed] = res.factors.w
    stats = {}
    for algo in algorithms:
        rows = runs[algo]
        mean_s, std_s, lo, hi = summarize([r.seconds for r in rows])
        stats[algo] = AlgorithmStats(
            mean_seconds=mean_s, std_seconds=std_s, ci95_seconds=(lo, hi),
            mean_objective=float(np.mean([r.objective for r in rows])),
            mean_objective_per_entry=float(np.mean([r.objective_per_entry for r in rows])),
            mean_kkt_w=float(np.mean([r.kkt_w for r in rows])),
            mean_kkt_h=float(np.mean([r.kkt_h for r in rows])),
            runs=rows)
    acceleration = agreement = None
    if "bmm" in stats and "jmm" in stats:
        b, j = stats["bmm"].mean_seconds, stats["jmm"].mean_seconds
        acceleration = 100.0 * (b - j) / b if b > 0 else None
        agreement = [{"seed": s, "mismatch": match_columns(final_w["bmm"][s], final_w["jmm"][s])[1]}
                     for s in seeds]
    return BenchReport(shape=(values.shape[0], values.shape[1]), beta=float(beta), rank=int(rank),
                       seeds=seeds, algorithms=stats, acceleration_pct=acceleration,
                       agreement=agreement, dtype=dtype)


def format_report(report):
    """Human-readable summary (bench.py:195-215)."""
    lines = [f"data {report.shape[0]} x {report.shape[1]}, beta={report.beta:g}, "
             f"rank={report.rank}, seeds={len(report.seeds)}, dtype={report.dtype}"]
    for algo, st in report.algorithms.items():
        lines.append(
            f"  {algo}: {st.mean_seconds:.4f}s (std {st.std_seconds:.4f}, "
            f"95% CI [{st.ci95_seconds[0]:.4f}, {st.ci95_seconds[1]:.4f}]), "
            f"objective {st.mean_objective:.6g} ({st.mean_objective_per_entry:.6g}/entry), "
            f"kkt ({st.mean_kkt_w:.3g}, {st.mean_kkt_h:.3g})")
    if report.acceleration_pct is not None:
        lines.append(f"  joint-update acceleration: {report.acceleration_pct:.1f}%")
    if report.agreement:
        lines.append(f"  worst per-seed column mismatch: "
                     f"{max(a['mismatch'] for a in report.agreement):.3g}")
    return "\n".join(lines)
