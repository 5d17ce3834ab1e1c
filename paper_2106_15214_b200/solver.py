"""Drop-in solver entry points: ``fit`` / ``run_jmm`` / ``run_bmm``.

Same names, arguments, defaults, errors and return type as the reference
(``/root/reference/pkg/src/betanmf/solver.py:49-326``); the outer loop runs in
libbnmf on a B200.  Host-side semantics that are not per-iteration work are
reproduced here: config validation (solver.py:62-114), kappa resolution and
domain checks (``_prepare``, solver.py:205-221), the seeded half-normal init
(solver.py:137-153) and the trace / termination assembly (solver.py:292-326).

Extensions (keyword-only, reference defaults preserved):
  ``dtype``     "fp64" (default; parity <= 1e-10) or "fp32" (B200 fast path)
  ``init``      a FactorPair / (W, H) replacing the seeded init
  ``device``    CUDA device index (default: current rank's device, else 0)
  ``kkt``       compute the per-iteration KKT residuals (default True, as the
                reference; they are excluded from ``TraceRow.seconds``)
  ``schedule``  "auto" | "reference" | "fused"
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from enum import Enum
from typing import NamedTuple

import numpy as np

from . import _native
from .core import (
    DEFAULT_FLOOR,
    DataMatrix,
    DivergenceDomainError,
    FactorPair,
    default_kappa,
    gamma_exponent,
)
from .updates import Algorithm, OpCounter  # noqa: F401  (re-exported)


class Termination(str, Enum):
    CONVERGED = "converged"
    MAX_ITERS = "max-iters"


class TraceRow(NamedTuple):
    iteration: int
    objective: float
    seconds: float
    kkt_w: float
    kkt_h: float


@dataclass
class SolverConfig:
    """Everything a fit needs besides the data (solver.py:62-114)."""

    beta: float
    rank: int
    algorithm: Algorithm = Algorithm.BMM
    sub_iters: int = 1
    sub_iters_w: int | None = None
    sub_iters_h: int | None = None
    tol: float = 1e-5
    kappa: float | None = None
    max_outer_iters: int = 5000
    seed: int = 0
    heuristic_gamma_one: bool = False
    denominator_floor: float = DEFAULT_FLOOR
    use_fast_path: bool | None = None

    def __post_init__(self):
        self.beta = float(self.beta)
        self.algorithm = Algorithm(self.algorithm)
        if self.rank < 1:
            raise ValueError("rank must be a positive integer")
        for name in ("sub_iters", "sub_iters_w", "sub_iters_h"):
            v = getattr(self, name)
            if v is not None and v < 1:
                raise ValueError(f"{name} must be a positive integer")
        if not self.tol > 0.0:
            raise ValueError("tol must be positive")
        if self.kappa is not None and self.kappa < 0.0:
            raise ValueError("kappa must be nonnegative")
        if self.max_outer_iters < 1:
            raise ValueError("max_outer_iters must be a positive integer")
        if not self.denominator_floor > 0.0:
            raise ValueError("denominator_floor must be positive")

    @property
    def gamma(self):
        return 1.0 if self.heuristic_gamma_one else gamma_exponent(self.beta)

    def fast_path_enabled(self):
        if self.use_fast_path is None:
            return self.beta in (0.0, 1.0, 2.0)
        return self.use_fast_path


@dataclass
class FitResult:
    """Final factors plus the per-iteration trace (solver.py:117-134)."""

    factors: FactorPair
    trace: list
    termination: Termination
    iterations: int
    config: SolverConfig = field(repr=False, default=None)

    @property
    def objective(self):
        return self.trace[-1].objective

    @property
    def kkt(self):
        last = self.trace[-1]
        return last.kkt_w, last.kkt_h


def init_factors(n_rows, n_cols, rank, seed):
    """Half-normal factors |z|, z ~ N(0,1) from numpy's PCG64 default_rng(seed),
    W drawn before H, exact zeros redrawn (solver.py:137-153)."""
    rng = np.random.default_rng(seed)

    def half_normal(shape):
        m = np.abs(rng.standard_normal(shape))
        while (m == 0.0).any():
            zeros = m == 0.0
            m[zeros] = np.abs(rng.standard_normal(int(zeros.sum())))
        return m

    return FactorPair(half_normal((n_rows, rank)), half_normal((rank, n_cols)))


def normalize(factors):
    """Unit-l2 columns of W, rows of H scaled inversely (solver.py:156-171)."""
    w, h = factors.w, factors.h
    norms = np.sqrt(np.sum(w * w, axis=0))
    if (norms == 0.0).any():
        raise ValueError("cannot normalize: a column of the first factor is zero")
    return FactorPair(w / norms, h * norms[:, None])


def should_stop(prev_obj, curr_obj, tol):
    """Relative-decrease rule (solver.py:174-180); also evaluated on device."""
    if curr_obj == prev_obj:
        return True
    if curr_obj <= 0.0:
        return False
    return (prev_obj - curr_obj) / curr_obj <= tol


def synthetic_low_rank(n_rows, n_cols, rank, noise=0.1, seed=0, density=1.0):
    """Low-rank plus folded-Gaussian noise test data (solver.py:183-202)."""
    rng = np.random.default_rng(seed + 0x5EED)
    truth = init_factors(n_rows, n_cols, rank, seed)
    w, h = truth.w, truth.h
    if density < 1.0:
        w = w * (rng.random(w.shape) < density)
        h = h * (rng.random(h.shape) < density)
    return w @ h + noise * np.abs(rng.standard_normal((n_rows, n_cols)))


def _prepare(data, config):
    """kappa resolution + domain checks (solver.py:205-221)."""
    if isinstance(data, DataMatrix):
        values = data.values
        kappa = config.kappa if config.kappa is not None else data.kappa
    else:
        values = np.asarray(data)
        if values.dtype not in (np.float64, np.float32):
            values = values.astype(np.float64)
        kappa = config.kappa
    if kappa is None:
        kappa = default_kappa(values, config.beta)
    data = DataMatrix(values, kappa)
    data.check_domain(config.beta)
    if config.beta <= 0.0 and float(data.values.min()) + data.kappa <= 0.0:
        raise DivergenceDomainError(
            f"data entries must be positive for beta={config.beta}; "
            f"set a positive kappa shift")
    return data


# Inputs at least this large are checked from device statistics of the
# upload (a host scan of V costs ~1 s per 10^9 entries); smaller ones are
# checked on the host before any device work, exactly like the reference.
_DEVICE_CHECK_MIN = 1 << 24


def _upload_checked(ctx, values, config):
    """Upload V and apply the checks of DataMatrix.__post_init__, check_domain
    and _prepare (core.py:188-228, solver.py:205-221) to device statistics of
    the upload, in the reference's order and with its messages.  Returns the
    (values-free) DataMatrix stand-in (shape, kappa) and F, N."""
    if values.dtype not in (np.float64, np.float32):
        values = values.astype(np.float64)
    if values.ndim != 2 or min(values.shape) < 1:
        raise ValueError("data must be a 2-D matrix with positive dimensions")
    kappa = config.kappa
    ctx.set_dense(values, 0.0 if kappa is None else kappa)
    vmin, _vmax, vsum, nonfinite, count = ctx.data_stats()
    kappa_in = kappa
    kappa = _check_global(vmin, nonfinite, vsum, count, config, kappa)
    if kappa_in is None and kappa != 0.0:
        ctx.set_dense(values, kappa)
    F, N = values.shape
    return _Checked((F, N), kappa), F, N


class _Checked:
    """shape / kappa of device-checked data (what _run reads of a DataMatrix)"""

    def __init__(self, shape, kappa):
        self.shape = shape
        self.kappa = kappa


# ----------------------------------------------------------------------------
# native execution

_ctx_cache = {}
_ctx_lock = threading.Lock()


def _default_device():
    import os
    lr = os.environ.get("LOCAL_RANK")
    return int(lr) if lr is not None else 0


def get_context(device=None, dtype="fp64"):
    """Shared per-(device, dtype) libbnmf context (created on first use)."""
    device = _default_device() if device is None else int(device)
    key = (device, dtype)
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            ctx = _native.Context(device, "fp32" if dtype == "fp32-sparse" else dtype)
            ctx.lock = threading.Lock()
            _ctx_cache[key] = ctx
        return ctx


def make_params(config, kappa, kkt=True, schedule="auto"):
    p = _native.Params()
    p.algorithm = _native.BNMF_JMM if config.algorithm == Algorithm.JMM else _native.BNMF_BMM
    p.sub_iters = int(config.sub_iters)
    p.sub_iters_w = int(config.sub_iters_w or 0)
    p.sub_iters_h = int(config.sub_iters_h or 0)
    p.beta = float(config.beta)
    p.gamma = float(config.gamma)
    p.kappa = float(kappa)
    p.floor = float(config.denominator_floor)
    p.tol = float(config.tol)
    p.compute_kkt = 1 if kkt else 0
    p.schedule = _native.SCHED[schedule]
    return p


def _count_ops(counter, config, iterations):
    if counter is None:
        return
    if config.algorithm == Algorithm.JMM:
        counter.anchor_products += iterations
        counter.w_updates += config.sub_iters * iterations
        counter.h_updates += config.sub_iters * iterations
    else:
        lw = config.sub_iters_w or config.sub_iters
        lh = config.sub_iters_h or config.sub_iters
        counter.kernel_products += (lw + lh) * iterations
        counter.w_updates += lw * iterations
        counter.h_updates += lh * iterations
    counter.objective_products += iterations


def _resolve_init(init, F, N, K, seed, device_checked=False):
    """FactorPair of the init.  ``device_checked``: an array init of >= 2^24
    entries skips the host finiteness / positivity scans, which
    Context.set_factors then makes on the device copy with the same messages
    (core.py FactorPair.__post_init__)."""
    if init is None:
        return init_factors(F, N, K, seed)
    if isinstance(init, FactorPair):
        pair = init
    elif device_checked and np.asarray(init[1]).size >= _DEVICE_CHECK_MIN:
        w = np.asarray(init[0], dtype=float)
        h = np.asarray(init[1], dtype=float)
        if w.ndim != 2 or h.ndim != 2:
            raise ValueError("factors must be 2-D matrices")
        if w.shape[1] != h.shape[0]:
            raise ValueError(f"inner dimensions disagree: w is {w.shape}, h is {h.shape}")
        pair = _unchecked_pair(w, h)
    else:
        pair = FactorPair(*init)
    if pair.w.shape != (F, K) or pair.h.shape != (K, N):
        raise ValueError(f"init shapes {pair.w.shape}, {pair.h.shape} do not match "
                         f"data {(F, N)} at rank {K}")
    return pair


def _unchecked_pair(w, h):
    pair = FactorPair.__new__(FactorPair)
    pair.w, pair.h = w, h
    return pair


def _attach_comm(ctx, n_global):
    """Join the NCCL communicator of the current process group (once per ctx)."""
    from . import parallel
    rank, world = parallel.dist_info()
    key = (rank, world, n_global)
    if getattr(ctx, "comm_key", None) == key:
        return
    uid = parallel.broadcast_uid(_native.Context.nccl_unique_id)
    ctx.init_comm(rank, world, uid, n_global)
    ctx.comm_key = key


def _run(data, config, counter, algorithm, *, dtype="fp64", init=None, device=None,
         kkt=True, schedule="auto", sharded=False):
    if config.algorithm != algorithm:
        raise ValueError(f"config.algorithm must be '{algorithm.value}' for "
                         f"run_{algorithm.value}")
    if dtype not in ("fp64", "fp32"):
        raise ValueError("dtype must be 'fp64' or 'fp32'")
    if sharded:
        # `data` is this rank's column block; kappa and the init are global
        return _run_sharded_dense(data, config, counter, dtype=dtype, init=init, device=device,
                                  kkt=kkt, schedule=schedule)
    if isinstance(data, DataMatrix) or np.asarray(data).size < _DEVICE_CHECK_MIN:
        data = _prepare(data, config)
        F, N = data.shape
        pair = _resolve_init(init, F, N, config.rank, config.seed)
    else:
        # plain array: the DataMatrix checks run on device statistics of the
        # upload (same order, same errors), not as host scans of V
        values = np.asarray(data)
        data = None
    ctx = get_context(device, dtype)
    with ctx.lock:
        if data is None:
            data, F, N = _upload_checked(ctx, values, config)
            pair = _resolve_init(init, F, N, config.rank, config.seed, device_checked=True)
        else:
            ctx.set_dense(data.values, data.kappa)
        ctx.set_factors(pair.w, pair.h)
        params = make_params(config, data.kappa, kkt=kkt, schedule=schedule)
        done, converged = ctx.run(params, config.max_outer_iters)
        obj, sec, kk = ctx.trace(done)
        w, h = ctx.factors()
    trace = [TraceRow(i + 1, float(obj[i]), float(sec[i]), float(kk[i, 0]), float(kk[i, 1]))
             for i in range(done)]
    _count_ops(counter, config, done)
    # the factors are produced by the device loop (strictly positive unless an
    # fp32 entry underflows to 0, which is reported as is): no host re-scan
    factors = _unchecked_pair(w, h)
    return FitResult(factors=factors, trace=trace,
                     termination=Termination.CONVERGED if converged else Termination.MAX_ITERS,
                     iterations=done, config=config)


def _check_global(vmin, nonfinite, vsum, count, config, kappa):
    """The checks of DataMatrix / check_domain / _prepare (core.py:188-228,
    solver.py:205-221) on statistics of the whole (possibly sharded) matrix;
    returns the resolved kappa."""
    if nonfinite > 0:
        raise ValueError("data entries must be finite")
    if vmin < 0.0:
        raise ValueError("data entries must be nonnegative")
    if kappa is None:
        # default_kappa (core.py:176-185)
        kappa = 0.0 if (1.0 <= config.beta <= 2.0 and vmin > 0.0) else 1e-9 * (vsum / count)
    kappa = float(kappa)
    if not np.isfinite(kappa) or kappa < 0.0:
        raise ValueError("kappa must be a nonnegative finite real")
    if config.beta < 1.0 and kappa == 0.0 and vmin == 0.0:
        raise DivergenceDomainError(
            f"data contains zeros, which is outside the domain of "
            f"d_beta for beta={config.beta}; set a positive kappa shift")
    if config.beta <= 0.0 and vmin + kappa <= 0.0:
        raise DivergenceDomainError(
            f"data entries must be positive for beta={config.beta}; "
            f"set a positive kappa shift")
    return kappa


def _run_sharded_dense(data, config, counter, *, dtype, init, device, kkt, schedule):
    """N-column sharded fit: this rank's column block of V.

    Every rank uploads its block and reads device statistics of it
    (bnmf_data_stats: min, non-finite count, fp64 sum); the statistics are
    allreduced, so every rank applies the reference's checks to the same
    global numbers and raises the same error before any communicator exists
    (no rank can be left waiting in a collective)."""
    from . import parallel
    if parallel.dist_info() is None:
        raise ValueError("sharded=True needs an initialised torch.distributed group")
    if isinstance(data, DataMatrix):
        vals = data.values
        kappa = config.kappa if config.kappa is not None else data.kappa
    else:
        vals = np.asarray(data)
        kappa = config.kappa
    if vals.dtype not in (np.float64, np.float32):
        vals = vals.astype(np.float64)
    # shape errors are local: agree on them first
    local_err = None
    if vals.ndim != 2 or min(vals.shape) < 1:
        local_err = ValueError("data must be a 2-D matrix with positive dimensions")
    parallel.agree_on_error(local_err)
    n0, n_global = parallel.column_offsets(vals.shape[1])
    F, N = vals.shape
    fs = parallel.allgather_int(F)
    if len(set(fs)) != 1:
        raise ValueError("every rank's column block must have the global row count")
    ctx = get_context(device, dtype)
    with ctx.lock:
        ctx.set_dense(vals, 0.0 if kappa is None else kappa)
        vmin, _vmax, vsum, nonfinite, count = ctx.data_stats()
        gmin = float(parallel.allreduce_scalars([vmin], "min")[0])
        gnf, gsum, gcnt = (float(x) for x in parallel.allreduce_scalars(
            [nonfinite, vsum, count], "sum"))
        kappa_in = kappa
        kappa = _check_global(gmin, gnf, gsum, gcnt, config, kappa)   # same on every rank
        if kappa_in is None and kappa != 0.0:
            ctx.set_dense(vals, kappa)
        local_err = None
        pair = None
        try:
            if init is None:
                full = init_factors(F, n_global, config.rank, config.seed)
                init = (full.w, full.h)
            w0, h0 = init if not isinstance(init, FactorPair) else (init.w, init.h)
            w0, h0 = parallel.slice_init(w0, h0, n0, N, n_global)
            pair = _resolve_init((w0, h0), F, N, config.rank, config.seed)
        except ValueError as e:
            local_err = e
        parallel.agree_on_error(local_err)
        _attach_comm(ctx, n_global)
        ctx.set_factors(pair.w, pair.h)
        params = make_params(config, kappa, kkt=kkt, schedule=schedule)
        done, converged = ctx.run(params, config.max_outer_iters)
        obj, sec, kk = ctx.trace(done)
        w, h = ctx.factors()
    trace = [TraceRow(i + 1, float(obj[i]), float(sec[i]), float(kk[i, 0]), float(kk[i, 1]))
             for i in range(done)]
    _count_ops(counter, config, done)
    return FitResult(factors=_unchecked_pair(w, h), trace=trace,
                     termination=Termination.CONVERGED if converged else Termination.MAX_ITERS,
                     iterations=done, config=config)


def _is_sparse(data):
    try:
        import scipy.sparse as sp
    except Exception:  # pragma: no cover
        return False
    return sp.issparse(data)


def csr_with_csc_view(data):
    """CSR arrays of a scipy.sparse matrix plus its CSC view (colptr, row
    indices, perm[j] = CSR position of CSC entry j) -- the deterministic
    column-sum layout of the sparse path."""
    import scipy.sparse as sp
    m = sp.csr_matrix(data, dtype=np.float32, copy=True)
    m.sum_duplicates()
    m.sort_indices()
    F, N = m.shape
    rows = np.repeat(np.arange(F, dtype=np.int64), np.diff(m.indptr))
    order = np.lexsort((rows, m.indices))           # by column, then row
    colptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(np.bincount(m.indices, minlength=N), out=colptr[1:])
    return (m.indptr.astype(np.int64), m.indices.astype(np.int32), m.data.astype(np.float32),
            colptr, rows[order].astype(np.int32), order.astype(np.int32)), (F, N)


def _run_sparse(data, config, counter, algorithm, *, dtype="fp32", init=None, device=None,
                kkt=True, schedule="auto", sharded=False):
    """Sparse KL path (config 5): beta = 1, kappa = 0, fp32 on the device.

    The reference densifies sparse input (matrixio.py:115-128) and would apply
    the default kappa rule (1e-9 * mean, core.py:176-185) because V has zeros;
    a positive shift densifies the problem, so the sparse path requires
    kappa = 0 (or None, read as 0)."""
    if config.algorithm != algorithm:
        raise ValueError(f"config.algorithm must be '{algorithm.value}' for "
                         f"run_{algorithm.value}")
    if config.beta != 1.0:
        raise ValueError("the sparse path implements beta = 1 (KL) only")
    if config.kappa not in (None, 0.0):
        raise ValueError("sparse input needs kappa = 0 (a positive shift densifies V)")
    if (config.sub_iters != 1 or (config.sub_iters_w or 1) != 1
            or (config.sub_iters_h or 1) != 1):
        raise ValueError("the sparse path implements one sub-iteration")
    import scipy.sparse as sp
    m = sp.csr_matrix(data, dtype=np.float32)
    local_err = None
    if not np.isfinite(m.data).all():
        local_err = ValueError("data entries must be finite")
    elif m.data.size and m.data.min() < 0.0:
        local_err = ValueError("data entries must be nonnegative")
    elif m.nnz >= 2**31 - 1:
        local_err = ValueError("the sparse path takes fewer than 2^31 - 1 nonzeros per device")
    if sharded:
        from . import parallel
        if parallel.dist_info() is None:
            raise ValueError("sharded=True needs an initialised torch.distributed group")
        parallel.agree_on_error(local_err)   # every rank raises, none waits in a collective
    elif local_err is not None:
        raise local_err
    arrays, (F, N) = csr_with_csc_view(m)
    if sharded:
        # `data` is this rank's row block: W rows are local,
        # H is replicated; the init is global (or this rank's W rows)
        f0, f_global = parallel.column_offsets(F)   # offsets of a 1-D partition
        counts = parallel.allgather_int(N)
        if len(set(counts)) != 1:
            raise ValueError("every rank's row block must have the global column count")
        K = config.rank
        if init is None:
            full = init_factors(f_global, N, K, config.seed)
            w0, h0 = full.w, full.h
        else:
            w0, h0 = (init.w, init.h) if isinstance(init, FactorPair) else init
        w0 = np.asarray(w0, dtype=np.float64)
        h0 = np.asarray(h0, dtype=np.float64)
        if w0.shape == (f_global, K):
            w0 = w0[f0:f0 + F]
        local_err = None
        if w0.shape != (F, K) or h0.shape != (K, N):
            local_err = ValueError(f"init shapes {w0.shape}, {h0.shape} do not match the global "
                                   f"{(f_global, N)} or local {(F, N)} data at rank {K}")
        parallel.agree_on_error(local_err)
        w_init, h_init = w0, h0
    else:
        pair = _resolve_init(init, F, N, config.rank, config.seed)
        w_init, h_init = pair.w, pair.h
    ctx = get_context(device, "fp32-sparse")
    with ctx.lock:
        ctx.set_csr(*arrays, (F, N))   # switches the context to the sparse engine first
        if sharded:
            _attach_comm(ctx, f_global)
        ctx.set_factors(w_init, h_init)
        params = make_params(config, 0.0, kkt=kkt, schedule="reference")
        done, converged = ctx.run(params, config.max_outer_iters)
        obj, sec, kk = ctx.trace(done)
        w, h = ctx.factors()
    trace = [TraceRow(i + 1, float(obj[i]), float(sec[i]), float(kk[i, 0]), float(kk[i, 1]))
             for i in range(done)]
    _count_ops(counter, config, done)
    try:
        factors = FactorPair(w, h)
    except ValueError:
        factors = _unchecked_pair(w, h)
    return FitResult(factors=factors, trace=trace,
                     termination=Termination.CONVERGED if converged else Termination.MAX_ITERS,
                     iterations=done, config=config)


def run_bmm(data, config, counter=None, **options):
    """Block (alternating) MU updates (solver.py:224-248).  A scipy.sparse
    ``data`` runs the sparse KL path."""
    if _is_sparse(data):
        return _run_sparse(data, config, counter, Algorithm.BMM, **options)
    return _run(data, config, counter, Algorithm.BMM, **options)


def run_jmm(data, config, counter=None, **options):
    """Joint MM updates (solver.py:251-282).  A scipy.sparse ``data`` runs the
    sparse KL path."""
    if _is_sparse(data):
        return _run_sparse(data, config, counter, Algorithm.JMM, **options)
    return _run(data, config, counter, Algorithm.JMM, **options)


def fit(data, config, counter=None, **options):
    """Run the family selected by ``config.algorithm`` (solver.py:285-289)."""
    if config.algorithm == Algorithm.BMM:
        return run_bmm(data, config, counter, **options)
    return run_jmm(data, config, counter, **options)
