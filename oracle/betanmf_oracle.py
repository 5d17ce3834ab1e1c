"""CPU ORACLE -- test infrastructure only.

This module is a plain-numpy restatement of the reference ``betanmf`` solver
(arXiv 2106.15214, joint-MM beta-NMF), used ONLY as the checker:

* by ``tests/`` (parity of the CUDA path against this restatement),
* by ``__graft_entry__.smoke()`` (one small check on cuda:0),
* by ``bench.py`` for the ``cpu_baseline`` leg and ``--impl reference``.

The product path (``paper_2106_15214_b200``) never imports it: it runs the
CUDA extension or fails.  Every function cites the reference file:line it
restates (paths relative to ``/root/reference/pkg/src/betanmf``).

Parity of this restatement is PINNED: ``tests/golden/gen_golden.py`` imports
the reference itself (in the build container) and records fits, hand
examples and update-kernel outputs as ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this module against every fixture.
"""

from __future__ import annotations

import numpy as np

DEFAULT_FLOOR = 1e-300  # core.py:18


# ----------------------------------------------------------------------------
# core.py restatements


def gamma_exponent(beta):
    """core.py:29-39 -- 1/(2-b) below 1, 1 on [1,2], 1/(b-1) above 2."""
    if beta < 1.0:
        return 1.0 / (2.0 - beta)
    if beta <= 2.0:
        return 1.0
    return 1.0 / (beta - 1.0)


def _xlogy(x, y):
    # scipy.special.xlogy semantics used at core.py:101: 0 where x == 0.
    out = np.zeros(np.broadcast_shapes(np.shape(x), np.shape(y)))
    x = np.broadcast_to(x, out.shape)
    y = np.broadcast_to(y, out.shape)
    nz = x != 0
    out[nz] = x[nz] * np.log(y[nz])
    return out


def beta_divergence_elements(x, y, beta):
    """core.py:89-109 -- entrywise d_beta(x | y)."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    if beta == 2.0:
        d = x - y
        return 0.5 * d * d
    if beta == 1.0:
        return _xlogy(x, x / y) - x + y
    if beta == 0.0:
        r = x / y
        return r - np.log(r) - 1.0
    return (np.power(x, beta) / (beta * (beta - 1.0))
            + np.power(y, beta) / beta
            - x * np.power(y, beta - 1.0) / (beta - 1.0))


def divergence_total(x, y, beta):
    """core.py:112-114."""
    return float(np.sum(beta_divergence_elements(x, y, beta)))


def guarded_divide(num, den, floor=DEFAULT_FLOOR):
    """core.py:117-130 -- num / max(den, floor)."""
    return num / np.maximum(den, floor)


def power_pair(m, p):
    """core.py:156-173 -- (m**p, m**(p+1)); None = all-ones."""
    if p == -2.0:
        a = 1.0 / (m * m)
        return a, 1.0 / m
    if p == -1.0:
        return 1.0 / m, None
    if p == 0.0:
        return None, m
    if p == 1.0:
        return m, m * m
    a = np.power(m, p)
    return a, a * m


def default_kappa(values, beta):
    """core.py:176-185."""
    values = np.asarray(values, dtype=float)
    if 1.0 <= beta <= 2.0 and values.min() > 0.0:
        return 0.0
    return 1e-9 * float(values.mean())


# ----------------------------------------------------------------------------
# updates.py restatements


def chi1(m, mt, beta):
    """updates.py:84-97."""
    if beta >= 2.0:
        return m
    if beta == 1.0:
        return mt
    if beta == 0.0:
        return (mt * mt) / m
    return np.power(mt, 2.0 - beta) * np.power(m, beta - 1.0)


def chi2(m, mt, beta):
    """updates.py:100-107."""
    if beta <= 1.0:
        return m
    if beta == 2.0:
        return (m * m) / mt
    return np.power(m, beta) / np.power(mt, beta - 1.0)


def apply_exponent(ratio, gamma):
    """updates.py:118-123."""
    if gamma == 1.0:
        return ratio
    if gamma == 0.5:
        return np.sqrt(ratio)
    return np.power(ratio, gamma)


def _times_ht(x, h, rows):
    """updates.py:126-130 -- x @ h.T, None -> row-sum broadcast."""
    if x is None:
        return np.broadcast_to(h.sum(axis=1), (rows, h.shape[0]))
    return x @ h.T


def _wt_times(w, x, cols):
    """updates.py:133-137 -- w.T @ x, None -> column-sum broadcast."""
    if x is None:
        return np.broadcast_to(w.sum(axis=0)[:, None], (w.shape[1], cols))
    return w.T @ x


def joint_bases(v, product, beta):
    """updates.py:184-200."""
    if beta == 2.0:
        return v, product
    if beta == 1.0:
        return v / product, None
    if beta == 0.0:
        return v / (product * product), 1.0 / product
    low, high = power_pair(product, beta - 2.0)
    return (v if low is None else v * low), high


def bmm_update_w(v, w, h, beta, kappa, gamma, floor):
    """updates.py:157-170 (general) / 243-259 (beta in {0,1,2})."""
    p = w @ h
    if kappa:
        p += kappa
    if beta == 0.0:
        num, den = (v / (p * p)) @ h.T, (1.0 / p) @ h.T
    elif beta == 1.0:
        num = (v / p) @ h.T
        den = np.broadcast_to(h.sum(axis=1), (w.shape[0], h.shape[0]))
    elif beta == 2.0:
        num, den = v @ h.T, p @ h.T
    else:
        low, high = power_pair(p, beta - 2.0)
        num = _times_ht(v if low is None else v * low, h, w.shape[0])
        den = _times_ht(high, h, w.shape[0])
    return w * apply_exponent(guarded_divide(num, den, floor), gamma)


def bmm_update_h(v, w, h, beta, kappa, gamma, floor):
    """updates.py:173-181 (general) / 262-278 (beta in {0,1,2})."""
    p = w @ h
    if kappa:
        p += kappa
    if beta == 0.0:
        num, den = w.T @ (v / (p * p)), w.T @ (1.0 / p)
    elif beta == 1.0:
        num = w.T @ (v / p)
        den = np.broadcast_to(w.sum(axis=0)[:, None], (h.shape[0], h.shape[1]))
    elif beta == 2.0:
        num, den = w.T @ v, w.T @ p
    else:
        low, high = power_pair(p, beta - 2.0)
        num = _wt_times(w, v if low is None else v * low, h.shape[1])
        den = _wt_times(w, high, h.shape[1])
    return h * apply_exponent(guarded_divide(num, den, floor), gamma)


def jmm_update_w(bases, wt, ht, h_cur, beta, gamma, floor):
    """updates.py:203-220 (general; == fast path 281-307 for beta in {0,1,2})."""
    num_base, den_base = bases
    rows = wt.shape[0]
    num = _times_ht(num_base, chi1(h_cur, ht, beta), rows)
    den = _times_ht(den_base, chi2(h_cur, ht, beta), rows)
    return wt * apply_exponent(guarded_divide(num, den, floor), gamma)


def jmm_update_h(bases, wt, ht, w_cur, beta, gamma, floor):
    """updates.py:223-235 (general; == fast path 310-331 for beta in {0,1,2})."""
    num_base, den_base = bases
    cols = ht.shape[1]
    num = _wt_times(chi1(w_cur, wt, beta), num_base, cols)
    den = _wt_times(chi2(w_cur, wt, beta), den_base, cols)
    return ht * apply_exponent(guarded_divide(num, den, floor), gamma)


# ----------------------------------------------------------------------------
# diagnostics.py / solver.py restatements


def kkt_residuals_arrays(x, w, h, beta, kappa=0.0):
    """diagnostics.py:46-59."""
    p = w @ h
    if kappa:
        p += kappa
    if beta == 2.0:
        g = p - x
    else:
        e = beta - 2.0
        if e == 0.0:
            pw = np.ones_like(p)
        elif e == 1.0:
            pw = p
        elif e == 2.0:
            pw = p * p
        elif e == -1.0:
            pw = 1.0 / p
        elif e == -2.0:
            pw = 1.0 / (p * p)
        elif e == 0.5:
            pw = np.sqrt(p)
        else:
            pw = np.power(p, e)
        g = pw * (p - x)
    gw = g @ h.T
    gh = w.T @ g
    res_w = float(np.abs(np.minimum(w, gw)).sum()) / (w.shape[0] * w.shape[1])
    res_h = float(np.abs(np.minimum(h, gh)).sum()) / (h.shape[0] * h.shape[1])
    return res_w, res_h


def init_factors(n_rows, n_cols, rank, seed):
    """solver.py:137-153 -- half-normal PCG64 draws, W first, zeros redrawn."""
    rng = np.random.default_rng(seed)

    def half_normal(shape):
        m = np.abs(rng.standard_normal(shape))
        while (m == 0.0).any():
            zeros = m == 0.0
            m[zeros] = np.abs(rng.standard_normal(int(zeros.sum())))
        return m

    w = half_normal((n_rows, rank))
    h = half_normal((rank, n_cols))
    return w, h


def normalize_arrays(w, h):
    """solver.py:167-171."""
    norms = np.sqrt(np.sum(w * w, axis=0))
    return w / norms, h * norms[:, None]


def should_stop(prev_obj, curr_obj, tol):
    """solver.py:174-180."""
    if curr_obj == prev_obj:
        return True
    if curr_obj <= 0.0:
        return False
    return (prev_obj - curr_obj) / curr_obj <= tol


def resolve_kappa(values, beta, kappa):
    """solver.py:205-221 (kappa None -> default rule)."""
    if kappa is None:
        kappa = default_kappa(values, beta)
    return float(kappa)


def run(v, beta, rank, algorithm="jmm", *, kappa=None, tol=1e-5,
        max_outer_iters=5000, seed=0, sub_iters=1, sub_iters_w=None,
        sub_iters_h=None, heuristic_gamma_one=False, floor=DEFAULT_FLOOR,
        init=None, kkt=True):
    """solver.py:224-326 -- run_bmm / run_jmm + _outer_loop.

    ``init`` replaces ``init_factors`` (the reference resolves that global at
    solver.py:293, which is how the golden fixtures inject it).  Returns
    ``(w, h, objectives, kkts, termination)``.
    """
    v0 = np.asarray(v, dtype=float)
    kappa = resolve_kappa(v0, beta, kappa)
    vs = v0 + kappa if kappa != 0.0 else v0
    gamma = 1.0 if heuristic_gamma_one else gamma_exponent(beta)
    if init is None:
        w, h = init_factors(vs.shape[0], vs.shape[1], rank, seed)
    else:
        w, h = (np.array(init[0], dtype=float), np.array(init[1], dtype=float))
    objs, kkts = [], []
    prev = None
    term = "max-iters"
    for _ in range(max_outer_iters):
        if algorithm == "bmm":
            for _ in range(sub_iters_w or sub_iters):
                w = bmm_update_w(vs, w, h, beta, kappa, gamma, floor)
            for _ in range(sub_iters_h or sub_iters):
                h = bmm_update_h(vs, w, h, beta, kappa, gamma, floor)
        else:
            wt, ht = w, h
            prod = wt @ ht
            if kappa:
                prod = prod + kappa
            bases = joint_bases(vs, prod, beta)
            for _ in range(sub_iters):
                w = jmm_update_w(bases, wt, ht, h, beta, gamma, floor)
                h = jmm_update_h(bases, wt, ht, w, beta, gamma, floor)
        p = w @ h
        if kappa:
            p += kappa
        obj = divergence_total(vs, p, beta)
        stop = prev is not None and should_stop(prev, obj, tol)
        w, h = normalize_arrays(w, h)
        kkts.append(kkt_residuals_arrays(vs, w, h, beta, kappa) if kkt
                    else (float("nan"), float("nan")))
        objs.append(obj)
        prev = obj
        if stop:
            term = "converged"
            break
    return w, h, np.array(objs), np.array(kkts), term


# ----------------------------------------------------------------------------
# Sparse KL (beta = 1) restatement.  The reference densifies sparse input
# (matrixio.py:115-128) and cannot ingest config 5; this follows exactly the
# dense beta=1 formulas at updates.py:301-303 (W), :325-327 (H), the loop order
# of solver.py:292-326 and xlogy at core.py:101, with kappa = 0.


def run_sparse_kl(csr, rank, algorithm="jmm", *, max_outer_iters=10, tol=1e-300,
                  init=None, seed=0, floor=DEFAULT_FLOOR):
    import scipy.sparse as sp

    v = sp.csr_matrix(csr, dtype=float)
    v.sort_indices()
    if init is None:
        w, h = init_factors(v.shape[0], v.shape[1], rank, seed)
    else:
        w, h = (np.array(init[0], dtype=float), np.array(init[1], dtype=float))
    rows = np.repeat(np.arange(v.shape[0]), np.diff(v.indptr))
    cols = v.indices
    x = v.data

    def sddmm(wm, hm):
        return np.einsum("ik,ki->i", wm[rows], hm[:, cols])

    def zmat(vals):
        return sp.csr_matrix((vals, cols, v.indptr), shape=v.shape)

    objs = []
    prev = None
    term = "max-iters"
    for _ in range(max_outer_iters):
        if algorithm == "bmm":
            z = zmat(x / sddmm(w, h))
            w = w * guarded_divide(np.asarray(z @ h.T), h.sum(axis=1)[None, :], floor)
            z = zmat(x / sddmm(w, h))
            h = h * guarded_divide(np.asarray((z.T @ w).T), w.sum(axis=0)[:, None], floor)
        else:
            wt, ht = w, h
            z = zmat(x / sddmm(wt, ht))
            w = wt * guarded_divide(np.asarray(z @ ht.T), ht.sum(axis=1)[None, :], floor)
            h = ht * guarded_divide(np.asarray((z.T @ wt).T), w.sum(axis=0)[:, None], floor)
        y = sddmm(w, h)
        # sum_fn d_1 = sum_nnz [x log(x/y) - x] + sum_all y, sum_all y = (1'W)(H1)
        obj = float(np.sum(x * np.log(x / y) - x) + w.sum(axis=0) @ h.sum(axis=1))
        stop = prev is not None and should_stop(prev, obj, tol)
        w, h = normalize_arrays(w, h)
        objs.append(obj)
        prev = obj
        if stop:
            term = "converged"
            break
    return w, h, np.array(objs), term
