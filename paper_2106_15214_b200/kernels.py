"""Device-backed versions of the reference's lower-level public kernels.

Same names, arguments and checks as the reference (file:line under
/root/reference/pkg/src/betanmf):

    objective(data, factors, beta)                         core.py:275-306
    kkt_residuals(data, factors, beta) -> KktResiduals     diagnostics.py:62-90
    bmm_update_w / bmm_update_h(v, w, h, beta, ...)        updates.py:157-181
    jmm_update_w / jmm_update_h(v, anchor, cur, beta, ...) updates.py:203-235
    MajorizerAnchor(.from_factors)                         majorizer.py:29-73

Every function uploads its operands, runs the corresponding libbnmf kernels
(include/bnmf.h: bnmf_kernel -- the reference-order SIMT kernels of
csrc/simt_kernels.cuh) and returns numpy fp64, so the reference's `verify`
suites and tests can run against the device.  The F x N model product is never
materialised: :class:`MajorizerAnchor` here holds the anchor factors and the
shift only (``product`` is formed on the host on demand, for callers that read it).

Keyword-only extensions: ``dtype`` ("fp64" default, "fp32") and ``device``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import DEFAULT_FLOOR, DataMatrix, DivergenceDomainError, FactorPair, gamma_exponent


@dataclass
class KktResiduals:
    """Normalized first-order residuals for the two factors (diagnostics.py:26-31)."""

    res_w: float
    res_h: float


class MajorizerAnchor:
    """Frozen factors of a joint outer iteration (majorizer.py:29-73).  The cached product of
    the reference stays implicit on the device; ``product`` materialises it on the host."""

    def __init__(self, w, h, product=None, kappa=0.0):
        self.w = np.asarray(w, dtype=float)
        self.h = np.asarray(h, dtype=float)
        self.kappa = float(kappa)
        self._product = product
        if self.w.shape[1] != self.h.shape[0]:
            raise ValueError("anchor factor dimensions disagree")
        if product is not None and product.shape != (self.w.shape[0], self.h.shape[1]):
            raise ValueError("cached product has the wrong shape")
        if self.w.min() <= 0.0 or self.h.min() <= 0.0:
            raise ValueError("anchor factors must be strictly positive")

    @classmethod
    def from_factors(cls, w, h, kappa=0.0, counter=None):
        if counter is not None:
            counter.anchor_products += 1
        return cls(w, h, None, kappa)

    @property
    def product(self):
        if self._product is None:
            self._product = self.w @ self.h + self.kappa
        return self._product

    def validate(self, rtol=1e-12):
        if self.product.min() <= 0.0:
            raise ValueError("anchor product must be strictly positive")
        fresh = self.w @ self.h + self.kappa
        err = np.max(np.abs(self.product - fresh) / np.maximum(np.abs(fresh), 1e-300))
        if err > rtol:
            raise ValueError(f"cached product is stale (relative error {err:.3e})")


def _params(beta, gamma, kappa, floor):
    p = _native.Params()
    p.algorithm = _native.BNMF_JMM
    p.sub_iters = 1
    p.sub_iters_w = p.sub_iters_h = 0
    p.beta = float(beta)
    p.gamma = gamma_exponent(beta) if gamma is None else float(gamma)
    p.kappa = float(kappa)
    p.floor = float(floor)
    p.tol = 0.0
    p.compute_kkt = 0
    p.schedule = _native.SCHED["reference"]
    return p


def _run(op, shifted, w, h, beta, *, kappa=0.0, gamma=None, floor=DEFAULT_FLOOR, cur=None,
         dtype="fp64", device=None):
    from .solver import get_context
    ctx = get_context(device, dtype)
    with ctx.lock:
        ctx.set_dense(np.asarray(shifted), 0.0)     # already V + kappa
        ctx.set_factors(w, h)
        return ctx.kernel(op, _params(beta, gamma, kappa, floor), cur)


def _as_data(data):
    return data if isinstance(data, DataMatrix) else DataMatrix(np.asarray(data, dtype=float))


def _check_model(data, factors):
    if data.shape != (factors.w.shape[0], factors.h.shape[1]):
        raise ValueError(f"dimension mismatch: data is {data.shape}, "
                         f"model is {(factors.w.shape[0], factors.h.shape[1])}")


def objective(data, factors, beta, *, dtype="fp64", device=None):
    """D_beta(V + kappa | W H + kappa) summed over all entries (core.py:275-306)."""
    data = _as_data(data)
    _check_model(data, factors)
    x = data.shifted()
    if beta <= 0.0 and x.min() <= 0.0:
        raise DivergenceDomainError(
            f"data entries must be positive for beta={beta}; set a positive kappa shift")
    if data.kappa <= 0.0 and (factors.w.min() <= 0.0 or factors.h.min() <= 0.0):
        raise DivergenceDomainError("model product has nonpositive entries")
    return _run(_native.OP_OBJECTIVE, x, factors.w, factors.h, beta, kappa=data.kappa,
                dtype=dtype, device=device)


def kkt_residuals(data, factors, beta, *, dtype="fp64", device=None):
    """First-order optimality residuals of a factor pair (diagnostics.py:62-90)."""
    data = _as_data(data)
    _check_model(data, factors)
    rw, rh = _run(_native.OP_KKT, data.shifted(), factors.w, factors.h, beta, kappa=data.kappa,
                  dtype=dtype, device=device)
    return KktResiduals(rw, rh)


def _count(counter, which, product):
    if counter is None:
        return
    if product:
        counter.kernel_products += 1
    if which == "w":
        counter.w_updates += 1
    else:
        counter.h_updates += 1


def bmm_update_w(v, w, h, beta, *, kappa=0.0, gamma=None, floor=DEFAULT_FLOOR, counter=None,
                 dtype="fp64", device=None):
    """One block update of the first factor; ``v`` is the already-shifted data
    (updates.py:157-170)."""
    _count(counter, "w", True)
    return _run(_native.OP_BMM_W, v, w, h, beta, kappa=kappa, gamma=gamma, floor=floor,
                dtype=dtype, device=device)


def bmm_update_h(v, w, h, beta, *, kappa=0.0, gamma=None, floor=DEFAULT_FLOOR, counter=None,
                 dtype="fp64", device=None):
    """One block update of the second factor (updates.py:173-181)."""
    _count(counter, "h", True)
    return _run(_native.OP_BMM_H, v, w, h, beta, kappa=kappa, gamma=gamma, floor=floor,
                dtype=dtype, device=device)


def jmm_update_w(v, anchor, h_current, beta, *, gamma=None, floor=DEFAULT_FLOOR, counter=None,
                 bases=None, dtype="fp64", device=None):
    """One joint update of the first factor against a frozen anchor (updates.py:203-220).
    ``bases`` (the host matrices of joint_bases) is accepted and ignored: the device forms the
    anchor-constant terms tile by tile."""
    _count(counter, "w", False)
    return _run(_native.OP_JMM_W, v, anchor.w, anchor.h, beta, kappa=anchor.kappa, gamma=gamma,
                floor=floor, cur=h_current, dtype=dtype, device=device)


def jmm_update_h(v, anchor, w_current, beta, *, gamma=None, floor=DEFAULT_FLOOR, counter=None,
                 bases=None, dtype="fp64", device=None):
    """One joint update of the second factor (updates.py:223-235)."""
    _count(counter, "h", False)
    return _run(_native.OP_JMM_H, v, anchor.w, anchor.h, beta, kappa=anchor.kappa, gamma=gamma,
                floor=floor, cur=w_current, dtype=dtype, device=device)
