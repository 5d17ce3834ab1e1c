"""Host-side value types and scalar rules of the reference ``betanmf.core``.

These are the validation and bookkeeping pieces that run once per fit on the
host (domain checks, kappa resolution, gamma); the per-iteration arithmetic
runs in libbnmf.  Names, argument meaning and error behaviour follow
``/root/reference/pkg/src/betanmf/core.py`` (cited per item).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

#: core.py:18
DEFAULT_FLOOR = 1e-300


class DivergenceDomainError(ValueError):
    """(x, y) outside the domain of d_beta (core.py:21-26)."""


def gamma_exponent(beta):
    """Update exponent gamma(beta): 1/(2-b) below 1, 1 on [1,2], 1/(b-1) above
    (core.py:29-39)."""
    if beta < 1.0:
        return 1.0 / (2.0 - beta)
    if beta <= 2.0:
        return 1.0
    return 1.0 / (beta - 1.0)


def beta_divergence(x, y, beta):
    """Scalar d_beta(x | y) with the reference's domain errors (core.py:42-86)."""
    import math

    if not np.isfinite(x) or not np.isfinite(y):
        raise DivergenceDomainError("divergence arguments must be finite")
    if y <= 0.0:
        raise DivergenceDomainError(f"second argument must be positive, got {y}")
    if x < 0.0 or (x == 0.0 and beta <= 0.0):
        raise DivergenceDomainError(
            f"first argument must be {'positive' if beta <= 0 else 'nonnegative'} "
            f"for beta={beta}, got {x}; a positive data shift restores the domain")
    if x == y:
        return 0.0
    if beta == 2.0:
        return 0.5 * (x - y) ** 2
    if beta == 1.0:
        return (x * math.log(x / y) if x > 0.0 else 0.0) - x + y
    if beta == 0.0:
        r = x / y
        return r - math.log(r) - 1.0
    return (x ** beta / (beta * (beta - 1.0)) + y ** beta / beta
            - x * y ** (beta - 1.0) / (beta - 1.0))


def default_kappa(values, beta):
    """0 for beta in [1,2] on zero-free data, else 1e-9 * mean (core.py:176-185)."""
    values = np.asarray(values)
    if 1.0 <= beta <= 2.0 and float(values.min()) > 0.0:
        return 0.0
    return 1e-9 * float(values.mean(dtype=np.float64))


@dataclass
class DataMatrix:
    """Dense nonnegative data with an optional shift (core.py:188-228)."""

    values: np.ndarray
    kappa: float = 0.0

    def __post_init__(self):
        v = np.asarray(self.values)
        if v.dtype not in (np.float64, np.float32):
            v = v.astype(np.float64)
        self.values = v
        if self.values.ndim != 2 or min(self.values.shape) < 1:
            raise ValueError("data must be a 2-D matrix with positive dimensions")
        if not np.isfinite(self.values).all():
            raise ValueError("data entries must be finite")
        if self.values.min() < 0.0:
            raise ValueError("data entries must be nonnegative")
        self.kappa = float(self.kappa)
        if not np.isfinite(self.kappa) or self.kappa < 0.0:
            raise ValueError("kappa must be a nonnegative finite real")

    @property
    def shape(self):
        return self.values.shape

    def shifted(self):
        if self.kappa == 0.0:
            return self.values
        return self.values + self.kappa

    def check_domain(self, beta):
        if beta < 1.0 and self.kappa == 0.0 and self.values.min() == 0.0:
            raise DivergenceDomainError(
                f"data contains zeros, which is outside the domain of "
                f"d_beta for beta={beta}; set a positive kappa shift")


@dataclass
class FactorPair:
    """Strictly positive factors w (F x K) and h (K x N) (core.py:231-260)."""

    w: np.ndarray
    h: np.ndarray

    def __post_init__(self):
        self.w = np.asarray(self.w, dtype=float)
        self.h = np.asarray(self.h, dtype=float)
        if self.w.ndim != 2 or self.h.ndim != 2:
            raise ValueError("factors must be 2-D matrices")
        if self.w.shape[1] != self.h.shape[0]:
            raise ValueError(
                f"inner dimensions disagree: w is {self.w.shape}, h is {self.h.shape}")
        if not (np.isfinite(self.w).all() and np.isfinite(self.h).all()):
            raise ValueError("factor entries must be finite")
        if self.w.min() <= 0.0 or self.h.min() <= 0.0:
            raise ValueError("factor entries must be strictly positive")

    @property
    def rank(self):
        return self.w.shape[1]

    def product(self, kappa=0.0):
        p = self.w @ self.h
        if kappa:
            p += kappa
        return p


@dataclass
class BetaParam:
    """beta with its derived exponent (core.py:263-272)."""

    beta: float
    gamma: float = field(init=False)

    def __post_init__(self):
        self.beta = float(self.beta)
        self.gamma = gamma_exponent(self.beta)
