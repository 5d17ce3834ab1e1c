"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

The paper's datasets (Olivetti, a spectrogram, TasteProfile, Moffett AVIRIS;
PAPER.md:853-1058) are not available, so each BASELINE.json config is
generated here with the shapes, ranks and value distributions it names.
Every generator is a pure function of ``(shape, seed)``; wide matrices are
produced in fixed column chunks with per-chunk seeds, so any column prefix of a
config is bitwise identical to the prefix of the full matrix (the oracle runs
on such prefixes).

``uniform_init`` is the "W and H initialised Uniform(0,1) from a seed" rule of
the configs; the reference itself draws half-normal factors
(solver.py:137-153, reproduced by :func:`paper_2106_15214_b200.init_factors`).
"""

from __future__ import annotations

import concurrent.futures as _cf
import os

import numpy as np

CHUNK = 1 << 16

#: name -> (F, N, K, beta, dtype, iterations) exactly as BASELINE.json states
CONFIGS = {
    1: dict(F=361, N=2429, K=49, beta=1.0, dtype="fp64", iters=200),
    2: dict(F=1024, N=8192, K=32, beta=2.0, dtype="fp32", iters=500),
    3: dict(F=1025, N=16384, K=20, beta=0.0, dtype="fp32", iters=300),
    4: dict(F=256, N=4194304, K=12, beta=1.5, dtype="fp32", iters=100),
    5: dict(F=1000000, N=200000, K=64, beta=1.0, dtype="fp32", iters=100,
            density=5e-4),
}


def uniform_init(F, N, K, seed):
    """W (F x K) then H (K x N) ~ Uniform(0,1), exact zeros redrawn."""
    rng = np.random.default_rng(seed)

    def draw(shape):
        m = rng.random(shape)
        while (m == 0.0).any():
            z = m == 0.0
            m[z] = rng.random(int(z.sum()))
        return m

    w = draw((F, K))
    return w, draw((K, N))


def config1(F=361, N=2429, K=49, seed=1):
    """Dense KL: V = W0 H0 + |N(0, 0.01)|, W0, H0 ~ Gamma(1,1), clip >= 1e-9."""
    rng = np.random.default_rng(seed)
    w0 = rng.gamma(1.0, 1.0, size=(F, K))
    h0 = rng.gamma(1.0, 1.0, size=(K, N))
    v = w0 @ h0 + np.abs(rng.normal(0.0, 0.01, size=(F, N)))
    return np.maximum(v, 1e-9)


def config2(F=1024, N=8192, K=32, seed=2):
    """Quadratic loss: exact rank-K V = W0 H0, W0, H0 ~ U(0,1)."""
    rng = np.random.default_rng(seed)
    w0 = rng.random((F, K))
    h0 = rng.random((K, N))
    return w0 @ h0


def config3(F=1025, N=16384, K=20, seed=3):
    """Itakura-Saito: V = (W0 H0) * E, W0 ~ Gamma(0.5,1) / f, H0 ~ Gamma(0.5,1),
    E ~ Exponential(1) (a spectrogram-like stand-in)."""
    rng = np.random.default_rng(seed)
    w0 = rng.gamma(0.5, 1.0, size=(F, K)) / np.arange(1, F + 1, dtype=float)[:, None]
    h0 = rng.gamma(0.5, 1.0, size=(K, N))
    e = rng.exponential(1.0, size=(F, N))
    return (w0 @ h0) * e


def _config4_chunk(endm, seed, c, n, dtype):
    rng = np.random.default_rng([seed, c])
    mix = rng.dirichlet(np.full(endm.shape[1], 0.3), size=n).T  # K x n
    noise = np.abs(rng.normal(0.0, 0.005, size=(endm.shape[0], n)))
    return (endm @ mix + noise).astype(dtype)


def config4(F=256, N=4194304, K=12, seed=4, dtype=np.float64, threads=None,
            col_range=None, out=None):
    """beta=1.5 hyperspectral stand-in: columns are Dirichlet(0.3) mixtures of K
    Uniform(0,1) endmember spectra plus |N(0, 0.005)| noise.
    Generated in 65536-column chunks so every prefix is stable.  ``col_range``
    = (n0, n1) returns only those columns of the N-column matrix (n0 must be a
    chunk boundary), which is how each rank builds its own shard."""
    endm = np.random.default_rng([seed, 0xE0D]).random((F, K))
    n0, n1 = col_range if col_range is not None else (0, N)
    if n0 % CHUNK:
        raise ValueError("col_range must start on a 65536-column chunk boundary")
    if out is None:
        out = np.empty((F, n1 - n0), dtype=dtype)
    nchunks = (n1 - n0 + CHUNK - 1) // CHUNK
    c_first = n0 // CHUNK

    def work(i):
        c = c_first + i
        lo = c * CHUNK
        hi = min(n1, lo + CHUNK)
        # always draw the whole chunk so that every prefix / shard is stable
        out[:, lo - n0:hi - n0] = _config4_chunk(endm, seed, c, CHUNK, out.dtype)[:, :hi - lo]

    threads = threads or min(8, os.cpu_count() or 1)
    if nchunks == 1 or threads == 1:
        for c in range(nchunks):
            work(c)
    else:
        with _cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, range(nchunks)))
    return out


def _config5_rows(cdf, perm, counts, row_fill, seed, chunk_id):
    """Column ids of a chunk of rows: Zipf draws without replacement within a
    row (first occurrences in draw order, the row's fill column drawn first),
    each row's ids returned sorted.  Returns (per-row counts, flat columns)."""
    rng = np.random.default_rng([seed, 0xC5, chunk_id])
    nr = counts.size
    N = perm.size
    out = [None] * nr
    todo = np.arange(nr)
    mult = 2
    while todo.size:
        c = counts[todo]
        M = int(min(max(c.max() * mult + 16, 32), 64 * N))
        u = rng.random((todo.size, M))
        draws = perm[np.minimum(np.searchsorted(cdf, u), N - 1)]
        draws[:, 0] = row_fill[todo]
        idx = np.argsort(draws, axis=1, kind="stable")
        srt = np.take_along_axis(draws, idx, axis=1)
        first_s = np.ones_like(srt, dtype=bool)
        first_s[:, 1:] = srt[:, 1:] != srt[:, :-1]
        first = np.empty_like(first_s)
        np.put_along_axis(first, idx, first_s, axis=1)
        cum = np.cumsum(first, axis=1)
        ok = cum[:, -1] >= c
        keep = first & (cum <= c[:, None])
        keep_s = np.take_along_axis(keep, idx, axis=1)
        for i in np.nonzero(ok)[0]:
            out[todo[i]] = srt[i][keep_s[i]]
        todo = todo[~ok]
        mult *= 2
    return counts, np.concatenate(out) if out else np.zeros(0, dtype=np.int32)


def config5(F=1000000, N=200000, density=5e-4, seed=5, alpha=1.1, threads=None):
    """Sparse counts (CSR) with exactly round(density * F * N) nonzeros
    (10^8 at the BASELINE size).

    Per-row nonzero counts ~ Poisson(density * N), rescaled by seeded +-1
    steps to the exact total; column ids ~ Zipf(alpha) popularity over a
    seeded column permutation, drawn WITHOUT replacement within a row (a
    duplicate draw is skipped, so heavy columns saturate instead of merging
    entries away); every row holds its fill column and every column at least
    one entry (an all-zero row or column of V drives its factor row/column to
    exactly 0 under MU, which the reference rejects, majorizer.py:50-51);
    values Geometric(0.3)+1 stored as fp32.  Rows are generated in seeded
    chunks, so the result does not depend on the thread count.

    Returns (indptr int64, indices int32, data float32, (F, N))."""
    rng = np.random.default_rng(seed)
    target = int(min(max(round(density * F * N), max(F, N)), F * N))
    ranks = np.arange(1, N + 1, dtype=float)
    p = ranks ** (-alpha)
    cdf = np.cumsum(p / p.sum())
    perm = rng.permutation(N).astype(np.int32)
    counts = np.clip(rng.poisson(density * N, size=F), 1, N).astype(np.int64)
    diff = target - int(counts.sum())
    while diff != 0:
        step = np.bincount(rng.integers(0, F, size=abs(diff)), minlength=F)
        counts += np.minimum(step, N - counts) if diff > 0 else -np.minimum(step, counts - 1)
        diff = target - int(counts.sum())
    row_fill = perm[np.arange(F) % N]
    RCH = 16384
    chunks = [(a, min(F, a + RCH)) for a in range(0, F, RCH)]

    def work(ci):
        a, b = chunks[ci]
        return _config5_rows(cdf, perm, counts[a:b], row_fill[a:b], seed, ci)

    threads = threads or min(8, os.cpu_count() or 1)
    if len(chunks) == 1 or threads == 1:
        parts = [work(i) for i in range(len(chunks))]
    else:
        with _cf.ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(work, range(len(chunks))))
    cols = np.concatenate([q[1] for q in parts]).astype(np.int32)
    indptr = np.zeros(F + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    # columns left empty: one entry each, replacing an entry of a random row
    # whose column is held elsewhere too (nnz stays exact)
    ccount = np.bincount(cols, minlength=N)
    for j in np.nonzero(ccount == 0)[0]:
        while True:
            r = int(rng.integers(0, F))
            lo, hi = indptr[r], indptr[r + 1]
            cand = np.nonzero(ccount[cols[lo:hi]] >= 2)[0]
            if cand.size:
                pos = lo + int(cand[rng.integers(0, cand.size)])
                ccount[cols[pos]] -= 1
                cols[pos] = j
                ccount[j] += 1
                cols[lo:hi].sort()
                break
    vals = (rng.geometric(0.3, size=cols.size) + 1).astype(np.float32)
    return indptr, cols, vals, (F, N)
