"""Seeded synthetic inputs for the five BASELINE.json configurations.

There is no public dataset behind BASELINE.json; each configuration is a
seeded synthetic system with the shape, size and distribution the config
names.  Every generator is deterministic in its seed so
the oracle and the CUDA path always see identical bytes.
"""

from __future__ import annotations

import numpy as np


def randcorr(n: int, rng: np.random.Generator) -> np.ndarray:
    """A·Aᵀ rescaled to unit diagonal, A (n×n) i.i.d. N(0,1)."""
    a = rng.standard_normal((n, n))
    s = a @ a.T
    d = np.sqrt(np.diag(s))
    r = s / np.outer(d, d)
    np.fill_diagonal(r, 1.0)
    return r


def _draw(c: np.ndarray, t: int, rng: np.random.Generator) -> np.ndarray:
    # the reference's sample_gaussian recipe: z @ chol(C)^T
    return rng.standard_normal((t, c.shape[0])) @ np.linalg.cholesky(c).T


def cfg1(seed: int = 0):
    """N=10, T=1000, latent random correlation; orders 3..10, no bias."""
    rng = np.random.default_rng(seed)
    c = randcorr(10, rng)
    return _draw(c, 1000, rng)


def cfg2(seed: int = 0):
    """N=12, T=10,000: redundant block 0-3, product 'synergy' 4-6, 7-11 noise."""
    rng = np.random.default_rng(seed)
    t = 10_000
    z = rng.standard_normal(t)
    red = z[:, None] + 0.3 * rng.standard_normal((t, 4))
    x45 = rng.standard_normal((t, 2))
    x6 = x45[:, 0] * x45[:, 1] + 0.1 * rng.standard_normal(t)
    rest = rng.standard_normal((t, 5))
    return np.column_stack([red, x45, x6, rest])


def cfg3(seed: int = 0):
    """N=20, T=10,000 float32, 4 blocks of 5 (0.5 within, 0.05 between) + perturbation."""
    rng = np.random.default_rng(seed)
    b0 = np.full((20, 20), 0.05)
    for i in range(4):
        b0[5 * i:5 * i + 5, 5 * i:5 * i + 5] = 0.5
    np.fill_diagonal(b0, 1.0)
    c = 0.9 * b0 + 0.1 * randcorr(20, rng)
    return _draw(c, 10_000, rng).astype(np.float32)


def cfg4(seed: int = 0):
    """N=30, T=2000, Student-t(3) marginals through a Gaussian latent."""
    from scipy.special import ndtr
    from scipy.stats import t as student_t
    rng = np.random.default_rng(seed)
    c = randcorr(30, rng)
    z = _draw(c, 2000, rng)
    return student_t.ppf(ndtr(z), 3)


def cfg5_data(d: int, n: int = 400, t: int = 1200) -> np.ndarray:
    """One AR(1) (phi=0.6) dataset with 10-cluster block-correlated innovations."""
    rng = np.random.default_rng(1000 + d)
    c = np.zeros((n, n))
    size = n // 10
    for i in range(10):
        c[i * size:(i + 1) * size, i * size:(i + 1) * size] = 0.4
    np.fill_diagonal(c, 1.0)
    e = _draw(c, t, rng)
    x = np.empty_like(e)
    x[0] = e[0]
    for i in range(1, t):
        x[i] = 0.6 * x[i - 1] + np.sqrt(1.0 - 0.36) * e[i]
    return x


def cfg5_nplets(b: int = 4_000_000, n: int = 400, k: int = 10, seed: int = 123) -> np.ndarray:
    """B rows of k distinct indices, uniform without replacement within a row.

    Each row takes the first k distinct values of an i.i.d. uniform integer
    stream (a uniform ordered sample without replacement), then sorts them.
    """
    rng = np.random.default_rng(seed)
    out = np.empty((b, k), dtype=np.int64)
    step = 1 << 18
    for lo in range(0, b, step):
        m = min(step, b - lo)
        rows = np.empty((m, k), dtype=np.int64)
        todo = np.arange(m)
        w = k + 8
        earlier = np.tril(np.ones((w, w), dtype=bool), -1)       # q < p
        while todo.size:
            cand = rng.integers(0, n, size=(todo.size, w))
            dup = ((cand[:, :, None] == cand[:, None, :]) & earlier[None]).any(axis=2)
            first = ~dup                                          # first occurrence
            ok = first.sum(axis=1) >= k
            sel = first & (np.cumsum(first, axis=1) <= k)
            picked = cand[ok][sel[ok]].reshape(-1, k)
            rows[todo[ok]] = np.sort(picked, axis=1)
            todo = todo[~ok]
        out[lo:lo + m] = rows
    return out
