"""CPU oracle for the n-plet HOI hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's hot
path (``/root/reference/pkg/src/hoi``; cited below as ``ref:<file>:<line>``).
It exists for three consumers and no others:

* ``tests/`` -- the parity checker for the CUDA path (and it is itself
  pinned against golden vectors produced by the real reference, see
  ``tests/golden/make_golden.py`` and ``tests/test_oracle_golden.py``);
* ``__graft_entry__.smoke()`` -- a one-shot cross-check;
* ``bench.py --impl reference`` / the ``cpu_baseline`` leg -- the CPU
  baseline timing (the reference is pure Python, it cannot travel to the
  GPU box, so this restatement of its algorithm is what is timed there).

The product package (``paper_2501_03381_b200``) never imports this file.
The restatement deliberately keeps the reference's numerical route
(LAPACK Cholesky + LU inverse per sub-matrix, numpy batching, a bounded
thread pool with ordered reduction) so that its timing is representative
of the reference's CPU cost.
"""

from __future__ import annotations

import itertools
import math
from collections import deque
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.special import ndtri, psi

LOG_2PI_E = float(np.log(2.0 * np.pi) + 1.0)       # ref:copula_core.py:22
H1 = 0.5 * LOG_2PI_E                                 # ref:copula_core.py:25
MEASURES = ("tc", "dtc", "o", "s")                   # ref:scanner.py:25


class OracleError(Exception):
    pass


class OracleNotPD(OracleError):
    def __init__(self, msg, coords=None):
        super().__init__(msg)
        self.coords = coords


# --------------------------------------------------------------------------
# data -> copula -> covariance            (ref:copula_core.py:44-62,155-189)
# --------------------------------------------------------------------------

def check_data(x) -> np.ndarray:
    """Cast and validate a (T, N) data matrix (ref:copula_core.py:44-62)."""
    v = np.asarray(x, dtype=np.float64)
    if v.ndim != 2 or v.shape[1] < 1:
        raise OracleError("bad shape")
    if v.shape[0] < 3:
        raise OracleError("T < 3")
    if not np.isfinite(v).all():
        raise OracleError("non-finite")
    if (v.max(axis=0) == v.min(axis=0)).any():
        raise OracleError("constant column")
    return v


def ranks(x) -> np.ndarray:
    """Ordinal ranks 1..T per column, ties by row order (ref:copula_core.py:155-162).

    The reference calls ``scipy.stats.rankdata(method='ordinal')``; a stable
    argsort followed by inversion yields the identical permutation.
    """
    v = check_data(x)
    order = np.argsort(v, axis=0, kind="stable")
    out = np.empty(v.shape, dtype=np.int64)
    cols = np.arange(v.shape[1])[None, :]
    out[order, cols] = np.arange(1, v.shape[0] + 1)[:, None]
    return out


def copula(x) -> np.ndarray:
    """Phi^-1(rank / (T + 1)) per column (ref:copula_core.py:165-174)."""
    v = check_data(x)
    return ndtri(ranks(v) / (v.shape[0] + 1.0))


def covariance(z) -> np.ndarray:
    """Centred X^T X / (T-1), symmetrised (ref:copula_core.py:177-189)."""
    z = check_data(z)
    t = z.shape[0]
    xc = z - z.mean(axis=0)
    s = (xc.T @ xc) / (t - 1)
    return 0.5 * (s + s.T)


def entropy_bias(n: int, t: int) -> float:
    """eta(n, T) (ref:copula_core.py:219-231)."""
    j = np.arange(1, n + 1)
    return float(0.5 * (n * np.log(2.0 / (t - 1)) + psi((t - j) / 2.0).sum()))


def bias_table(t: int, k_max: int) -> np.ndarray:
    """eta(k, T) for k = 0..k_max with the reference's cumsum route
    (ref:copula_core.py:234-244)."""
    if t <= k_max:
        raise OracleError("T <= k_max")
    eta = np.zeros(k_max + 1)
    if k_max >= 1:
        j = np.arange(1, k_max + 1)
        eta[1:] = 0.5 * (j * np.log(2.0 / (t - 1)) + np.cumsum(psi((t - j) / 2.0)))
    return eta


# --------------------------------------------------------------------------
# enumeration                              (ref:nplet_engine.py:26-33,118-136)
# --------------------------------------------------------------------------

def count(n: int, lo: int, hi: int) -> int:
    return sum(math.comb(n, k) for k in range(lo, hi + 1))


def order_batches(n: int, k: int, batch_size: int):
    """Lexicographic k-subsets in chunks of <= batch_size rows
    (ref:nplet_engine.py:118-136)."""
    it = itertools.combinations(range(n), k)
    while True:
        flat = np.fromiter(itertools.chain.from_iterable(itertools.islice(it, batch_size)),
                           dtype=np.int64)
        if flat.size == 0:
            return
        yield flat.reshape(-1, k)


def all_rows(n: int, lo: int, hi: int) -> list:
    """Every n-plet, order-major then lexicographic (ref:scanner.py:345-347)."""
    return [c for k in range(lo, hi + 1) for c in itertools.combinations(range(n), k)]


# --------------------------------------------------------------------------
# batched log-determinant / inverse diagonal     (ref:nplet_engine.py:227-281)
# --------------------------------------------------------------------------

def _one(m):
    try:
        c = np.linalg.cholesky(m)
        inv = np.linalg.inv(m)
    except np.linalg.LinAlgError:
        return None
    return 2.0 * np.log(np.diagonal(c)).sum(), np.diagonal(inv).copy()


def logdet_invdiag(mats: np.ndarray):
    """(logdet, invdiag) of a (..., K, K) stack; per-matrix jitter retry
    eps = 1e-10 trace/K only for the failing ones (ref:nplet_engine.py:237-281)."""
    try:
        c = np.linalg.cholesky(mats)
        inv = np.linalg.inv(mats)
        return (2.0 * np.log(np.diagonal(c, axis1=-2, axis2=-1)).sum(axis=-1),
                np.diagonal(inv, axis1=-2, axis2=-1))
    except np.linalg.LinAlgError:
        pass
    lead, k = mats.shape[:-2], mats.shape[-1]
    ld = np.empty(lead)
    idg = np.empty(lead + (k,))
    bad = []
    for co in np.ndindex(lead):
        m = mats[co]
        r = _one(m)
        if r is None:
            r = _one(m + (1e-10 * np.trace(m) / k) * np.eye(k))
        if r is None:
            bad.append(co)
            continue
        ld[co], idg[co] = r
    if bad:
        raise OracleNotPD("not positive definite after jitter", coords=bad)
    return ld, idg


# --------------------------------------------------------------------------
# entropy terms and measures      (ref:nplet_engine.py:284-351, measures.py:41-81)
# --------------------------------------------------------------------------

def _tables(t_used, k_max):
    t_used = np.asarray(t_used)
    if (t_used <= 0).any():
        raise OracleError("bias needs sample counts")
    return np.stack([bias_table(int(t), k_max) for t in t_used])


def terms_fixed(sig, t_used, idx, bias=False):
    """Excess terms for a fixed-order batch: (x_joint (B,D), x_singles (B,D,K),
    x_loo (B,D,K)) (ref:nplet_engine.py:305-330)."""
    idx = np.asarray(idx, dtype=np.int64)
    k = idx.shape[1]
    xs_all = 0.5 * np.log(np.diagonal(sig, axis1=-2, axis2=-1))       # (D, N)
    if bias:
        tab = _tables(t_used, k)
        xs_all = xs_all - tab[:, 1][:, None]
    d_ax = np.arange(sig.shape[0])[None, :, None, None]
    sub = sig[d_ax, idx[:, None, :, None], idx[:, None, None, :]]     # (B, D, K, K)
    ld, idg = logdet_invdiag(sub)
    xj = 0.5 * ld
    xl = 0.5 * (ld[..., None] + np.log(idg))
    xs = xs_all[:, idx].transpose(1, 0, 2)
    if bias:
        xj = xj - tab[:, k][None, :]
        xl = xl - tab[:, k - 1][None, :, None]
    return xj, xs, xl


def terms_mixed(sig, t_used, masks, bias=False):
    """Excess terms for an identity-padded mixed-order batch
    (ref:nplet_engine.py:204-224,332-351)."""
    masks = np.asarray(masks, dtype=bool)
    n = sig.shape[-1]
    orders = masks.sum(axis=1).astype(np.int64)
    xs_all = 0.5 * np.log(np.diagonal(sig, axis1=-2, axis2=-1))
    if bias:
        tab = _tables(t_used, int(orders.max()))
        xs_all = xs_all - tab[:, 1][:, None]
    keep = masks[:, None, :, None] & masks[:, None, None, :]
    mats = np.where(keep, sig[None], np.eye(n))
    ld, idg = logdet_invdiag(mats)
    xj = 0.5 * ld
    xl = 0.5 * (ld[..., None] + np.log(idg))
    in_set = masks[:, None, :]
    if bias:
        xj = xj - tab[:, orders].T
        xl = xl - tab[:, orders - 1].T[..., None]
    xs = np.where(in_set, xs_all[None], 0.0)
    xl = np.where(in_set, xl, 0.0)
    return xj, xs, xl, orders


def measures(xj, xs, xl, orders):
    """tc, dtc, o (expanded form), s = tc + dtc (ref:measures.py:41-81)."""
    k = np.asarray(orders, dtype=np.float64)[:, None]
    tc = xs.sum(axis=-1) - xj
    dtc = (1.0 - k) * xj + xl.sum(axis=-1)
    o = (k - 2.0) * xj + (xs - xl).sum(axis=-1)
    return tc, dtc, o, tc + dtc


def hoi_batch(sig, t_used, idx=None, masks=None, bias=False):
    """All four measures (B, D) for one batch (ref:measures.py:72-81)."""
    sig = np.asarray(sig, dtype=np.float64)
    if sig.ndim == 2:
        sig = sig[None]
    if idx is not None:
        idx = np.asarray(idx, dtype=np.int64)
        xj, xs, xl = terms_fixed(sig, t_used, idx, bias)
        orders = np.full(idx.shape[0], idx.shape[1], dtype=np.int64)
    else:
        xj, xs, xl, orders = terms_mixed(sig, t_used, masks, bias)
    return measures(xj, xs, xl, orders) + (orders,)


# --------------------------------------------------------------------------
# scan driver and reducers                        (ref:scanner.py:27-365)
# --------------------------------------------------------------------------

class TopKR:
    """Per-dataset best-k by (sign*value, index tuple) (ref:scanner.py:50-105)."""

    def __init__(self, measure, direction, k):
        self.m, self.sign, self.k = MEASURES.index(measure), (-1.0 if direction == "max" else 1.0), k
        self.best = None

    def update(self, idx, vals):          # vals: (4, B, D)
        v = vals[self.m]
        b, dd = v.shape
        if self.best is None:
            self.best = [[] for _ in range(dd)]
        ke = min(self.k, b)
        for d in range(dd):
            col = self.sign * v[:, d]
            thr = np.partition(col, ke - 1)[ke - 1]
            for i in np.flatnonzero(col <= thr):
                tup = tuple(int(x) for x in idx[i])
                self.best[d].append(((float(col[i]), tup),
                                     (tup, float(v[i, d])) + tuple(float(vals[m][i, d]) for m in range(4))))
            self.best[d].sort(key=lambda p: p[0])
            del self.best[d][self.k:]

    def finalize(self):
        # list over datasets of (indices, value, tc, dtc, o, s)
        return [] if self.best is None else [[e for _, e in per] for per in self.best]


class HistR:
    """Clipped fixed-range histogram per dataset (ref:scanner.py:108-137)."""

    def __init__(self, measure, bins, lo, hi):
        self.m = MEASURES.index(measure)
        self.edges = np.linspace(lo, hi, bins + 1)
        self.counts = None

    def update(self, idx, vals):
        v = vals[self.m]
        if self.counts is None:
            self.counts = np.zeros((v.shape[1], len(self.edges) - 1), dtype=np.int64)
        for d in range(v.shape[1]):
            self.counts[d] += np.histogram(np.clip(v[:, d], self.edges[0], self.edges[-1]),
                                           bins=self.edges)[0]

    def finalize(self):
        return self.edges, self.counts


class CollectR:
    """Collects every row in enumeration order (a Callback that keeps all)."""

    def __init__(self):
        self.rows, self.vals = [], []

    def update(self, idx, vals):
        self.rows.append(idx)
        self.vals.append(vals)

    def finalize(self):
        return self.rows, np.concatenate(self.vals, axis=1)


class FeaturesR:
    """21-feature fingerprint accumulator (ref:scanner.py:205-287)."""

    def __init__(self, n):
        self.n = n
        self.st = None

    def update(self, idx, vals):
        v = np.stack(vals, axis=-1)                     # (B, D, 4)
        dd = v.shape[1]
        k = idx.shape[1]
        if self.st is None:
            self.st = dict(sum=np.zeros((dd, 4)), mx=np.full((dd, 4), -np.inf),
                           mn=np.full((dd, 4), np.inf), cnt=0, omax=np.zeros(dd, np.int64),
                           omin=np.zeros(dd, np.int64), syn=np.zeros(dd, np.int64),
                           mis=np.zeros(dd), mis2=np.zeros(dd), micnt=0,
                           whole=np.full((dd, 4), np.nan))
        s = self.st
        if k == 2:
            mi = vals[0]
            s["mis"] += mi.sum(axis=0)
            s["mis2"] += (mi * mi).sum(axis=0)
            s["micnt"] += mi.shape[0]
        if k >= 3:
            o = vals[2]
            for d in range(dd):
                i = int(np.argmax(o[:, d]))
                if o[i, d] > s["mx"][d, 2]:
                    s["omax"][d] = k
                i = int(np.argmin(o[:, d]))
                if o[i, d] < s["mn"][d, 2]:
                    s["omin"][d] = k
            np.maximum(s["mx"], v.max(axis=0), out=s["mx"])
            np.minimum(s["mn"], v.min(axis=0), out=s["mn"])
            s["sum"] += v.sum(axis=0)
            s["cnt"] += v.shape[0]
            s["syn"] += (o < 0.0).sum(axis=0)
            if k == self.n:
                s["whole"] = v[0]

    def finalize(self):
        s = self.st
        out = []
        for d in range(s["sum"].shape[0]):
            mean = s["sum"][d] / s["cnt"]
            mim = s["mis"][d] / s["micnt"]
            var = max(s["mis2"][d] / s["micnt"] - mim * mim, 0.0)
            f = {}
            for i, m in enumerate(MEASURES):
                f[m + "_max"] = float(s["mx"][d, i])
                f[m + "_min"] = float(s["mn"][d, i])
                f[m + "_mean"] = float(mean[i])
                f[m + "_whole"] = float(s["whole"][d, i])
            f["mi_mean"] = float(mim)
            f["mi_std"] = float(np.sqrt(var))
            f["o_max_order_norm"] = float(s["omax"][d] / self.n)
            f["o_min_order_norm"] = float(s["omin"][d] / self.n)
            f["prop_synergistic"] = float(s["syn"][d] / s["cnt"])
            out.append(f)
        return out


def _ordered(fn, items, workers):
    """Bounded thread pool yielding in input order (ref:scanner.py:290-305)."""
    if workers <= 1:
        for it in items:
            yield fn(it)
        return
    items = iter(items)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        q = deque(pool.submit(fn, it) for it in itertools.islice(items, workers + 2))
        while q:
            f = q.popleft()
            for it in itertools.islice(items, 1):
                q.append(pool.submit(fn, it))
            yield f.result()


def scan(sig, t_used, lo, hi, reducer, batch_size=10000, bias=False, workers=1,
         batches=None):
    """Order-major lexicographic exhaustive scan (ref:scanner.py:308-365).

    ``batches`` optionally overrides the batch stream (used by the bounded
    CPU-baseline samples)."""
    sig = np.asarray(sig, dtype=np.float64)
    if sig.ndim == 2:
        sig = sig[None]
    n = sig.shape[-1]
    if batches is None:
        batches = itertools.chain.from_iterable(order_batches(n, k, batch_size)
                                                for k in range(lo, hi + 1))

    def score(idx):
        tc, dtc, o, s, _ = hoi_batch(sig, t_used, idx=idx, bias=bias)
        return idx, (tc, dtc, o, s)

    for idx, vals in _ordered(score, batches, workers):
        reducer.update(idx, vals)
    return reducer.finalize()


# --------------------------------------------------------------------------
# analytic fixtures used by the tests          (ref:synthetic.py:23-86)
# --------------------------------------------------------------------------

def r_system(m, c):
    s = np.full((m + 1, m + 1), c * c)
    np.fill_diagonal(s, c * c + 1.0)
    s[m, :] = c
    s[:, m] = c
    s[m, m] = 1.0
    return s


def s_system(m, c):
    s = np.eye(m + 1)
    s[m, :m] = c
    s[:m, m] = c
    s[m, m] = m * c * c + 1.0
    return s


def block_diag(blocks):
    n = sum(b.shape[0] for b in blocks)
    out = np.zeros((n, n))
    at = 0
    for b in blocks:
        out[at:at + b.shape[0], at:at + b.shape[0]] = b
        at += b.shape[0]
    return out


def sample_gaussian(sigma, t, seed):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((t, sigma.shape[0]))
    return z @ np.linalg.cholesky(sigma).T
