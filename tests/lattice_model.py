"""Pure-numpy model of the lattice engine's data layout (test helper).

Mirrors csrc/lattice.cu step by step -- table index of a subset, the
phase-1 elimination order (fixed prefix, expanded prefix, lane bits, leaf
bits), the phase-2 stencil and the lexicographic run placement -- so the
layout arithmetic is checked on the CPU against the oracle.
"""

import math
from itertools import combinations

import numpy as np

CB = 10


def table_logdets(r: np.ndarray) -> np.ndarray:
    """T[idx] = log det R_S with idx = (prefix bits << CB) | suffix bits."""
    n = r.shape[0]
    np_ = n - CB
    t = np.empty(1 << n)
    for blk in range(1 << np_):
        pre = [j for j in range(np_) if (blk >> j) & 1]
        for q in range(1 << CB):
            suf = [np_ + b for b in range(CB) if (q >> b) & 1]
            s = pre + suf
            t[(blk << CB) | q] = np.linalg.slogdet(r[np.ix_(s, s)])[1] if s else 0.0
    return t


def lexrank(n, s):
    k = len(s)
    rank = math.comb(n, k) - 1
    for i, v in enumerate(s):
        rank -= math.comb(n - 1 - v, k - i)
    return rank


def measures_full(r: np.ndarray, lo: int, hi: int):
    n = r.shape[0]
    np_ = n - CB
    t = table_logdets(r)
    offs, acc = {}, 0
    for k in range(lo, hi + 1):
        offs[k] = acc
        acc += math.comb(n, k)
    out = np.full((4, acc), np.nan)
    runs = {q: sorted([sum(1 << b for b in c) for c in combinations(range(CB), q)],
                      key=lambda m: [b for b in range(CB) if (m >> b) & 1])
            for q in range(CB + 1)}
    for blk in range(1 << np_):
        kp = bin(blk).count("1")
        own = t[blk << CB:(blk + 1) << CB]
        acc_nb = np.zeros(1 << CB)
        for j in range(np_):
            if (blk >> j) & 1:
                acc_nb += t[(blk ^ (1 << j)) << CB:((blk ^ (1 << j)) + 1) << CB]
        nbs = acc_nb.copy()
        for e in range(1 << CB):
            for b in range(CB):
                if (e >> b) & 1:
                    nbs[e] += own[e ^ (1 << b)]
        pre = [j for j in range(np_) if (blk >> j) & 1]
        for q in range(CB + 1):
            k = kp + q
            if k < lo or k > hi or k < 1:
                continue
            base = offs[k] + lexrank(n, pre + [np_ + i for i in range(q)])
            for i, e in enumerate(runs[q]):
                l, nb = own[e], nbs[e]
                tc = -0.5 * l
                dtc = 0.5 * ((1 - k) * l + nb)
                o = 0.5 * ((k - 2) * l - nb)
                out[:, base + i] = (tc, dtc, o, tc + dtc)
    return out
