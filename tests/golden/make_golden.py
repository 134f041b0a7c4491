"""Generate golden vectors from the REAL reference package.

Run in the build container only (it imports /root/reference, which does
not exist on the GPU box):

    python tests/golden/make_golden.py

Everything it writes is a small .npz / .json fixture committed under
tests/golden/.  The fixtures pin the CPU oracle (tests/test_oracle_golden.py)
and are compared directly against the CUDA path (tests/test_gpu_parity.py).
Inputs come from paper_2501_03381_b200.workloads (seeded) or from small
literal matrices, so the GPU-side tests can regenerate identical bytes.
"""

import hashlib
import itertools
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, str(REPO))

import hoi  # noqa: E402  (the reference)
import reference as ref_slow  # noqa: E402  (the reference's own slow oracle)
from hoi.nplet_engine import _batched_logdet_invdiag  # noqa: E402

from paper_2501_03381_b200 import workloads  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def covset_of(x):
    return hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(hoi.DataMatrix(x)))])


def full_scan(covs, lo, hi, bias, batch_size=10000):
    vals = []

    def keep(batch, h):
        vals.append(np.stack([h.tc, h.dtc, h.o, h.s], axis=0))  # (4, B, D)

    hoi.scan(covs, lo, hi, hoi.Callback(keep), batch_size=batch_size, bias_correct=bias)
    return np.concatenate(vals, axis=1)


def unrank(n, lo, hi, g):
    """Reference-order n-plet at global rank g (by brute itertools walk)."""
    for k in range(lo, hi + 1):
        c = math.comb(n, k)
        if g < c:
            return next(itertools.islice(itertools.combinations(range(n), k), g, None))
        g -= c
    raise IndexError


def sampled_ranks(n, lo, hi, count, seed):
    total = hoi.count_nplets(n, lo, hi)
    rng = np.random.default_rng(seed)
    pick = set(rng.integers(0, total, size=count).tolist())
    off = 0
    for k in range(lo, hi + 1):
        c = math.comb(n, k)
        pick.update([off, off + c - 1])   # first and last of each order
        off += c
    return np.array(sorted(pick), dtype=np.int64)


def lex_rank(n, tup):
    k = len(tup)
    r, prev = 0, -1
    for p, s in enumerate(tup):
        for c in range(prev + 1, s):
            r += math.comb(n - 1 - c, k - 1 - p)
        prev = s
    return r


def sample_measures(covs, n, lo, hi, ranks, bias):
    tuples = []
    offs = {}
    off = 0
    for k in range(lo, hi + 1):
        offs[k] = off
        off += math.comb(n, k)
    # group by order for compute_hoi_batch; unrank with the combinatorial
    # number system and verify against itertools on a few
    out = np.empty((4, len(ranks), covs.n_datasets))
    idx_pad = np.full((len(ranks), hi), -1, dtype=np.int64)
    for i, g in enumerate(ranks):
        k = max(kk for kk in range(lo, hi + 1) if offs[kk] <= g)
        r = int(g - offs[k])
        tup, prev = [], -1
        for p in range(k):
            c = prev + 1
            while math.comb(n - 1 - c, k - 1 - p) <= r:
                r -= math.comb(n - 1 - c, k - 1 - p)
                c += 1
            tup.append(c)
            prev = c
        tuples.append(tuple(tup))
        idx_pad[i, :k] = tup
    for i in range(min(5, len(ranks))):
        assert tuples[i] == unrank(n, lo, hi, int(ranks[i]))
    by_k = {}
    for i, t in enumerate(tuples):
        by_k.setdefault(len(t), []).append(i)
    for k, rows_i in by_k.items():
        idx = np.array([tuples[i] for i in rows_i], dtype=np.int64)
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(n, indices=idx), bias_correct=bias)
        out[:, rows_i, :] = np.stack([h.tc, h.dtc, h.o, h.s])
    return idx_pad, out


def main():
    meta = {}

    # ---- copula core --------------------------------------------------
    rng = np.random.default_rng(1)
    x = rng.standard_normal((40, 3))
    x[::5, 1] = 0.25                      # ties
    x[3, 2] = -0.0
    x[7, 2] = 0.0                         # signed-zero tie
    tie = np.array([[2.0], [1.0], [2.0], [1.0]])
    cov_small = hoi.estimate_covariance(hoi.copula_transform(hoi.DataMatrix(x)))
    bias_pairs = [(n, t) for n in range(1, 11) for t in (n + 1, 50, 937)]
    np.savez_compressed(
        HERE / "copula.npz",
        x=x, ranks=hoi.rank_columns(hoi.DataMatrix(x)),
        z=hoi.copula_transform(hoi.DataMatrix(x)).values, cov=cov_small.sigma,
        tie=tie, tie_ranks=hoi.rank_columns(hoi.DataMatrix(tie)),
        bias_pairs=np.array(bias_pairs),
        bias_vals=np.array([hoi.entropy_bias(n, t) for n, t in bias_pairs]),
        bias_tab_60=hoi.copula_core._bias_table(60, 12),
        bias_tab_2000=hoi.copula_core._bias_table(2000, 30),
        bias_tab_10000=hoi.copula_core._bias_table(10000, 20),
        gauss_ent=np.array([hoi.gaussian_entropy_nats(np.array([[1.0, 0.5], [0.5, 1.0]])).nats]),
    )

    # ---- cfg1: full scan, no bias ------------------------------------
    x1 = workloads.cfg1()
    c1 = covset_of(x1)
    v1 = full_scan(c1, 3, 10, False)
    np.savez_compressed(HERE / "cfg1.npz", x=x1, cov=c1.covs[0].sigma, vals=v1[:, :, 0])
    meta["cfg1"] = {"rows": int(v1.shape[1]), "x_sha": sha(x1)}

    # ---- cfg2: full scan, bias on -------------------------------------
    x2 = workloads.cfg2()
    c2 = covset_of(x2)
    v2 = full_scan(c2, 3, 12, True)
    np.savez_compressed(HERE / "cfg2.npz", cov=c2.covs[0].sigma, t=x2.shape[0],
                        vals=v2[:, :, 0])
    meta["cfg2"] = {"rows": int(v2.shape[1]), "x_sha": sha(x2),
                    "o_0123": float(v2[2, lex_rank(12, (0, 1, 2, 3)) + math.comb(12, 3), 0]),
                    "o_456": float(v2[2, lex_rank(12, (4, 5, 6)), 0])}

    # ---- cfg3: ties, top-k / histogram over the full scan ------------
    x3 = workloads.cfg3()
    d3 = hoi.DataMatrix(x3)
    r3 = hoi.rank_columns(d3)
    c3 = covset_of(x3)
    top_o = hoi.scan(c3, 3, 20, hoi.TopK("o", "min", 10))
    top_s = hoi.scan(c3, 3, 20, hoi.TopK("s", "max", 10), bias_correct=True)
    edges, counts = hoi.scan(c3, 3, 20, hoi.Histogram("o", 16, -0.5, 2.0))
    g3 = sampled_ranks(20, 3, 20, 1500, seed=3)
    i3, m3 = sample_measures(c3, 20, 3, 20, g3, False)
    _, m3b = sample_measures(c3, 20, 3, 20, g3, True)
    np.savez_compressed(HERE / "cfg3.npz", cov=c3.covs[0].sigma, t=x3.shape[0],
                        ranks_sha=np.array(sha(r3)),
                        n_ties=np.array(int(sum(len(x3[:, j]) - len(np.unique(x3[:, j]))
                                                for j in range(20)))),
                        g=g3, idx=i3, vals=m3, vals_bias=m3b,
                        hist_edges=edges, hist_counts=counts)
    meta["cfg3"] = {
        "top_o_min": [[list(e.indices), e.value, e.tc, e.dtc, e.o, e.s] for e in top_o[0]],
        "top_s_max_bias": [[list(e.indices), e.value, e.tc, e.dtc, e.o, e.s] for e in top_s[0]],
        "x_sha": sha(x3),
    }

    # ---- cfg4: sampled global ranks ----------------------------------
    x4 = workloads.cfg4()
    c4 = covset_of(x4)
    g4 = sampled_ranks(30, 2, 30, 3000, seed=4)
    i4, m4 = sample_measures(c4, 30, 2, 30, g4, False)
    _, m4b = sample_measures(c4, 30, 2, 30, g4, True)
    np.savez_compressed(HERE / "cfg4.npz", x=x4, cov=c4.covs[0].sigma, t=x4.shape[0],
                        g=g4, idx=i4, vals=m4, vals_bias=m4b)
    meta["cfg4"] = {"x_sha": sha(x4), "count": hoi.count_nplets(30, 2, 30)}

    # ---- edge cases --------------------------------------------------
    ident = hoi.CovSet([hoi.CovarianceMatrix(np.eye(6))])
    idv = {}
    for k in (2, 3, 4, 6):
        idx = np.array(list(itertools.combinations(range(6), k)))
        h = hoi.compute_hoi_batch(ident, hoi.NpletBatch(6, indices=idx))
        idv[k] = np.stack([h.tc, h.dtc, h.o, h.s])
    rs = {}
    for m in (2, 3, 4):
        for kind, fn in (("r", hoi.r_system_cov), ("s", hoi.s_system_cov)):
            cov = fn(m, 1.0)
            h = hoi.compute_hoi_batch(hoi.CovSet([cov]),
                                      hoi.NpletBatch(m + 1, indices=np.arange(m + 1)[None]))
            rs[f"{kind}{m}"] = np.array([h.tc[0, 0], h.dtc[0, 0], h.o[0, 0], h.s[0, 0]])
    # not-PD coordinates and jitter rescue (tests/test_nplet_engine.py:155-173)
    bad = np.array([[1.0, 2.0], [2.0, 1.0]])
    try:
        _batched_logdet_invdiag(np.stack([np.eye(2), bad])[:, None])
        npd = None
    except hoi.NotPositiveDefinite as e:
        npd = [list(c) for c in e.coords]
    singular = np.ones((3, 3)) + np.eye(3) * 1e-14
    ld_s, id_s = _batched_logdet_invdiag(singular[None, None])
    # mixed masks (acceptance criterion 2 inputs)
    analytic = hoi.block_concat([hoi.r_system_cov(7, 0.8), hoi.s_system_cov(6, 0.9)])
    rng = np.random.default_rng(2)
    seen = set()
    while len(seen) < 300:
        k = int(rng.integers(1, 16))
        seen.add(tuple(sorted(int(v) for v in rng.choice(15, size=k, replace=False))))
    masks = np.zeros((300, 15), dtype=bool)
    for r, t in enumerate(sorted(seen)):
        masks[r, list(t)] = True
    hm = hoi.compute_hoi_batch(hoi.CovSet([analytic]), hoi.NpletBatch(15, masks=masks))
    tm = hoi.entropy_terms(hoi.CovSet([analytic]), hoi.NpletBatch(15, masks=masks))
    # random fixed batch with 2 datasets, terms + measures, bias on
    rng = np.random.default_rng(4)
    covs2 = []
    for _ in range(2):
        a = rng.standard_normal((12, 6))
        covs2.append(hoi.CovarianceMatrix(a.T @ a / 12 + 0.5 * np.eye(6), n_samples_used=60))
    cs2 = hoi.CovSet(covs2)
    idx3 = np.array(list(itertools.combinations(range(6), 3)))
    te = hoi.entropy_terms(cs2, hoi.NpletBatch(6, indices=idx3), bias_correct=True)
    he = hoi.compute_hoi_batch(cs2, hoi.NpletBatch(6, indices=idx3), bias_correct=True)
    np.savez_compressed(
        HERE / "edge.npz",
        ident2=idv[2], ident3=idv[3], ident4=idv[4], ident6=idv[6],
        singular_ld=ld_s, singular_id=id_s,
        mix_sigma=analytic.sigma, mix_masks=masks,
        mix_vals=np.stack([hm.tc, hm.dtc, hm.o, hm.s]),
        mix_hj=tm.h_joint, mix_hs=tm.h_singles, mix_hl=tm.h_leave_one_out,
        t2_sig=cs2.stacked(), t2_idx=idx3, t2_hj=te.h_joint, t2_hs=te.h_singles,
        t2_hl=te.h_leave_one_out, t2_vals=np.stack([he.tc, he.dtc, he.o, he.s]),
        **{f"rs_{k}": v for k, v in rs.items()},
    )
    meta["edge"] = {"npd_coords": npd,
                    "counts": {f"{n},{lo},{hi}": hoi.count_nplets(n, lo, hi)
                               for n, lo, hi in [(3, 1, 3), (8, 3, 8), (12, 2, 7), (20, 1, 20),
                                                 (30, 3, 30), (30, 2, 30), (64, 1, 4)]}}

    # ---- reducers on toy covsets (tests/test_scanner.py) -------------
    def toy(seed, n, d):
        rng = np.random.default_rng(seed)
        cs = []
        for _ in range(d):
            a = rng.standard_normal((3 * n, n))
            cs.append(hoi.CovarianceMatrix(a.T @ a / (3 * n)))
        return hoi.CovSet(cs)

    red = {}
    t1 = toy(1, 6, 1)
    for direction in ("max", "min"):
        got = hoi.scan(t1, 3, 5, hoi.TopK("o", direction, 7))
        red[f"top_o_{direction}"] = [[list(e.indices), e.value, e.tc, e.dtc, e.o, e.s]
                                     for e in got[0]]
    t2 = toy(2, 7, 2)
    got = hoi.scan(t2, 3, 6, hoi.TopK("s", "max", 9))
    red["top_s_max_d2"] = [[[list(e.indices), e.value, e.tc, e.dtc, e.o, e.s] for e in per]
                           for per in got]
    eye5 = hoi.CovSet([hoi.CovarianceMatrix(np.eye(5))])
    red["top_tie"] = [list(e.indices) for e in hoi.scan(eye5, 3, 3, hoi.TopK("o", "max", 4))[0]]
    t3 = toy(3, 6, 2)
    e1, c1h = hoi.scan(t3, 2, 4, hoi.Histogram("tc", 8, 0.0, 0.5))
    e2, c2h = hoi.scan(t3, 2, 4, hoi.Histogram("tc", 2, 0.20, 0.21))
    red["hist_8"] = c1h.tolist()
    red["hist_2"] = c2h.tolist()
    t7 = toy(7, 6, 3)
    red["features_t7"] = [f.as_dict() for f in hoi.extract_features(t7)]
    red["features_r3"] = [f.as_dict() for f in hoi.extract_features(hoi.CovSet([hoi.r_system_cov(3, 1.0)]))]
    red["features_eye5"] = [f.as_dict() for f in hoi.extract_features(eye5)]
    meta["reducers"] = red
    meta["toy_sigmas"] = {"t1": t1.stacked().tolist(), "t2": t2.stacked().tolist(),
                          "t3": t3.stacked().tolist(), "t7": t7.stacked().tolist()}
    meta["frozen"] = {"BIAS_1_2": ref_slow.entropy_bias(1, 2),
                      "count_30_3_30": ref_slow.count_subsets(30, 3, 30)}
    meta["versions"] = {"numpy": np.__version__, "python": sys.version.split()[0]}
    import scipy
    meta["versions"]["scipy"] = scipy.__version__
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, os.path.getsize(p))


if __name__ == "__main__":
    main()
