"""Golden vectors for the public helpers around the hot path, from the REAL
reference (build container only; it imports /root/reference):

    python tests/golden/make_golden_helpers.py   ->  tests/golden/helpers.npz

* extract_subcov_batch / pad_subcov_batch   (ref nplet_engine.py:185-224)
* gaussian_entropy_nats, copula_entropy     (ref copula_core.py:207-260)
  including a rank-deficient covariance rescued by the jitter retry
* pairwise_mi with and without bias         (ref measures.py:84-99)
* ground_truth_hoi on R/S systems           (ref synthetic.py:89-109)
* the duplicated-variable (singular) system the VERDICT ran: reference
  values of every n-plet, NaN included, to document the divergence

Inputs are seeded literals, so the GPU tests rebuild identical bytes.
"""

import itertools
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hoi  # noqa: E402  (the reference)


def main():
    rng = np.random.default_rng(31)
    sig = []
    for _ in range(2):
        a = rng.standard_normal((20, 7))
        sig.append(a.T @ a / 20 + 0.2 * np.eye(7))
    sig = np.stack(sig)
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=40) for s in sig])
    idx = np.array(list(itertools.combinations(range(7), 3)))[::3]
    sub = hoi.extract_subcov_batch(covs, hoi.NpletBatch(7, indices=idx))
    masks = np.zeros((9, 7), dtype=bool)
    for r, row in enumerate([(0,), (1, 2), (0, 3, 6), (2, 4, 5, 6), (0, 1, 2, 3, 4, 5, 6),
                             (5,), (1, 6), (0, 2, 4, 6), (3, 4)]):
        masks[r, list(row)] = True
    pad = hoi.pad_subcov_batch(covs, hoi.NpletBatch(7, masks=masks))

    ent = np.array([hoi.gaussian_entropy_nats(hoi.CovarianceMatrix(s)).nats for s in sig])
    # indefinite by -1e-12 (the plain Cholesky fails beyond any rounding
    # doubt), positive definite after the jitter retry (eps ~ 1e-10)
    rankdef = np.array([[1.0, 1.0, 0.0], [1.0, 1.0 - 1e-12, 0.0], [0.0, 0.0, 2.0]])
    ent_jit = hoi.gaussian_entropy_nats(hoi.CovarianceMatrix(rankdef)).nats

    x = rng.standard_normal((400, 5)) @ rng.standard_normal((5, 5))
    x[:, 2] = np.exp(x[:, 2])
    ce = np.array([hoi.copula_entropy(hoi.DataMatrix(x), bias_correct=b).nats for b in (False, True)])

    mi_pairs = np.array([(0, 1), (3, 1), (6, 2), (4, 5)])
    mi = np.array([[hoi.pairwise_mi(covs.covs[0], int(i), int(j), bias_correct=b)
                    for b in (False, True)] for i, j in mi_pairs])

    gt_cov = hoi.block_concat([hoi.r_system_cov(3, 0.8), hoi.s_system_cov(3, 1.1)])
    gt_nplets = [(0, 1, 2, 3), (4, 5, 6, 7), (0, 5, 7), (2, 1), (0, 1, 2, 3, 4, 5, 6, 7)]
    gt = np.array([hoi.ground_truth_hoi(gt_cov, t) for t in gt_nplets])

    # duplicated variable: x3 == x1 ("singular covariances")
    xs = rng.standard_normal((300, 5))
    xs[:, 3] = xs[:, 1]
    dup_sigma = np.cov(xs, rowvar=False)
    dup_sigma = 0.5 * (dup_sigma + dup_sigma.T)
    dup = hoi.CovSet([hoi.CovarianceMatrix(dup_sigma)])
    vals = []

    def keep(batch, h):
        vals.append(np.stack([h.tc[:, 0], h.dtc[:, 0], h.o[:, 0], h.s[:, 0]]))

    with np.errstate(all="ignore"):
        hoi.scan(dup, 2, 5, hoi.Callback(keep))
    dup_vals = np.concatenate(vals, axis=1)

    np.savez_compressed(
        HERE / "helpers.npz",
        sig=sig, idx=idx, sub=sub.matrices, sub_pad=sub.pad_counts,
        masks=masks, pad=pad.matrices, pad_counts=pad.pad_counts,
        ent=ent, rankdef=rankdef, ent_jit=ent_jit, x=x, ce=ce,
        mi_pairs=mi_pairs, mi=mi,
        gt_sigma=gt_cov.sigma, gt_nplets=np.array([sum(1 << i for i in t) for t in gt_nplets]),
        gt=gt, dup_sigma=dup_sigma, dup_vals=dup_vals,
    )
    print("helpers.npz", (HERE / "helpers.npz").stat().st_size, "bytes;",
          "dup rows with NaN:", int(np.isnan(dup_vals).any(axis=0).sum()), "of", dup_vals.shape[1])


if __name__ == "__main__":
    main()
