"""Golden results of the REAL reference for a system beyond the device
unranking table (N = 100 > 64): scan TopK, greedy and anneal.

Build container only (imports /root/reference):

    python tests/golden/make_golden_large.py  ->  tests/golden/large.npz, large.json
"""

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hoi  # noqa: E402  (the reference)


def main():
    n = 100
    rng = np.random.default_rng(100)
    sig = []
    for d in range(2):
        a = rng.standard_normal((n, n // 4))
        s = a @ a.T / (n // 4) + np.eye(n)
        dd = np.sqrt(np.diag(s))
        s = s / np.outer(dd, dd)
        sig.append(0.5 * (s + s.T))
    sig = np.stack(sig)
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=500) for s in sig])
    out = {}
    top = hoi.scan(covs, 2, 3, hoi.TopK("o", "min", 12))
    out["scan_top"] = [[[list(e.indices), e.value, e.tc, e.dtc, e.o, e.s] for e in per]
                       for per in top]
    spec = hoi.ObjectiveSpec("o", "max")
    g = hoi.greedy(covs, spec, 3, 5, kappa=4)
    out["greedy"] = [[e.order, list(e.indices), e.energy, e.value] for e in g.per_order]
    st = hoi.anneal(covs, spec, hoi.AnnealSchedule(max_iters=40, min_order=3, max_order=8),
                    kappa=6, seed=1)
    out["anneal"] = {"best_indices": list(st.best_indices), "best_energy": st.best_energy,
                     "iterations": st.iterations, "energies": st.energies.tolist()}
    np.savez_compressed(HERE / "large.npz", sigma=sig)
    (HERE / "large.json").write_text(json.dumps(out, indent=1))
    print("ok")


if __name__ == "__main__":
    main()
