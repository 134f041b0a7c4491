"""Golden results of the REAL reference optimisers (greedy, anneal,
evaluate_objective; ref:optimizers.py) and PgmSpec (ref:synthetic.py).

Run in the build container only (imports /root/reference):

    python tests/golden/make_golden_optim.py

Writes tests/golden/optim.npz (the covariance stack the runs use) and
tests/golden/optim.json (results).  The covariances are stored, not
regenerated, so the GPU tests feed byte-identical inputs.
"""

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hoi  # noqa: E402  (the reference)


def covset():
    """D=4 sample covariances of a 12-variable system: an R block, an S
    block, independent noise, each dataset a different seeded sample."""
    spec = hoi.PgmSpec([hoi.PgmBlock("r", 3, 0.8), hoi.PgmBlock("s", 3, 0.9),
                        hoi.PgmBlock("independent", 4)])
    sig = spec.build()
    covs = []
    for d in range(4):
        x = hoi.sample_gaussian(sig, 400 + 100 * d, seed=100 + d)
        covs.append(hoi.estimate_covariance(hoi.copula_transform(x)))
    return spec, hoi.CovSet(covs)


def main():
    spec, covs = covset()
    out = {"pgm_json": spec.to_json(), "pgm_names": spec.variable_names(),
           "pgm_n": spec.n_variables}
    runs = {}
    specs = {
        "mean_o_max": hoi.ObjectiveSpec("o", "max"),
        "mean_s_min": hoi.ObjectiveSpec("s", "min"),
        "effect_tc_max": hoi.ObjectiveSpec("tc", "max", "effect", (0, 1), (2, 3)),
    }
    for name, sp in specs.items():
        for bias in (False, True):
            ev = []
            # start at order 3: at order 2 the O-information of every pair is
            # exactly 0 in exact arithmetic, so its ranking is rounding noise
            g = hoi.greedy(covs, sp, 3, 7, kappa=5, bias_correct=bias,
                           progress=lambda p, ev=ev: ev.append({k: p[k] for k in ("order", "batches", "nplets")}))
            runs[f"greedy_{name}_{int(bias)}"] = {
                "per_order": [[e.order, list(e.indices), e.energy, e.value] for e in g.per_order],
                "progress": ev}
    g = hoi.greedy(covs, specs["mean_o_max"], 3, 6, kappa=4, seed=7, restarts=3, batch_size=50)
    runs["greedy_restarts"] = {"per_order": [[e.order, list(e.indices), e.energy, e.value]
                                             for e in g.per_order]}
    for name, sched in {
        "anneal_across": hoi.AnnealSchedule(max_iters=80),
        "anneal_within": hoi.AnnealSchedule(temp0=0.05, mode="within-order", patience=15,
                                            max_iters=200, min_order=4, max_order=8),
    }.items():
        st = hoi.anneal(covs, specs["mean_o_max"], sched, kappa=8, seed=3)
        runs[name] = {"best_indices": list(st.best_indices), "best_energy": st.best_energy,
                      "iterations": st.iterations, "temperature": st.temperature,
                      "masks": st.masks.astype(int).tolist(), "energies": st.energies.tolist()}
    idx = np.array([[0, 1, 2], [3, 4, 5, ], [1, 6, 9], [2, 7, 11]])
    h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(12, indices=idx))
    out["objective"] = {name: hoi.evaluate_objective(h, sp).tolist() for name, sp in specs.items()}
    out["objective_idx"] = idx.tolist()
    out["runs"] = runs
    np.savez_compressed(HERE / "optim.npz", sigma=covs.stacked(),
                        t=np.array([c.n_samples_used for c in covs.covs]))
    (HERE / "optim.json").write_text(json.dumps(out, indent=1))
    print("ok", len(runs))


if __name__ == "__main__":
    main()
