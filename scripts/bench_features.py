"""The paper's many-dataset workload (~920 datasets, N = 5..20,
all orders 2..N, the 21-feature fingerprint): seeded synthetic stand-in.
920 datasets, N drawn uniformly from 5..20, T = 1000 samples of a random
correlation latent; datasets of equal N share one CovSet (one scan with D
datasets).  Device wall time of extract_features for all 920, and the
CPU oracle (the reference algorithm) on a bounded sample, extrapolated."""
import json, math, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np
import torch
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, workloads


def main():
    _build.build()
    rng = np.random.default_rng(920)
    ns = rng.integers(5, 21, size=920)
    groups = {}
    for n in ns:
        c = workloads.randcorr(int(n), rng)
        x = rng.standard_normal((1000, int(n))) @ np.linalg.cholesky(c).T
        groups.setdefault(int(n), []).append(hoi.estimate_covariance(hoi.copula_transform(x)))
    covsets = {n: hoi.CovSet(v) for n, v in groups.items()}
    hoi.extract_features(covsets[min(covsets)])          # warm-up (build, tables)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    feats = {n: hoi.extract_features(cs) for n, cs in covsets.items()}
    torch.cuda.synchronize()
    dev = time.perf_counter() - t0
    nplets = sum(len(v) * hoi.count_nplets(n, 2, n) for n, v in groups.items())
    # CPU oracle: one dataset of every N (the same scan + accumulator), scaled by the counts
    import hoi_oracle as ora
    cpu = 0.0
    for n, v in groups.items():
        sig = v[0].sigma
        t0 = time.perf_counter()
        ora.scan(sig, [0], 2, n, ora.FeaturesR(n))
        cpu += (time.perf_counter() - t0) * len(v)
    print(json.dumps({"datasets": int(len(ns)), "nplet_dataset_units": int(nplets),
                      "device_s": dev, "units_per_s": nplets / dev,
                      "cpu_oracle_s_extrapolated": cpu, "cpu_cores": 1,
                      "groups": {int(n): len(v) for n, v in sorted(groups.items())}}))


if __name__ == "__main__":
    main()
