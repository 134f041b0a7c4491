"""Per-group timing of the 920-dataset feature workload (scripts/bench_features.py's
inputs) and the device kernel list of the largest group (diagnostic)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, workloads

_build.build()
rng = np.random.default_rng(920)
ns = rng.integers(5, 21, size=920)
groups = {}
for n in ns:
    c = workloads.randcorr(int(n), rng)
    x = rng.standard_normal((1000, int(n))) @ np.linalg.cholesky(c).T
    groups.setdefault(int(n), []).append(hoi.estimate_covariance(hoi.copula_transform(x)))
covsets = {n: hoi.CovSet(v) for n, v in groups.items()}
for cs in covsets.values():
    hoi.extract_features(cs)
torch.cuda.synchronize()
import gc
for label in ("gc on", "gc off", "gc on"):
    if label == "gc off":
        gc.disable()
    else:
        gc.enable()
    per = {}
    for n, cs in sorted(covsets.items()):
        t0 = time.perf_counter()
        hoi.extract_features(cs)
        torch.cuda.synchronize()
        per[n] = (len(groups[n]), round((time.perf_counter() - t0) * 1e3, 3))
    print(label, json.dumps({"per_group_ms": per, "total_ms": sum(v[1] for v in per.values())}))
gc.enable()
from torch.profiler import profile, ProfilerActivity
big = max(covsets, key=lambda n: len(groups[n]) * 2 ** n)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    hoi.extract_features(covsets[big])
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
tot = {}
for e in evs:
    tot.setdefault(e.name[:70], [0, 0.0])
    tot[e.name[:70]][0] += 1
    tot[e.name[:70]][1] += e.time_range.elapsed_us() / 1e3
print("group N =", big, "datasets", len(groups[big]))
for k, (c, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"{ms:9.3f} ms  {c:5d}x  {k}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); hoi.extract_features(covsets[big]); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(22)
