"""Stage timing of bench.py's e2e leg (cfg4, public API, TopK('o','min',1000)):
host-clock per stage with a sync on each side, then one profiled call's
device kernel list (CUPTI via torch.profiler)."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import workloads

x = workloads.cfg4()
pinned = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = x
xh = pinned.numpy()


def once():
    t = [time.perf_counter()]
    dm = hoi.DataMatrix(xh)
    cop = hoi.copula_transform(dm)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    cov = hoi.estimate_covariance(cop)
    covs = hoi.CovSet([cov])
    torch.cuda.synchronize(); t.append(time.perf_counter())
    res = hoi.scan(covs, 2, 30, hoi.TopK("o", "min", 1000))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    return np.diff(t) * 1e3


rows = [once() for _ in range(6)][1:]
med = np.median(np.array(rows), axis=0)
print(json.dumps({"copula_ms": med[0], "cov_ms": med[1], "scan_ms": med[2], "total_ms": med.sum()}))

from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    once()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  {e.time_range.elapsed_us() / 1e3:8.3f} ms  {e.name[:90]}")
