"""Lattice full-output scan time at N = 20 (orders 2..20) against the number
of datasets D (diagnostic: output layout (rows, D) interleaves datasets)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, workloads
from paper_2501_03381_b200.scanner import _ScanCtx

_build.build()
rng = np.random.default_rng(7)
res = {}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for d in (1, 2, 4, 8, 16, 52):
    covs = hoi.CovSet([hoi.CovarianceMatrix(workloads.randcorr(n, rng)) for _ in range(d)])
    ctx = _ScanCtx(covs, 2, n, False)
    total = hoi.count_nplets(n, 2, n)
    out = torch.empty((4, total, d), dtype=torch.float64, device="cuda")
    ctx.full(0, total, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.full(0, total, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[d] = {"ms": round(ms, 3), "ms_per_dataset": round(ms / d, 4),
              "out_GBps": round(32 * total * d / (ms * 1e-3) / 1e9, 1)}
    del out
print(json.dumps({"n": n, "by_D": res}))
