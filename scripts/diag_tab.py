"""Diagnostic: stability of the stacked log-det tables across rebuilds."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import workloads, _build
from paper_2501_03381_b200.scanner import _ScanCtx
_build.build()
N, D = 20, 8
covl = [hoi.CovarianceMatrix(workloads.randcorr(N, np.random.default_rng(s))) for s in range(D)]
ctx = _ScanCtx(hoi.CovSet(covl), 2, N, False)
total = hoi.count_nplets(N, 2, N)
o = torch.empty((4, total, D), dtype=torch.float64, device="cuda")
t = 8 << N
off = t + 4096 + (4 << (N - 10)); off = (off + 255) & ~255
off += (4 << (N - 9)) + 64 + 8192; off = (off + 255) & ~255
tabs = []
for r in range(4):
    ctx.full(0, total, o)
    torch.cuda.synchronize()
    tabs.append(ctx.ws[off:off + D * t].clone())
print("table rebuild mismatches (bytes)", [int((tabs[i] != tabs[0]).sum()) for i in range(4)])
