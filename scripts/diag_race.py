"""Diagnostic: run-to-run stability of full lattice scans, single dataset at
larger N (more blocks per persistent CTA) and stacked datasets."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import workloads, _build
from paper_2501_03381_b200.scanner import _ScanCtx
_build.build()
for N, D in [(int(a.split("x")[0]), int(a.split("x")[1])) for a in sys.argv[1:]]:
    total = hoi.count_nplets(N, 2, N)
    covl = [hoi.CovarianceMatrix(workloads.randcorr(N, np.random.default_rng(s))) for s in range(D)]
    ctx = _ScanCtx(hoi.CovSet(covl), 2, N, False)
    ref = torch.empty((4, total, D), dtype=torch.float64, device="cuda")
    ctx.full(0, total, ref)
    o = torch.empty_like(ref)
    mism = []
    for r in range(4):
        ctx.full(0, total, o)
        torch.cuda.synchronize()
        mism.append(int((o != ref).sum()))
    print(f"N={N} D={D} blocks/dataset={2 ** (N - 10)} run-to-run mismatches {mism}", flush=True)
    del ref, o
    torch.cuda.empty_cache()
