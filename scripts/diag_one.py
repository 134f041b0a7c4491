"""One N=20, D=8 lattice full scan (for compute-sanitizer)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import workloads, _native
from paper_2501_03381_b200.scanner import _ScanCtx
_native.load()
N, D = int(sys.argv[1]), int(sys.argv[2])
covl = [hoi.CovarianceMatrix(workloads.randcorr(N, np.random.default_rng(s))) for s in range(D)]
ctx = _ScanCtx(hoi.CovSet(covl), 2, N, False)
total = hoi.count_nplets(N, 2, N)
o = torch.empty((4, total, D), dtype=torch.float64, device="cuda")
ctx.full(0, total, o)
torch.cuda.synchronize()
print("done", float(o[1].sum()))
