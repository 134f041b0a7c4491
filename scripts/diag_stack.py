"""Diagnostic: run-to-run stability of lattice scans (stacked and single)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import workloads, _build
from paper_2501_03381_b200.scanner import _ScanCtx
from paper_2501_03381_b200.nplet_engine import unrank_device
_build.build()
N = 20
total = hoi.count_nplets(N, 2, N)
for D in (1, 8):
    covl = [hoi.CovarianceMatrix(workloads.randcorr(N, np.random.default_rng(s))) for s in range(D)]
    ctx = _ScanCtx(hoi.CovSet(covl), 2, N, False)
    outs = []
    for r in range(4):
        o = torch.empty((4, total, D), dtype=torch.float64, device="cuda")
        ctx.full(0, total, o)
        torch.cuda.synchronize()
        outs.append(o)
    diffs = [(outs[i] != outs[0]) for i in range(1, 4)]
    print("D", D, "run-to-run mismatches", [int(x.sum()) for x in diffs])
    m = diffs[0] | diffs[1] | diffs[2]
    if int(m.sum()):
        idx = m.nonzero().cpu().numpy()
        rows = np.unique(idx[:, 1])
        print("planes", np.unique(idx[:, 0]), "datasets", np.unique(idx[:, 2]), "rows", len(rows))
        tup, orders = unrank_device(N, 2, N, 0, total)
        tup = tup.cpu().numpy(); orders = orders.cpu().numpy()
        Ps = []
        for r in rows[:400]:
            mem = tup[r, :orders[r]]
            P = sum(1 << int(v) for v in mem if v < N - 10)
            Ps.append(P)
        Ps = np.array(Ps)
        print("distinct blocks", len(np.unique(Ps)), "popc", np.bincount([bin(p).count('1') for p in Ps]), "orders", np.bincount(orders[rows[:400]]))
        print("sample blocks", np.unique(Ps)[:20])
    del outs
