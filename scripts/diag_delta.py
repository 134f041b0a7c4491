"""Diagnostic: explain wrong neighbour sums of stacked lattice scans."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import workloads, _build
from paper_2501_03381_b200.scanner import _ScanCtx
from paper_2501_03381_b200.nplet_engine import unrank_device
_build.build()
N, D = 20, 8
nP = N - 10
covl = [hoi.CovarianceMatrix(workloads.randcorr(N, np.random.default_rng(s))) for s in range(D)]
ctx = _ScanCtx(hoi.CovSet(covl), 2, N, False)
total = hoi.count_nplets(N, 2, N)
outs = []
for r in range(3):
    o = torch.empty((4, total, D), dtype=torch.float64, device="cuda")
    ctx.full(0, total, o)
    torch.cuda.synchronize()
    outs.append(o.cpu().numpy())
t = 8 << N
off = t + 4096 + (4 << (N - 10)); off = (off + 255) & ~255
off += (4 << (N - 9)) + 64 + 8192; off = (off + 255) & ~255
T = ctx.ws[off:off + D * t].view(torch.float64).view(D, 1 << N).cpu().numpy()
tup, orders = unrank_device(N, 2, N, 0, total)
tup, orders = tup.cpu().numpy(), orders.cpu().numpy()
def swz(e): return (e & ~31) | ((e ^ (e >> 5)) & 31)
def addr(mask):
    P = mask & ((1 << nP) - 1); e = mask >> nP
    return P * 1024 + swz(e)
# majority value per entry across runs (2 of 3 agree) as "truth" for the check
A, B, C = outs
bad = np.argwhere((A[1] != B[1]) | (A[1] != C[1]))
print("entries differing between runs", len(bad))
stats = {}
for r, d in bad[:300]:
    k = int(orders[r]); S = [int(v) for v in tup[r, :k]]
    mask = sum(1 << v for v in S)
    l = T[d, addr(mask)]
    nb_true = sum(T[d, addr(mask & ~(1 << v))] for v in S)
    for name, o in (("A", A), ("B", B), ("C", C)):
        nb = 2 * o[1, r, d] - (1 - k) * l
        delta = nb - nb_true
        if abs(delta) < 1e-9 * (1 + abs(nb_true)):
            continue
        expl = "?"
        for v in S:
            if v >= nP: continue
            nbv = mask & ~(1 << v)
            tv = T[d, addr(nbv)]
            if abs(delta + tv) < 1e-9: expl = "missing neighbour block"; break
            if abs(delta - tv) < 1e-9: expl = "neighbour block twice"; break
            for d2 in range(D):
                if d2 != d and abs(delta - (T[d2, addr(nbv)] - tv)) < 1e-9:
                    expl = f"neighbour from dataset offset {d2 - d:+d}"; break
            if expl != "?": break
        stats[expl] = stats.get(expl, 0) + 1
print(stats)
# is the wrong nb the true nb of the same in-block entry e in another block / dataset?
Tm = T.reshape(D, 1 << nP, 1024)
def nb_all(e_mask):
    """true nb for entry e in every (dataset, block): (D, 2^nP)"""
    res = np.zeros((D, 1 << nP))
    for P in range(1 << nP):
        mask = P | (e_mask << nP)
        bits = [v for v in range(N) if (mask >> v) & 1]
        res[:, P] = sum(T[:, addr(mask & ~(1 << v))] for v in bits)
    return res
shown = 0
for r, d in bad[:40]:
    k = int(orders[r]); S = [int(v) for v in tup[r, :k]]
    mask = sum(1 << v for v in S); P = mask & ((1 << nP) - 1); e = mask >> nP
    l = T[d, addr(mask)]
    for name, o in (("A", A), ("B", B), ("C", C)):
        nb = 2 * o[1, r, d] - (1 - k) * l
        allnb = nb_all(e)
        hit = np.argwhere(np.abs(allnb - nb) < 1e-9 * (1 + abs(nb)))
        if abs(nb - allnb[d, P]) > 1e-9 * (1 + abs(nb)):
            print(f"row {r} d {d} P {P} e {e} run {name}: nb {nb:.6f} true {allnb[d, P]:.6f} matches (d,P) {hit[:4].tolist()}")
            shown += 1
    if shown > 12:
        break
