"""cProfile of the cfg5 batched TopK stage (diagnostic)."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, workloads
from paper_2501_03381_b200.nplet_engine import eval_device
from paper_2501_03381_b200.scanner import _BatchCtx, _topk_plane

_build.build()
covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d))) for d in range(16)])
idx = workloads.cfg5_nplets()
batch = hoi.NpletBatch(400, indices=idx, check_unique=False)
out, _, _ = eval_device(covs, batch, False)
torch.cuda.synchronize()
def run():
    red = hoi.TopK("o", "min", 1000)
    _topk_plane(_BatchCtx(16, torch), red, out, 0, 2, lambda pos: [tuple(r) for r in idx[np.asarray(pos)].tolist()])
    torch.cuda.synchronize()
run()
t = time.perf_counter(); run(); print("topk stage", time.perf_counter() - t)
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)

# stage times of bench.py's cfg5 e2e call (topk_batch from host index arrays)
def e2e():
    torch.cuda.synchronize()
    t = time.perf_counter()
    hoi.topk_batch(covs, batch, hoi.TopK("o", "min", 1000)).finalize()
    torch.cuda.synchronize()
    return time.perf_counter() - t
e2e(); print("e2e", e2e())
t = time.perf_counter()
for d in range(16):
    hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d)))
torch.cuda.synchronize(); print("16 copula+cov (incl. data gen)", time.perf_counter() - t)
pr = cProfile.Profile(); pr.enable(); e2e(); pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)

import gc
def med(f, n=7):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts))
print("median topk stage", med(run), "e2e", med(e2e))
gc.disable()
print("gc off: median topk stage", med(run), "e2e", med(e2e))
gc.enable()
