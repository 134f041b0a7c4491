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
