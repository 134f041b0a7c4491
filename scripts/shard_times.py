"""Per-rank block-shard step times for G = 2, 4, 8 GPUs (block_shard_plan:
two complementary shards per rank), measured one rank at a time on ONE B200
(each rank's own work: the table chunks its shards read and its stencil
share, CUDA events).  The multi-GPU step is bounded below by the
slowest rank; this is that bound, not a concurrent multi-GPU measurement."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, workloads
from paper_2501_03381_b200.scanner import _ScanCtx
from paper_2501_03381_b200.sharding import block_shard_plan

_build.build()
N, LO, HI = 30, 2, 30
covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg4()))])
ctx = _ScanCtx(covs, LO, HI, False)
total = hoi.count_nplets(N, LO, HI)
out = torch.empty((4, total, 1), dtype=torch.float64, device="cuda")
res = {}
ctx.full(0, total, out)                  # single-GPU step for reference
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    ctx.full(0, total, out)
e1.record(); torch.cuda.synchronize()
one = e0.elapsed_time(e1) / 3
res["1"] = {"step_ms": round(one, 3)}
for g in (2, 4, 8):
    sb, masks = block_shard_plan(N, g)
    per = []
    for r in range(g):
        ctx.full_shard_set(masks[r], sb, out)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            ctx.full_shard_set(masks[r], sb, out)
        e1.record(); torch.cuda.synchronize()
        per.append(round(e0.elapsed_time(e1) / 3, 3))
    res[str(g)] = {"per_rank_ms": per, "max_ms": max(per),
                   "speedup_bound": round(one / max(per), 2),
                   "efficiency_bound": round(one / max(per) / g, 3)}
print(json.dumps({"workload": "cfg4 full output, block shards", "by_gpus": res}))
