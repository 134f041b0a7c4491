"""BASELINE config 5 TopK timing breakdown: kernel, device TopK (select +
exact order + winners to host), and topk_batch end to end from host indices."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_03381_b200 as hoi  # noqa: E402
from paper_2501_03381_b200 import _build, workloads  # noqa: E402


def main():
    _build.build()
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d)))
                       for d in range(16)])
    idx = workloads.cfg5_nplets()
    batch = hoi.NpletBatch(400, indices=idx, check_unique=False)
    res = {}
    times = []
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        top = hoi.topk_batch(covs, batch, hoi.TopK("o", "min", 1000)).finalize()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    res["e2e_ms"] = [round(t * 1e3, 2) for t in times]
    t0 = time.perf_counter()
    ent = [list(t) for t in top]
    res["materialize_16000_entries_ms"] = (time.perf_counter() - t0) * 1e3
    # breakdown with torch profiler-free CUDA events around the stages
    from paper_2501_03381_b200.nplet_engine import eval_device
    keep = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, _, _ = eval_device(covs, batch, False, keep_idx=keep)
    torch.cuda.synchronize()
    res["eval_device_ms"] = (time.perf_counter() - t0) * 1e3
    from paper_2501_03381_b200.scanner import _BatchCtx, _topk_batch_device
    red = hoi.TopK("o", "min", 1000)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ok = _topk_batch_device(_BatchCtx(16, torch), red, out, keep[0], batch)
    torch.cuda.synchronize()
    res["device_topk_ms"] = (time.perf_counter() - t0) * 1e3
    res["device_path"] = ok
    print(json.dumps(res))


if __name__ == "__main__":
    main()
