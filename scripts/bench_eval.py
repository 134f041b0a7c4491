"""Per-n-plet engine timing: cfg5 batched K=10 (D=16, N=400) and cfg4
per-order segments (engine 1).  Diagnostic; prints one JSON line."""
import json, math, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, _native as nat, workloads
from paper_2501_03381_b200._device import device_covs
from paper_2501_03381_b200.sharding import nplet_flops
from paper_2501_03381_b200.scanner import _ScanCtx


def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    _build.build()
    lib = nat.lib()
    res = {}
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d))) for d in range(16)])
    st = device_covs(covs)
    B = 1 << 20
    idx = torch.from_numpy(workloads.cfg5_nplets(b=B).astype(np.int32)).cuda()
    out = torch.empty((4, B, 16), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    coords = torch.zeros(2 * 64, dtype=torch.int64, device="cuda")
    s = nat.stream_handle(torch)
    def run():
        nat.check(lib.hoi_eval_indices(st.corr.data_ptr(), st.sdiag.data_ptr(), None, 0, 400, 16,
                                       idx.data_ptr(), B, 10, out.data_ptr(), None, None,
                                       cnt.data_ptr(), coords.data_ptr(), 64, s))
    ms = ev_time(run)
    units = B * 16
    res["cfg5_k10"] = {"ms": ms, "units_per_s": units / (ms * 1e-3),
                       "tflops": units * nplet_flops(10) / (ms * 1e-3) / 1e12}
    del out
    covs4 = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg4()))])
    ctx = _ScanCtx(covs4, 2, 30, False, 1)
    per = {}
    off = 0
    for k in range(2, 31):
        c = math.comb(30, k)
        n = min(c, 1 << 22)
        seg = torch.empty((4, n, 1), dtype=torch.float64, device="cuda")
        ms = ev_time(lambda: ctx.full(off, off + n, seg), reps=3)
        per[k] = {"ms": round(ms, 4), "tflops": round(n * nplet_flops(k) / (ms * 1e-3) / 1e12, 3)}
        off += c
    res["cfg4_orders"] = per
    print(json.dumps(res))


if __name__ == "__main__":
    main()
