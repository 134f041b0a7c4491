"""Time the per-n-plet kernel on BASELINE config 5 (4M order-10 n-plets x
16 datasets, N = 400): device-resident indices, CUDA events, FP64 TF/s
against the DFMA probe peak."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = sys.argv[:2]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_03381_b200 as hoi  # noqa: E402
from paper_2501_03381_b200 import _build, _native as nat, workloads  # noqa: E402
from paper_2501_03381_b200._device import device_covs  # noqa: E402
from paper_2501_03381_b200.sharding import nplet_flops  # noqa: E402


def main():
    _build.build()
    lib = nat.lib()
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d)))
                       for d in range(16)])
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
    idx = workloads.cfg5_nplets(b=b)
    B, D, K = idx.shape[0], 16, 10
    st = device_covs(covs)
    didx = torch.from_numpy(idx.astype(np.int32)).cuda()
    out = torch.empty((4, B, D), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    coords = torch.zeros(128, dtype=torch.int64, device="cuda")
    s = nat.stream_handle(torch)

    def ev():
        nat.check(lib.hoi_eval_indices(st.corr.data_ptr(), st.sdiag.data_ptr(), None, 0, 400, D,
                                       didx.data_ptr(), B, K, out.data_ptr(), None, None,
                                       cnt.data_ptr(), coords.data_ptr(), 64, s), "eval")
    for _ in range(3):
        ev()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    steps = 20
    e[0].record()
    for _ in range(steps):
        ev()
    e[1].record()
    torch.cuda.synchronize()
    kms = e[0].elapsed_time(e[1]) / steps
    peak = None
    try:
        from bench import fp64_peak  # noqa
        peak = fp64_peak(torch, lib, nat)
    except Exception:
        pass
    tf = B * D * nplet_flops(K) / (kms * 1e-3) / 1e12
    print(json.dumps({"kernel_ms": kms, "tflops": tf, "peak": peak,
                      "frac": tf / peak if peak else None, "units": B * D}))


if __name__ == "__main__":
    main()
