"""Small, fixed workloads for ncu captures (one kernel family each).

    python scripts/profile_target.py lattice   # cfg4 exhaustive scan, lattice engine
    python scripts/profile_target.py copula5   # cfg5 copula + covariance (16 x 1200 x 400)
    python scripts/profile_target.py eval10    # cfg5-like batch: K=10, N=400, D=16
    python scripts/profile_target.py eval16    # cfg4 order-16 segment, per-n-plet engine (any order: evalK)
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_03381_b200 as hoi  # noqa: E402
from paper_2501_03381_b200 import _build, workloads  # noqa: E402
from paper_2501_03381_b200.scanner import _ScanCtx  # noqa: E402


def main(mode):
    _build.build()
    if mode == "lattice":
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg4()))])
        ctx = _ScanCtx(covs, 2, 30, False, 2)
        total = hoi.count_nplets(30, 2, 30)
        out = torch.empty((4, total, 1), dtype=torch.float64, device="cuda")
        for _ in range(2):
            ctx.full(0, total, out)
    elif mode == "topk":
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg4()))])
        for _ in range(2):
            hoi.scan(covs, 2, 30, hoi.TopK("o", "min", 1000))
    elif mode == "eval10":
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d)))
                           for d in range(16)])
        idx = workloads.cfg5_nplets(b=1 << 18)
        batch = hoi.NpletBatch(400, indices=idx, check_unique=False)
        for _ in range(2):
            hoi.compute_hoi_batch(covs, batch)
    elif mode == "copula5":
        # BASELINE config 5's copula + covariance stage for all 16 datasets in
        # one batched call of each kernel family (D = 16, T = 1200, N = 400)
        import ctypes
        from paper_2501_03381_b200 import _native as nat
        from paper_2501_03381_b200.copula_core import quantile_grid
        lib = nat.lib()
        x = torch.from_numpy(np.stack([workloads.cfg5_data(d) for d in range(16)])).cuda()
        D, T, N = x.shape
        q = torch.from_numpy(quantile_grid(T)).cuda()
        zt = torch.empty((D, N, T), dtype=torch.float64, device="cuda")
        cov = torch.empty((D, N, N), dtype=torch.float64, device="cuda")
        need = ctypes.c_size_t(0)
        nat.check(lib.hoi_rank_copula_cols(None, T, N, D, None, None, None, None,
                                           ctypes.byref(need), None))
        ws = torch.empty(int(need.value), dtype=torch.uint8, device="cuda")
        s = nat.stream_handle(torch)
        for _ in range(2):
            nat.check(lib.hoi_rank_copula_cols(x.data_ptr(), T, N, D, q.data_ptr(), None,
                                               zt.data_ptr(), ws.data_ptr(), ctypes.byref(need), s))
            nat.check(lib.hoi_covariance_cols(zt.data_ptr(), T, N, D, cov.data_ptr(), s))
    elif mode.startswith("eval") and mode[4:].isdigit():
        import math
        k = int(mode[4:])
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg4()))])
        ctx = _ScanCtx(covs, k, k, False, 1)
        n = math.comb(30, k) // 16
        out = torch.empty((4, n, 1), dtype=torch.float64, device="cuda")
        for _ in range(2):
            ctx.full(0, n, out)
    torch.cuda.synchronize()
    print("ok", mode)


if __name__ == "__main__":
    main(sys.argv[1])
