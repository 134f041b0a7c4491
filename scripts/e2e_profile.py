"""Stage-by-stage wall-clock breakdown of the public-API e2e call used by
bench.py (diagnostic only)."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2501_03381_b200 as hoi  # noqa: E402
from paper_2501_03381_b200 import _build, scanner, workloads  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main():
    _build.build()
    x = workloads.cfg4()
    for it in range(3):
        t0 = t()
        dm = hoi.DataMatrix(x)
        t1 = t()
        z = hoi.copula_transform(dm)
        t2 = t()
        cov = hoi.estimate_covariance(z)
        t3 = t()
        covs = hoi.CovSet([cov])
        ctx = scanner._ScanCtx(covs, 2, 30, False)
        t4 = t()
        total = hoi.count_nplets(30, 2, 30)
        out, cnt, coords = ctx.full(0, total)
        t5 = t()
        red = hoi.TopK("o", "min", 1000)
        scanner._topk_plane(ctx, red, out, 0, 2)
        t6 = t()
        res = red.finalize()
        t7 = t()
        print(f"iter {it}: data {1e3*(t1-t0):.1f} copula {1e3*(t2-t1):.1f} cov {1e3*(t3-t2):.1f} "
              f"ctx {1e3*(t4-t3):.1f} scan {1e3*(t5-t4):.1f} topk {1e3*(t6-t5):.1f} "
              f"fin {1e3*(t7-t6):.1f} ms; {len(res[0])} entries")
        del out
    import cProfile
    import pstats
    for it in range(3):
        t0 = t()
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(hoi.DataMatrix(x)))])
        t1 = t()
        pr = cProfile.Profile() if it == 2 else None
        if pr:
            pr.enable()
        res = hoi.scan(covs, 2, 30, hoi.TopK("o", "min", 1000))
        t2 = t()
        if pr:
            pr.disable()
            pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
        print(f"public api iter {it}: covs {1e3*(t1-t0):.1f} ms scan+topk {1e3*(t2-t1):.1f} ms "
              f"({len(res[0])} entries)")


if __name__ == "__main__":
    main()
