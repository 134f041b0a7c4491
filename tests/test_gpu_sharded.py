"""The multi-GPU path on the device (-m gpu): two ranks in two processes
share the one GPU of the test box over gloo (the data path is the same
device code; NCCL replaces gloo on a multi-GPU node).  Every reducer and the
FULL output, merged across the ranks, must equal the single-GPU scan bit for
bit (ref:scanner.py:290-305: an ordered merge leaves no trace of the
partition).  Each rank's kernels are independent -- no rank waits on
another's kernel -- so sharing one GPU is a correctness run, not a timing."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _covs(n, seed, d=1):
    import paper_2501_03381_b200 as hoi
    rng = np.random.default_rng(seed)
    cs = []
    for _ in range(d):
        a = rng.standard_normal((3 * n, n))
        s = a.T @ a / (3 * n) + 0.2 * np.eye(n)
        cs.append(hoi.CovarianceMatrix(0.5 * (s + s.T), n_samples_used=3 * n))
    return hoi.CovSet(cs)


CASES = [(18, 2, 18, 1), (18, 3, 9, 2), (14, 2, 14, 1), (10, 2, 10, 1)]   # (N, lo, hi, D)


def _worker(rank, world, port, q, tmpdir):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    import paper_2501_03381_b200 as hoi
    from paper_2501_03381_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        for n, lo, hi, d in CASES:
            covs = _covs(n, 100 + n + d, d)
            key = f"{n}_{lo}_{hi}_{d}"
            sh = sharding.scan_sharded(covs, lo, hi, None)
            full = sh.gather(0)
            saved = sh.save(os.path.join(tmpdir, f"{key}.scan"), dst=0)
            top = sharding.scan_sharded(covs, lo, hi, hoi.TopK("o", "min", 25))
            hist = sharding.scan_sharded(covs, lo, hi, hoi.Histogram("tc", 16, 0.0, 2.0))
            feats = None
            if lo == 2 and hi == n:
                feats = sharding.scan_sharded(covs, 2, n, hoi.FeatureAccumulator(n))
            if rank == 0:
                single = hoi.scan_device(covs, lo, hi).out
                res[key] = {
                    "kind": sh.kind,
                    "full_equal": bool(torch.equal(full.out, single)),
                    "save_equal": bool(np.array_equal(hoi.read_scan(saved)[1],
                                                      single.cpu().numpy())),
                    "local_rows": [sh.local_rows],
                    "top": [[(e.indices, e.o) for e in per] for per in top],
                    "top_single": [[(e.indices, e.o) for e in per]
                                   for per in hoi.scan(covs, lo, hi, hoi.TopK("o", "min", 25))],
                    "hist": [c.tolist() for c in hist[1]],
                    "hist_single": [c.tolist() for c in
                                    hoi.scan(covs, lo, hi, hoi.Histogram("tc", 16, 0.0, 2.0))[1]],
                }
                if feats is not None:
                    single_f = hoi.extract_features(covs, limit=n)
                    res[key]["feat"] = [f.as_dict() for f in feats]
                    res[key]["feat_single"] = [f.as_dict() for f in single_f]
            else:
                res[key] = {"local_rows": [sh.local_rows]}
        q.put((rank, res))
    except Exception as e:   # surface the failure to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
        raise e
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_on_one_gpu_equal_the_single_gpu_scan(tmp_path):
    import math
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        assert "error" not in got[r], got[r].get("error")
    for p in procs:
        assert p.exitcode == 0
    for n, lo, hi, d in CASES:
        key = f"{n}_{lo}_{hi}_{d}"
        r0 = got[0][key]
        assert r0["kind"] == ("blocks" if n >= 17 else "ranges")
        assert r0["full_equal"], key
        assert r0["save_equal"], key            # ShardedScan.save = the single-GPU scan file
        assert r0["top"] == r0["top_single"], key
        assert r0["hist"] == r0["hist_single"], key
        if "feat" in r0:
            assert r0["feat"] == r0["feat_single"], key
        # no rank holds the whole output: compact shards
        rows = r0["local_rows"][0] + got[1][key]["local_rows"][0]
        if r0["kind"] == "blocks":
            assert rows == 1 << n                    # 1024 slots per table block, holes included
        else:
            assert rows == sum(math.comb(n, k) for k in range(lo, hi + 1))
