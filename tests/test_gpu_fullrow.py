"""Every-row checks of the two largest BASELINE configurations (-m gpu).

* cfg4 (N = 30, orders 2..30): the subset-lattice engine (engine 2, the
  headline path) against the per-n-plet engine (engine 1, the north-star
  batched LDL^T, itself pinned to the reference at sampled ranks in
  test_gpu_parity) over all 1,073,741,793 rows and all four measures:
  max(|a - b| - 1e-9 |b|) <= 1e-11 (the FP64 tolerance, rtol 1e-9 /
  atol 1e-11, ref tests/test_acceptance.py:81) reduced on the device.
* cfg5 (D = 16, N = 400, 4M order-10 n-plets, TopK('o', 'min', 1000)):
  every returned entry re-evaluated by the CPU oracle, and a 200,000-row
  uniform sample evaluated by the oracle must not hold an n-plet that
  beats a dataset's 1000-th entry yet is missing from its list.
"""

import math

import numpy as np
import pytest
import torch

import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, _native, workloads

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-9, 1e-11


@pytest.fixture(scope="module", autouse=True)
def device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _build.build()
    _native.load()
    yield


def test_cfg4_lattice_equals_per_nplet_engine_on_every_row(golden):
    g = golden.npz("cfg4")
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"], n_samples_used=int(g["t"]))])
    total = hoi.count_nplets(30, 2, 30)
    for bias in (False, True):
        lat = hoi.scan_device(covs, 2, 30, engine=2, bias_correct=bias).out
        per = hoi.scan_device(covs, 2, 30, engine=1, bias_correct=bias).out
        assert lat.shape == per.shape == (4, total, 1)
        worst = -math.inf
        step = 1 << 26
        for m in range(4):
            for a in range(0, total, step):
                x = lat[m, a:a + step, 0]
                y = per[m, a:a + step, 0]
                excess = (x - y).abs() - RTOL * y.abs()
                worst = max(worst, float(excess.max()))
        assert worst <= ATOL, (bias, worst)
        del lat, per
        torch.cuda.empty_cache()


def test_cfg5_topk_every_entry_and_a_uniform_sample_against_the_oracle(oracle):
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d)))
                       for d in range(16)])
    sig = covs.stacked()
    idx = workloads.cfg5_nplets()
    k = 1000
    top = hoi.topk_batch(covs, hoi.NpletBatch(400, indices=idx), hoi.TopK("o", "min", k)).finalize()
    assert len(top) == 16 and all(len(t) == k for t in top)
    # every returned entry, re-evaluated on the CPU
    for d, entries in enumerate(top):
        rows = np.array([e.indices for e in entries])
        tc, dtc, o, s, _ = oracle.hoi_batch(sig[d:d + 1], [1200], idx=rows)
        got = np.array([[e.tc, e.dtc, e.o, e.s] for e in entries]).T
        np.testing.assert_allclose(got, np.stack([tc[:, 0], dtc[:, 0], o[:, 0], s[:, 0]]),
                                   rtol=RTOL, atol=ATOL)
        assert [e.value for e in entries] == [e.o for e in entries]
        vals = [e.value for e in entries]
        assert vals == sorted(vals)
    # a uniform sample of the 4M rows: nothing the oracle ranks ahead of a
    # dataset's k-th entry may be missing from that dataset's list
    pick = np.random.default_rng(9).choice(idx.shape[0], 200_000, replace=False)
    o_s = np.concatenate([oracle.hoi_batch(sig, [1200] * 16, idx=idx[pick[a:a + 25_000]])[2]
                          for a in range(0, pick.size, 25_000)])
    for d, entries in enumerate(top):
        kth = entries[-1].o
        listed = {e.indices for e in entries}
        better = np.flatnonzero(o_s[:, d] < kth - (RTOL * abs(kth) + ATOL))
        missing = [tuple(int(v) for v in idx[pick[i]]) for i in better
                   if tuple(int(v) for v in idx[pick[i]]) not in listed]
        assert not missing, (d, missing[:3])
