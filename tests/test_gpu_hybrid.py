"""Engine 1 at orders 17..22: the bordered one-thread-per-unit kernel
(csrc/eval_hybrid.cu) against the CPU oracle.

test_gpu_parity.py::test_mid_orders_vs_oracle runs these orders with the
correlation matrix staged in shared memory (N = 40); here N = 80 puts R
(102 KB) in global memory, and a duplicated variable drives the jitter
retry (ref nplet_engine.py:237-264).  The every-row cfg4 comparison of
test_gpu_fullrow.py covers the unranking mode at N = 30.  Tolerance: the
FP64 bound, rtol 1e-9 / atol 1e-11 (ref tests/test_acceptance.py:81).
"""

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


def _cov(n, seed):
    rng = np.random.default_rng(seed)
    r = workloads.randcorr(n, rng)
    d = np.sqrt(rng.uniform(0.5, 3.0, n))
    s = r * np.outer(d, d)
    return 0.5 * (s + s.T)


@pytest.mark.parametrize("k", [17, 18, 19, 20, 21, 22, 23])
def test_hybrid_orders_global_R_vs_oracle(oracle, k):
    n, d, t = 80, 2, 1500
    sig = np.stack([_cov(n, 500 + 7 * k + s) for s in range(d)])
    rng = np.random.default_rng(k)
    idx = np.sort(np.stack([rng.choice(n, k, replace=False) for _ in range(400)]), axis=1)
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=t) for s in sig])
    batch = hoi.NpletBatch(n, indices=idx)
    for bias in (False, True):
        h = hoi.compute_hoi_batch(covs, batch, bias_correct=bias)
        want = oracle.hoi_batch(sig, [t] * d, idx=idx, bias=bias)
        np.testing.assert_allclose(np.stack([h.tc, h.dtc, h.o, h.s]), np.stack(want[:4]),
                                   rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("k", [17, 20, 22])
def test_hybrid_duplicated_variable_jitter_retry(oracle, k):
    """Variable 5 is an exact copy of variable 2: every n-plet holding both is
    exactly singular, its first factorisation meets a non-positive pivot and
    the unit reruns with the reference's jittered diagonal.  As for the
    low orders (test_gpu_helpers.py::test_duplicated_variable_...): rows
    without the pair equal the oracle at the FP64 tolerance, singular rows
    are finite and reported near-singular (TC > 5), and healthy rows of
    the same batch are unaffected."""
    n, t = 26, 2000
    rng = np.random.default_rng(40 + k)
    x = rng.standard_normal((t, n)) @ np.linalg.cholesky(workloads.randcorr(n, rng)).T
    x[:, 5] = x[:, 2]
    sig = np.cov(x, rowvar=False)
    sig = 0.5 * (sig + sig.T)
    pool = [np.arange(n), np.delete(np.arange(n), 5), np.delete(np.arange(n), 2)]
    idx = np.sort(np.stack([rng.choice(pool[r % 3], k, replace=False) for r in range(300)]), axis=1)
    idx = np.unique(idx, axis=0)
    combos = [tuple(c) for c in idx]
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig, n_samples_used=t)])
    h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(n, indices=idx))
    got = np.stack([h.tc[:, 0], h.dtc[:, 0], h.o[:, 0], h.s[:, 0]])
    sing = np.array([2 in c and 5 in c for c in combos])
    assert sing.any() and (~sing).any()
    assert np.isfinite(got[:, sing]).all() and (got[0, sing] > 5.0).all()
    want = oracle.hoi_batch(sig[None], [t], idx=idx[~sing])
    np.testing.assert_allclose(got[:, ~sing], np.stack(want[:4])[:, :, 0], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("k", [18, 21])
def test_hybrid_indefinite_rows_fail_after_the_retry(k):
    """An indefinite 2 x 2 block (variables 2 and 5, correlation 1.5): every
    n-plet holding both meets a negative pivot, the jittered retry fails
    too, and the batch raises NotPositiveDefinite with exactly those rows
    (dataset 0) as coordinates (ref nplet_engine.py:237-264, errors.py)."""
    n = 30
    sig = np.eye(n)
    sig[2, 5] = sig[5, 2] = 1.5
    rng = np.random.default_rng(k)
    pool = [np.arange(n), np.delete(np.arange(n), 5)]
    idx = np.unique(np.sort(np.stack([rng.choice(pool[r % 2], k, replace=False)
                                      for r in range(200)]), axis=1), axis=0)
    want = sorted((r, 0) for r, c in enumerate(idx) if 2 in c and 5 in c)
    assert want
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig, n_samples_used=500)])
    with pytest.raises(hoi.NotPositiveDefinite) as err:
        hoi.compute_hoi_batch(covs, hoi.NpletBatch(n, indices=idx))
    assert sorted(tuple(int(v) for v in c) for c in err.value.coords) == want
