"""Host-side logic of the drop-in API that needs no GPU: validation,
counts, batch bookkeeping, and the no-fallback guarantee."""

import itertools
import math

import numpy as np
import pytest
import torch

import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _native, scanner


def test_count_and_range_validation():
    assert hoi.count_nplets(30, 3, 30) == 1_073_741_358
    assert hoi.count_nplets(30, 2, 30) == 2**30 - 1 - 30
    for bad in [(5, 0, 3), (5, 3, 2), (5, 2, 6), (0, 1, 1)]:
        with pytest.raises(hoi.InvalidOrderRange):
            hoi.count_nplets(*bad)


def test_nplet_batch_validation_matches_reference_rules():
    with pytest.raises(hoi.InvalidNplet):
        hoi.NpletBatch(4)
    with pytest.raises(hoi.InvalidNplet):
        hoi.NpletBatch(4, indices=np.array([[0, 4]]))
    with pytest.raises(hoi.InvalidNplet):
        hoi.NpletBatch(4, indices=np.array([[2, 1]]))
    with pytest.raises(hoi.InvalidNplet):
        hoi.NpletBatch(4, indices=np.array([[0, 1], [0, 1]]))
    with pytest.raises(hoi.InvalidNplet):
        hoi.NpletBatch(4, masks=np.zeros((1, 4), dtype=bool))
    with pytest.raises(hoi.InvalidNplet):
        hoi.NpletBatch(4, masks=np.ones((1, 4), dtype=np.int64))
    b = hoi.NpletBatch(4, indices=np.array([[0, 1], [0, 1]]), check_unique=False)
    assert b.batch_size == 2
    m = hoi.NpletBatch(5, masks=hoi.NpletBatch(5, indices=np.array([[0, 2, 3]])).to_masks())
    assert m.row_indices(0) == (0, 2, 3)
    with pytest.raises(hoi.InvalidNplet):
        m.order


def test_batch_bounds_follow_reference_batching():
    for n, lo, hi, bs in [(7, 3, 3, 1), (7, 2, 5, 7), (8, 1, 8, 64), (6, 2, 4, 5)]:
        bounds = list(scanner._batch_bounds(n, lo, hi, bs))
        # batches tile the rank space, never cross orders, never exceed bs
        assert bounds[0][0] == 0 and bounds[-1][1] == hoi.count_nplets(n, lo, hi)
        for (a, b, k), (c, _, _) in zip(bounds, bounds[1:]):
            assert b == c
        off = 0
        for k in range(lo, hi + 1):
            mine = [(a, b) for a, b, kk in bounds if kk == k]
            assert all(b - a <= bs for a, b in mine)
            want = [(off + s, off + min(s + bs, math.comb(n, k))) for s in range(0, math.comb(n, k), bs)]
            assert mine == want
            off += math.comb(n, k)


def test_scan_validates_before_touching_the_device():
    covs = hoi.CovSet([hoi.CovarianceMatrix(np.eye(4))])
    with pytest.raises(hoi.InvalidData):
        hoi.scan(covs, 2, 3, reducer=sorted)
    with pytest.raises(hoi.InvalidOrderRange):
        hoi.scan(covs, 3, 9, hoi.TopK("o", "max", 1))
    with pytest.raises(hoi.InvalidData):
        hoi.scan(covs, 2, 3, hoi.TopK("o", "max", 1), workers=0)
    with pytest.raises(hoi.InvalidData):
        hoi.TopK("bogus", "max", 3)
    with pytest.raises(hoi.InvalidData):
        hoi.Histogram("o", 4, 1.0, 1.0)
    with pytest.raises(hoi.ExhaustiveLimitExceeded):
        hoi.extract_features(hoi.CovSet([hoi.CovarianceMatrix(np.eye(21))]))


def test_containers_validate_like_reference():
    with pytest.raises(hoi.InvalidData):
        hoi.DataMatrix(np.zeros(5))
    with pytest.raises(hoi.InsufficientSamples):
        hoi.DataMatrix(np.ones((2, 3)))
    with pytest.raises(hoi.DegenerateColumn):
        hoi.DataMatrix(np.column_stack([np.arange(5.0), np.full(5, 2.0)]))
    with pytest.raises(hoi.InvalidData):
        hoi.CovarianceMatrix(np.array([[1.0, 0.2], [0.1, 1.0]]))
    with pytest.raises(hoi.InvalidData):
        hoi.CovSet([])
    assert hoi.entropy_bias(1, 2) == pytest.approx(-0.6351814227307391, abs=1e-15)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    covs = hoi.CovSet([hoi.CovarianceMatrix(np.eye(4))])
    with pytest.raises(_native.BackendUnavailable):
        hoi.compute_hoi_batch(covs, hoi.NpletBatch(4, indices=np.array([[0, 1, 2]])))
    with pytest.raises(_native.BackendUnavailable):
        hoi.scan(covs, 2, 3, hoi.TopK("o", "max", 1))


def test_lattice_layout_model_matches_oracle(oracle):
    """The lattice engine's table layout, stencil and lexicographic run
    placement (modelled in numpy by tests/lattice_model.py, mirroring
    csrc/lattice.cu) reproduce the reference order and values."""
    import lattice_model as lm
    from paper_2501_03381_b200 import workloads
    rng = np.random.default_rng(5)
    r = workloads.randcorr(12, rng)
    got = lm.measures_full(r, 2, 12)
    rows, vals = oracle.scan(r, [0], 2, 12, oracle.CollectR())
    np.testing.assert_allclose(got, vals[:, :, 0], rtol=1e-9, atol=1e-11)
