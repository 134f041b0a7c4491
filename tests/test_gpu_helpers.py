"""Public helpers around the hot path, the radix select's exactness, and
the singular-input behaviour, on the device (-m gpu).

Golden vectors: tests/golden/helpers.npz, written by
tests/golden/make_golden_helpers.py from the real reference.
"""

import itertools
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, _native

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-9, 1e-11
H = np.load(Path(__file__).resolve().parent / "golden" / "helpers.npz")


@pytest.fixture(scope="module", autouse=True)
def device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _build.build()
    _native.load()
    yield


def _covs():
    return hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=40) for s in H["sig"]])


# ---------------------------------------------- ref nplet_engine.py:185-224

def test_extract_subcov_batch_equals_reference():
    sub = hoi.extract_subcov_batch(_covs(), hoi.NpletBatch(7, indices=H["idx"]))
    assert sub.matrices.shape == H["sub"].shape
    assert np.array_equal(sub.matrices, H["sub"])              # a gather: bit-exact
    assert np.array_equal(sub.pad_counts, H["sub_pad"])
    with pytest.raises(hoi.InvalidNplet):
        hoi.extract_subcov_batch(_covs(), hoi.NpletBatch(7, masks=H["masks"]))
    with pytest.raises(hoi.InvalidNplet):
        hoi.extract_subcov_batch(_covs(), hoi.NpletBatch(8, indices=np.array([[0, 7]])))


def test_pad_subcov_batch_equals_reference():
    pad = hoi.pad_subcov_batch(_covs(), hoi.NpletBatch(7, masks=H["masks"]))
    assert pad.matrices.shape == H["pad"].shape
    assert np.array_equal(pad.matrices, H["pad"])
    assert np.array_equal(pad.pad_counts, H["pad_counts"])
    with pytest.raises(hoi.InvalidNplet):
        hoi.pad_subcov_batch(_covs(), hoi.NpletBatch(7, indices=H["idx"]))


# ------------------------------- ref copula_core.py:207-260, measures.py:84-99

def test_gaussian_entropy_nats_equals_reference():
    for s, want in zip(H["sig"], H["ent"]):
        got = hoi.gaussian_entropy_nats(hoi.CovarianceMatrix(s))
        assert got.nats == pytest.approx(want, rel=1e-12)
        assert got.bias_corrected is False
    # indefinite by 1e-12: the plain factorisation fails and the jitter
    # retry (eps = 1e-10 trace / n) rescues it, as in the reference.  The
    # rescued pivot (~2e-10) comes out of an O(1) cancellation, so it is only
    # defined to ~1e-6 relative in any summation order: rel 1e-6 here.
    got = hoi.gaussian_entropy_nats(hoi.CovarianceMatrix(H["rankdef"])).nats
    assert got == pytest.approx(float(H["ent_jit"]), rel=1e-6)
    with pytest.raises(hoi.NotPositiveDefinite):
        hoi.gaussian_entropy_nats(hoi.CovarianceMatrix(np.array([[1.0, 2.0], [2.0, 1.0]])))


def test_copula_entropy_equals_reference():
    for b, want in zip((False, True), H["ce"]):
        got = hoi.copula_entropy(hoi.DataMatrix(H["x"]), bias_correct=b)
        assert got.nats == pytest.approx(want, rel=1e-10)
        assert got.bias_corrected is b


def test_pairwise_mi_equals_reference():
    c = _covs().covs[0]
    for (i, j), want in zip(H["mi_pairs"], H["mi"]):
        for b, w in zip((False, True), want):
            assert hoi.pairwise_mi(c, int(i), int(j), bias_correct=b) == pytest.approx(
                w, rel=RTOL, abs=ATOL)
    with pytest.raises(hoi.InvalidNplet):
        hoi.pairwise_mi(c, 2, 2)
    with pytest.raises(hoi.InvalidNplet):
        hoi.pairwise_mi(c, 0, 7)


def test_ground_truth_hoi_equals_reference():
    cov = hoi.CovarianceMatrix(H["gt_sigma"])
    for mask, want in zip(H["gt_nplets"], H["gt"]):
        t = [i for i in range(8) if (int(mask) >> i) & 1]
        got = hoi.ground_truth_hoi(cov, t[::-1])                 # order-insensitive
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    with pytest.raises(hoi.InvalidNplet):
        hoi.ground_truth_hoi(cov, [1, 1])
    with pytest.raises(hoi.InvalidNplet):
        hoi.ground_truth_hoi(cov, [])


# ------------------------------------------------- singular covariances --

def test_duplicated_variable_divergence_is_confined_to_singular_rows():
    """x3 == x1: every n-plet holding both is exactly singular.  The
    reference's LAPACK Cholesky fails on (most of) them and its jitter
    retry returns log(eps)-scale values (TC ~ 11); which rows fail and the
    exact values are decided by rounding, so the GPU is held to: every
    n-plet without the pair equals the reference at the FP64 tolerance,
    every singular one is finite and reported as (near-)singular (TC > 5).
    DESIGN.md §2 documents this."""
    covs = hoi.CovSet([hoi.CovarianceMatrix(H["dup_sigma"])])
    rows = [c for k in range(2, 6) for c in itertools.combinations(range(5), k)]
    idx_by_k = {}
    for r, c in enumerate(rows):
        idx_by_k.setdefault(len(c), []).append((r, c))
    want = H["dup_vals"]
    for k, items in idx_by_k.items():
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(5, indices=np.array([c for _, c in items])))
        got = np.stack([h.tc[:, 0], h.dtc[:, 0], h.o[:, 0], h.s[:, 0]])
        for j, (r, c) in enumerate(items):
            if 1 in c and 3 in c:
                assert np.isfinite(got[:, j]).all() and got[0, j] > 5.0, c
            else:
                np.testing.assert_allclose(got[:, j], want[:, r], rtol=RTOL, atol=ATOL)


# ----------------------------------------------------- radix selection --

def _okey(v):
    """The kernels' orderable key (csrc/common.cuh orderable_key)."""
    v = np.where(v == 0.0, 0.0, v)
    b = v.view(np.uint64)
    neg = (b >> np.uint64(63)) == 1
    return np.where(neg, ~b, b | np.uint64(1 << 63))


def test_topk_threshold_is_the_exact_kth_key():
    """hoi_topk_threshold against numpy's sorted orderable keys, on values
    whose keys share long prefixes (the last 4-bit radix round decides)."""
    rng = np.random.default_rng(11)
    lib, s = _native.lib(), _native.stream_handle(torch)
    ws = torch.empty(4096 + 64, dtype=torch.int64, device="cuda")
    key = torch.empty(1, dtype=torch.int64, device="cuda")
    for case in range(60):
        n, D = int(rng.integers(100, 20000)), int(rng.integers(1, 4))
        base = rng.standard_normal()
        kind = case % 3
        if kind == 0:
            v = rng.standard_normal((n, D))
        elif kind == 1:      # values a few ulps apart: keys differ only in low bits
            v = base + rng.integers(-300, 300, (n, D)) * np.spacing(abs(base))
        else:                # many exact ties plus spread
            v = np.where(rng.random((n, D)) < 0.5, base, rng.standard_normal((n, D)))
        d = int(rng.integers(0, D))
        sign = float(rng.choice([-1.0, 1.0]))
        k = int(rng.integers(1, n))
        t = torch.as_tensor(np.ascontiguousarray(v), device="cuda")
        _native.check(lib.hoi_topk_threshold(t.data_ptr(), n, D, d, sign, k, key.data_ptr(),
                                             ws.data_ptr(), s), "threshold")
        got = int(key.item()) & (2 ** 64 - 1)
        want = int(np.sort(_okey(sign * v[:, d]))[k - 1])
        assert got == want, (case, kind, n, k)


def test_topk_select_keeps_every_tie_beyond_the_bucket_cap():
    """5,000 exact non-zero ties at the k-th key (more than the 4,096-entry
    bucket cap): the candidate set must hold the k smallest keys and every
    tie at the k-th, or report a count above capacity for the host rule."""
    rng = np.random.default_rng(5)
    n = 40000
    v = rng.standard_normal(n)
    tie = 0.731
    v[rng.choice(n, 5000, replace=False)] = tie
    lib, s = _native.lib(), _native.stream_handle(torch)
    t = torch.as_tensor(v, device="cuda")
    ws = torch.empty(4096 + 64, dtype=torch.int64, device="cuda")
    for k in (10, 3000, 19000):
        kth = np.sort(v)[k - 1]
        cap = k + 12000
        cand = torch.empty(cap, dtype=torch.int64, device="cuda")
        import ctypes
        cnt = ctypes.c_int64(0)
        _native.check(lib.hoi_topk_select(t.data_ptr(), n, 1, 0, 1.0, k, 4096, cand.data_ptr(),
                                          cap, ctypes.byref(cnt), ws.data_ptr(), s), "select")
        c = int(cnt.value)
        must = set(np.flatnonzero(v <= kth).tolist())
        if c <= cap:
            got = set(cand[:c].cpu().numpy().tolist())
            assert must <= got, k
        else:
            assert c >= len(must)


def test_topk_batch_with_wide_exact_ties():
    """Exchangeable covariance: every order-6 n-plet of N = 16 has the same
    sub-matrix, so the per-n-plet engine gives bit-identical values for all
    8,008 rows and the reference's key falls back to the index tuple: the
    first k tuples in lexicographic order."""
    n, rho = 16, 0.35
    sig = np.full((n, n), rho) + (1 - rho) * np.eye(n)
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig)])
    idx = np.array(list(itertools.combinations(range(n), 6)))[::-1].copy()   # reversed rows
    batch = hoi.NpletBatch(n, indices=idx)
    h = hoi.compute_hoi_batch(covs, batch)
    assert (h.o == h.o[0, 0]).all() and h.o[0, 0] != 0.0
    for direction in ("max", "min"):
        got = hoi.topk_batch(covs, batch, hoi.TopK("o", direction, 10)).finalize()[0]
        want = sorted(tuple(r) for r in idx)[:10]
        assert [e.indices for e in got] == want


# ------------------------------------------- beyond the unranking table --

LARGE = np.load(Path(__file__).resolve().parent / "golden" / "large.npz")
LARGE_J = __import__("json").loads(
    (Path(__file__).resolve().parent / "golden" / "large.json").read_text())


def _large_covs():
    return hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=500) for s in LARGE["sigma"]])


def test_enumerate_order_beyond_64_variables():
    got = list(hoi.enumerate_order(70, 2, batch_size=1000))
    assert [b.batch_size for b in got] == [1000, 1000, 415]
    rows = np.concatenate([b.indices for b in got])
    assert [tuple(r) for r in rows] == list(itertools.combinations(range(70), 2))
    first = next(hoi.enumerate_order(100, 4, batch_size=5))
    assert [tuple(r) for r in first.indices] == list(itertools.islice(
        itertools.combinations(range(100), 4), 5))


def test_scan_topk_beyond_64_variables_equals_reference():
    got = hoi.scan(_large_covs(), 2, 3, hoi.TopK("o", "min", 12))
    for per, want in zip(got, LARGE_J["scan_top"]):
        assert [list(e.indices) for e in per] == [w[0] for w in want]
        np.testing.assert_allclose([[e.value, e.tc, e.dtc, e.o, e.s] for e in per],
                                   [w[1:] for w in want], rtol=RTOL, atol=ATOL)


def test_scan_device_beyond_64_variables(oracle):
    covs = _large_covs()
    n = 100
    total = hoi.count_nplets(n, 2, 3)
    dev = hoi.scan_device(covs, 2, 3, g_begin=4000, g_end=total)
    rows = list(itertools.islice(itertools.chain(itertools.combinations(range(n), 2),
                                                 itertools.combinations(range(n), 3)), 4000, None))
    pick = np.random.default_rng(0).choice(len(rows), 500, replace=False)
    got = dev.out[:, torch.as_tensor(pick, device="cuda")].cpu().numpy()
    for k in (2, 3):
        sel = [i for i in pick if len(rows[i]) == k]
        pos = [int(np.flatnonzero(pick == i)[0]) for i in sel]
        tc, dtc, o, s, _ = oracle.hoi_batch(covs.stacked(), [500, 500],
                                            idx=np.array([rows[i] for i in sel]))
        np.testing.assert_allclose(got[:, pos], np.stack([tc, dtc, o, s]), rtol=RTOL, atol=ATOL)


def test_greedy_and_anneal_beyond_64_variables_equal_reference():
    covs = _large_covs()
    spec = hoi.ObjectiveSpec("o", "max")
    g = hoi.greedy(covs, spec, 3, 5, kappa=4)
    for e, w in zip(g.per_order, LARGE_J["greedy"]):
        assert (e.order, list(e.indices)) == (w[0], w[1])
        assert e.energy == pytest.approx(w[2], rel=RTOL, abs=ATOL)
    st = hoi.anneal(covs, spec, hoi.AnnealSchedule(max_iters=40, min_order=3, max_order=8),
                    kappa=6, seed=1)
    w = LARGE_J["anneal"]
    assert list(st.best_indices) == w["best_indices"] and st.iterations == w["iterations"]
    np.testing.assert_allclose(st.energies, w["energies"], rtol=RTOL, atol=ATOL)


def test_device_objective_sums_in_numpys_order():
    """hoi_objective's mean and paired Cohen's d equal the reference's
    vals.mean(axis=1) and diff.mean / diff.std(ddof=1) bit for bit
    (ref:optimizers.py:74-102) for D from 1 to 150 -- numpy sums the
    C-ordered plane pairwise and the list-indexed (column-major) diff
    sequentially -- so near-tied energies order as in the reference."""
    lib, s = _native.lib(), _native.stream_handle(torch)
    rng = np.random.default_rng(21)
    for d in list(range(1, 40)) + [64, 100, 129, 150]:
        vals = rng.standard_normal((257, d)) * 10.0 ** rng.uniform(-4, 4, (257, d))
        v = torch.as_tensor(vals, device="cuda")
        energy = torch.empty(257, dtype=torch.float64, device="cuda")
        degen = torch.zeros(1, dtype=torch.int32, device="cuda")
        _native.check(lib.hoi_objective(v.data_ptr(), 257, d, 0, None, None, 0, -1.0,
                                        energy.data_ptr(), degen.data_ptr(), s), "objective")
        assert np.array_equal(energy.cpu().numpy(), -vals.mean(axis=1)), d
        if d >= 4:
            a_idx = np.arange(0, d // 2, dtype=np.int32)
            b_idx = np.arange(d // 2, 2 * (d // 2), dtype=np.int32)
            ca, cb = torch.as_tensor(a_idx, device="cuda"), torch.as_tensor(b_idx, device="cuda")
            _native.check(lib.hoi_objective(v.data_ptr(), 257, d, 1, ca.data_ptr(), cb.data_ptr(),
                                            len(a_idx), 1.0, energy.data_ptr(), degen.data_ptr(),
                                            s), "objective")
            diff = vals[:, list(a_idx)] - vals[:, list(b_idx)]     # as the reference builds it
            want = diff.mean(axis=1) / diff.std(axis=1, ddof=1)
            assert np.array_equal(energy.cpu().numpy(), want), d


# ------------------------------------------------- device TopK results --

def test_topk_entries_behave_like_the_reference_lists():
    """topk_batch's lazy TopEntries: equal to the host reducer's lists,
    indexable, sliceable, and a later update() merges exactly as the
    reference's TopK would (the compact state is materialised first)."""
    rng = np.random.default_rng(8)
    n = 24
    a = rng.standard_normal((3 * n, n))
    sig = a.T @ a / (3 * n) + 0.3 * np.eye(n)
    covs = hoi.CovSet([hoi.CovarianceMatrix(0.5 * (sig + sig.T)), hoi.CovarianceMatrix(np.eye(n))])
    idx1 = np.array(sorted({tuple(sorted(rng.choice(n, 6, replace=False))) for _ in range(3000)}))
    idx2 = np.array(sorted({tuple(sorted(rng.choice(n, 6, replace=False))) for _ in range(3000)}))
    b1, b2 = hoi.NpletBatch(n, indices=idx1), hoi.NpletBatch(n, indices=idx2)
    dev = hoi.topk_batch(covs, b1, hoi.TopK("s", "max", 40))
    got = dev.finalize()
    host = hoi.TopK("s", "max", 40)
    host.update(b1, hoi.compute_hoi_batch(covs, b1))
    want = host.finalize()
    for g, w in zip(got, want):
        assert len(g) == len(w) == 40
        assert g == w and list(g) == w
        assert g[0] == w[0] and g[-1] == w[-1] and g[3:7] == w[3:7]
    dev.update(b2, hoi.compute_hoi_batch(covs, b2))
    host.update(b2, hoi.compute_hoi_batch(covs, b2))
    assert dev.finalize() == host.finalize()
    # fewer rows than k: every row, in the reference's order
    few = hoi.NpletBatch(n, indices=idx1[:5])
    small = hoi.topk_batch(covs, few, hoi.TopK("o", "min", 10)).finalize()
    ref = hoi.TopK("o", "min", 10)
    ref.update(few, hoi.compute_hoi_batch(covs, few))
    assert small == ref.finalize() and all(len(s) == 5 for s in small)


def test_streamed_batch_reports_not_pd_rows_across_chunks():
    """A 2M-row order-10 batch (streamed to the device in 512k-row chunks)
    over a covariance whose variables 0 and 1 form an indefinite pair: every
    row holding both fails the jitter retry, and NotPositiveDefinite names
    (row, dataset) coordinates of such rows in every chunk they occur."""
    n = 20
    sig = np.eye(n)
    sig[0, 1] = sig[1, 0] = 2.0
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig)])
    rng = np.random.default_rng(3)
    idx = np.sort(np.argsort(rng.random((2_000_000, n)), axis=1)[:, :10], axis=1)
    bad = np.flatnonzero((idx == 0).any(axis=1) & (idx == 1).any(axis=1))
    with pytest.raises(hoi.NotPositiveDefinite) as ei:
        hoi.compute_hoi_batch(covs, hoi.NpletBatch(n, indices=idx, check_unique=False))
    coords = ei.value.coords
    assert coords and all(d == 0 for _, d in coords)
    rows = np.array([r for r, _ in coords])
    assert np.isin(rows, bad).all()
    assert len({int(r) // (1 << 19) for r in rows}) >= 2      # coordinates from several chunks
