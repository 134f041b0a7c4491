"""CUDA path vs the reference's golden vectors and the CPU oracle.

Tolerances: measures rtol 1e-9 / atol 1e-11 (the reference's own
acceptance tolerance, ref tests/test_acceptance.py:81 and the north_star's
FP64 bound); covariance rtol 1e-12; ranks, copula values, enumeration
and n-plet order bit-exact.
"""

import itertools
import math

import numpy as np
import pytest
import torch

import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import _build, _native, workloads
from paper_2501_03381_b200.nplet_engine import _batched_logdet_invdiag, unrank_device

import hoi_oracle as ora  # checker only (analytic R/S fixtures)

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-9, 1e-11


@pytest.fixture(scope="module", autouse=True)
def device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _build.build()
    _native.load()
    yield


def collect(covs, lo, hi, bias=False, batch_size=10000):
    rows, vals = [], []

    def keep(batch, h):
        rows.extend(batch.row_indices(i) for i in range(batch.batch_size))
        vals.append(np.stack([h.tc, h.dtc, h.o, h.s]))

    hoi.scan(covs, lo, hi, hoi.Callback(keep), batch_size=batch_size, bias_correct=bias)
    return rows, np.concatenate(vals, axis=1)


# ------------------------------------------------------------ copula ----

def test_rank_copula_bit_exact(golden):
    g = golden.npz("copula")
    np.testing.assert_array_equal(hoi.rank_columns(g["x"]), g["ranks"])
    np.testing.assert_array_equal(hoi.copula_transform(hoi.DataMatrix(g["x"])).values, g["z"])
    np.testing.assert_array_equal(hoi.rank_columns(g["tie"])[:, 0], [3, 1, 4, 2])
    cov = hoi.estimate_covariance(hoi.copula_transform(g["x"]))
    np.testing.assert_allclose(cov.sigma, g["cov"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(cov.sigma, cov.sigma.T)
    assert cov.n_samples_used == 40


def test_copula_multichunk_with_ties(golden):
    import hashlib
    g = golden.npz("cfg3")
    x = workloads.cfg3()                       # T = 10,000 > one 8192-row chunk, 13 ties
    r = hoi.rank_columns(x)
    assert hashlib.sha256(np.ascontiguousarray(r).tobytes()).hexdigest() == str(g["ranks_sha"])
    cov = hoi.estimate_covariance(hoi.copula_transform(x))
    np.testing.assert_allclose(cov.sigma, g["cov"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(cov.sigma, cov.sigma.T)


def test_copula_monotone_invariance_and_cfg4(golden):
    x = workloads.cfg4()
    z = hoi.copula_transform(x).values
    np.testing.assert_array_equal(hoi.copula_transform(np.exp(x / 10.0)).values, z)
    cov = hoi.estimate_covariance(hoi.copula_transform(x))
    np.testing.assert_allclose(cov.sigma, golden.npz("cfg4")["cov"], rtol=1e-12, atol=1e-15)


# -------------------------------------------------------- enumeration ---

def test_unranking_is_itertools_order():
    for n, lo, hi in [(12, 1, 12), (7, 3, 3), (20, 18, 20)]:
        total = hoi.count_nplets(n, lo, hi)
        idx, orders = unrank_device(n, lo, hi, 0, total)
        idx, orders = idx.cpu().numpy(), orders.cpu().numpy()
        want = [c for k in range(lo, hi + 1) for c in itertools.combinations(range(n), k)]
        got = [tuple(int(v) for v in idx[i, :orders[i]]) for i in range(total)]
        assert got == want
    # 64-variable edges (largest binomials in the table)
    for k in (1, 2, 63, 64):
        c = math.comb(64, k)
        idx, _ = unrank_device(64, k, k, c - 1, 1)
        assert tuple(idx[0].tolist()) == tuple(range(64 - k, 64))


def test_enumerate_order_batches():
    got = []
    for batch in hoi.enumerate_order(7, 3, batch_size=4):
        assert batch.batch_size <= 4
        got.extend(batch.row_indices(i) for i in range(batch.batch_size))
    assert got == list(itertools.combinations(range(7), 3))


# ------------------------------------------------------ full scans ------

@pytest.mark.parametrize("batch_size", [7, 10000])
def test_cfg1_full_scan(golden, batch_size):
    g = golden.npz("cfg1")
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(g["x"]))])
    rows, vals = collect(covs, 3, 10, batch_size=batch_size)
    assert rows == [c for k in range(3, 11) for c in itertools.combinations(range(10), k)]
    np.testing.assert_allclose(vals[:, :, 0], g["vals"], rtol=RTOL, atol=ATOL)
    np.testing.assert_array_equal(vals[3], vals[0] + vals[1])      # s == tc + dtc exactly


def test_cfg2_full_scan_with_bias(golden):
    g = golden.npz("cfg2")
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"], n_samples_used=int(g["t"]))])
    _, vals = collect(covs, 3, 12, bias=True)
    np.testing.assert_allclose(vals[:, :, 0], g["vals"], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("cfg,lo,hi", [("cfg3", 3, 20), ("cfg4", 2, 30)])
@pytest.mark.parametrize("bias", [False, True])
def test_sampled_ranks_batched_and_scanned(golden, cfg, lo, hi, bias):
    g = golden.npz(cfg)
    key = "vals_bias" if bias else "vals"
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"], n_samples_used=int(g["t"]))])
    rows = [tuple(int(v) for v in r if v >= 0) for r in g["idx"]]
    by_k = {}
    for i, t in enumerate(rows):
        by_k.setdefault(len(t), []).append(i)
    got = np.empty_like(g[key])
    for k, sel in by_k.items():
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(covs.n_variables,
                                                       indices=np.array([rows[i] for i in sel])),
                                  bias_correct=bias)
        got[:, sel, :] = np.stack([h.tc, h.dtc, h.o, h.s])
    np.testing.assert_allclose(got, g[key], rtol=RTOL, atol=ATOL)
    if cfg == "cfg3":   # whole 1,048,365-row scan on the device, checked at the sampled ranks
        dev = hoi.scan_device(covs, lo, hi, bias_correct=bias)
        out = dev.out[:, torch.as_tensor(g["g"], device="cuda"), :].cpu().numpy()
        np.testing.assert_allclose(out, g[key], rtol=RTOL, atol=ATOL)


def test_cfg4_full_exhaustive_scan(golden):
    """The headline configuration: all 1,073,741,793 n-plets of orders 2..30."""
    g = golden.npz("cfg4")
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"], n_samples_used=int(g["t"]))])
    dev = hoi.scan_device(covs, 2, 30)
    out = dev.out
    assert out.shape == (4, hoi.count_nplets(30, 2, 30), 1)
    sel = torch.as_tensor(g["g"], device="cuda")
    np.testing.assert_allclose(out[:, sel, :].cpu().numpy(), g["vals"], rtol=RTOL, atol=ATOL)
    # size-independent properties over every row
    assert bool(torch.isfinite(out).all())
    assert bool((out[3] == out[0] + out[1]).all())
    n2 = math.comb(30, 2)
    assert float(out[2, :n2].abs().max()) < 1e-12                # O = 0 at order 2
    assert bool((out[0] >= -1e-12).all())                        # TC >= 0
    del out, dev
    torch.cuda.empty_cache()


# ------------------------------------------------------------- edges ----

def test_identity_exact_zeros_and_closed_forms(golden):
    e = golden.npz("edge")
    covs = hoi.CovSet([hoi.CovarianceMatrix(np.eye(6))])
    for k in (2, 3, 4, 6):
        idx = np.array(list(itertools.combinations(range(6), k)))
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(6, indices=idx))
        for m in (h.tc, h.dtc, h.o, h.s):
            assert (m == 0.0).all()
    for m in (2, 3, 4):
        for kind, fn in (("r", ora.r_system), ("s", ora.s_system)):
            cov = hoi.CovarianceMatrix(fn(m, 1.0))
            h = hoi.compute_hoi_batch(hoi.CovSet([cov]),
                                      hoi.NpletBatch(m + 1, indices=np.arange(m + 1)[None]))
            np.testing.assert_allclose([h.tc[0, 0], h.dtc[0, 0], h.o[0, 0], h.s[0, 0]],
                                       e[f"rs_{kind}{m}"], atol=1e-13)
    r2 = e["rs_r2"]
    assert r2[0] == pytest.approx(math.log(2.0), abs=1e-14)
    assert r2[2] == pytest.approx(0.5 * math.log(4.0 / 3.0), abs=1e-14)


def test_not_pd_coords_and_jitter(golden):
    e = golden.npz("edge")
    bad = np.array([[1.0, 2.0], [2.0, 1.0]])
    with pytest.raises(hoi.NotPositiveDefinite) as err:
        _batched_logdet_invdiag(np.stack([np.eye(2), bad])[:, None])
    assert [list(c) for c in err.value.coords] == golden.meta["edge"]["npd_coords"]
    ld, idg = _batched_logdet_invdiag((np.ones((3, 3)) + np.eye(3) * 1e-14)[None, None])
    # ones + 1e-14 I factors with ~1e-14 pivots on both sides (no jitter
    # needed); those pivots carry ~1% rounding, so only finiteness and the
    # magnitude are comparable (the reference test asserts finiteness)
    assert np.isfinite(ld).all()
    assert abs(ld[0, 0] - e["singular_ld"][0, 0]) < 0.1
    # healthy matrices are unaffected by a failing neighbour (bit-identical)
    rng = np.random.default_rng(3)
    a = rng.standard_normal((8, 3))
    good = (a.T @ a / 8 + 0.5 * np.eye(3))[None, None]
    stack = np.concatenate([good, (np.ones((3, 3)) + np.eye(3) * 1e-14)[None, None]])
    l1, i1 = _batched_logdet_invdiag(stack)
    l0, i0 = _batched_logdet_invdiag(good)
    assert l1[0, 0] == l0[0, 0]
    np.testing.assert_array_equal(i1[0, 0], i0[0, 0])


def test_logdet_invdiag_vs_slogdet():
    rng = np.random.default_rng(2)
    mats = np.empty((4, 3, 5, 5))
    for b in range(4):
        for d in range(3):
            a = rng.standard_normal((8, 5))
            mats[b, d] = a.T @ a / 8 + 0.3 * np.eye(5)
    ld, idg = _batched_logdet_invdiag(mats)
    for b in range(4):
        for d in range(3):
            assert ld[b, d] == pytest.approx(np.linalg.slogdet(mats[b, d])[1], rel=1e-10)
            np.testing.assert_allclose(idg[b, d], np.diag(np.linalg.inv(mats[b, d])), rtol=1e-10)


def test_mixed_masks_and_terms(golden):
    e = golden.npz("edge")
    covs = hoi.CovSet([hoi.CovarianceMatrix(e["mix_sigma"])])
    batch = hoi.NpletBatch(15, masks=e["mix_masks"])
    h = hoi.compute_hoi_batch(covs, batch)
    np.testing.assert_allclose(np.stack([h.tc, h.dtc, h.o, h.s]), e["mix_vals"], rtol=RTOL,
                               atol=ATOL)
    t = hoi.entropy_terms(covs, batch)
    np.testing.assert_allclose(t.h_joint, e["mix_hj"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(t.h_singles, e["mix_hs"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(t.h_leave_one_out, e["mix_hl"], rtol=1e-12, atol=1e-12)
    cs2 = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=60) for s in e["t2_sig"]])
    b2 = hoi.NpletBatch(6, indices=e["t2_idx"])
    t2 = hoi.entropy_terms(cs2, b2, bias_correct=True)
    np.testing.assert_allclose(t2.h_joint, e["t2_hj"], rtol=1e-12)
    np.testing.assert_allclose(t2.h_singles, e["t2_hs"], rtol=1e-12)
    np.testing.assert_allclose(t2.h_leave_one_out, e["t2_hl"], rtol=1e-12)
    h2 = hoi.compute_hoi_batch(cs2, b2, bias_correct=True)
    np.testing.assert_allclose(np.stack([h2.tc, h2.dtc, h2.o, h2.s]), e["t2_vals"], rtol=RTOL,
                               atol=ATOL)


# ----------------------------------------------------------- reducers ---

def _entries(lst):
    return [[list(e.indices), e.value, e.tc, e.dtc, e.o, e.s] for e in lst]


def test_topk_and_histogram_on_toy_covsets(golden):
    red = golden.meta["reducers"]
    sig = {k: np.array(v) for k, v in golden.meta["toy_sigmas"].items()}
    t1 = hoi.CovSet([hoi.CovarianceMatrix(sig["t1"][0])])
    for direction in ("max", "min"):
        got = _entries(hoi.scan(t1, 3, 5, hoi.TopK("o", direction, 7))[0])
        want = red[f"top_o_{direction}"]
        assert [g[0] for g in got] == [w[0] for w in want]
        np.testing.assert_allclose([g[1:] for g in got], [w[1:] for w in want], rtol=RTOL, atol=ATOL)
    t2 = hoi.CovSet([hoi.CovarianceMatrix(s) for s in sig["t2"]])
    base = hoi.scan(t2, 3, 6, hoi.TopK("s", "max", 9))
    for per_got, per_want in zip(base, red["top_s_max_d2"]):
        assert [list(e.indices) for e in per_got] == [w[0] for w in per_want]
    for bs, w in [(1, 1), (13, 1), (64, 3)]:
        assert hoi.scan(t2, 3, 6, hoi.TopK("s", "max", 9), batch_size=bs, workers=w) == base
    eye5 = hoi.CovSet([hoi.CovarianceMatrix(np.eye(5))])
    got = hoi.scan(eye5, 3, 3, hoi.TopK("o", "max", 4), batch_size=2)
    assert [list(e.indices) for e in got[0]] == red["top_tie"]
    assert all(e.value == 0.0 for e in got[0])
    t3 = hoi.CovSet([hoi.CovarianceMatrix(s) for s in sig["t3"]])
    edges, c8 = hoi.scan(t3, 2, 4, hoi.Histogram("tc", 8, 0.0, 0.5))
    assert c8.tolist() == red["hist_8"]
    np.testing.assert_allclose(edges, np.linspace(0.0, 0.5, 9))
    _, c2 = hoi.scan(t3, 2, 4, hoi.Histogram("tc", 2, 0.20, 0.21))
    assert c2.tolist() == red["hist_2"]


def test_cfg3_topk_histogram(golden):
    g = golden.npz("cfg3")
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"], n_samples_used=int(g["t"]))])
    got = _entries(hoi.scan(covs, 3, 20, hoi.TopK("o", "min", 10))[0])
    want = golden.meta["cfg3"]["top_o_min"]
    assert [x[0] for x in got] == [w[0] for w in want]
    np.testing.assert_allclose([x[1:] for x in got], [w[1:] for w in want], rtol=RTOL, atol=ATOL)
    got = _entries(hoi.scan(covs, 3, 20, hoi.TopK("s", "max", 10), bias_correct=True)[0])
    want = golden.meta["cfg3"]["top_s_max_bias"]
    assert [x[0] for x in got] == [w[0] for w in want]
    edges, counts = hoi.scan(covs, 3, 20, hoi.Histogram("o", 16, -0.5, 2.0))
    np.testing.assert_array_equal(edges, g["hist_edges"])
    assert int(np.abs(counts - g["hist_counts"]).sum()) <= 2   # edge-straddling rows only
    assert counts.sum() == hoi.count_nplets(20, 3, 20)


def test_features_and_callback_order(golden):
    red = golden.meta["reducers"]
    sig = {k: np.array(v) for k, v in golden.meta["toy_sigmas"].items()}
    t7 = hoi.CovSet([hoi.CovarianceMatrix(s) for s in sig["t7"]])
    feats = hoi.extract_features(t7)
    for f, w in zip(feats, red["features_t7"]):
        for name, v in w.items():
            assert getattr(f, name) == pytest.approx(v, abs=1e-12), name
    for f, w in zip(hoi.extract_features(hoi.CovSet([hoi.CovarianceMatrix(ora.r_system(3, 1.0))])), red["features_r3"]):
        for name, v in w.items():
            assert getattr(f, name) == pytest.approx(v, abs=1e-12), name
    ident = hoi.extract_features(hoi.CovSet([hoi.CovarianceMatrix(np.eye(5))]))[0]
    for name, v in ident.as_dict().items():
        assert v == (3 / 5 if name.endswith("order_norm") else 0.0), name
    ticks = []
    hoi.scan(t7, 2, 4, hoi.TopK("o", "max", 1), batch_size=7, progress=ticks.append)
    assert ticks[-1]["nplets"] == ticks[-1]["total"] == hoi.count_nplets(6, 2, 4)
    assert [t["batches"] for t in ticks] == list(range(1, len(ticks) + 1))


def test_cfg5_batched_large_system(oracle):
    """D=16 datasets x N=400, order-10 n-plets (B x D pairing), vs the oracle."""
    covs_np = []
    for d in range(16):
        x = workloads.cfg5_data(d)
        covs_np.append(oracle.covariance(oracle.copula(x)))
    sig = np.stack(covs_np)
    idx = workloads.cfg5_nplets(b=2048)
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=1200) for s in sig])
    for bias in (False, True):
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(400, indices=idx), bias_correct=bias)
        tc, dtc, o, s, _ = oracle.hoi_batch(sig, [1200] * 16, idx=idx, bias=bias)
        np.testing.assert_allclose(np.stack([h.tc, h.dtc, h.o, h.s]), np.stack([tc, dtc, o, s]),
                                   rtol=RTOL, atol=ATOL)
    # the device copula path agrees with the oracle on one dataset
    cov0 = hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(0)))
    np.testing.assert_allclose(cov0.sigma, sig[0], rtol=1e-12, atol=1e-15)


# ------------------------------------------------------ lattice engine --

def _random_cov(n, seed):
    rng = np.random.default_rng(seed)
    r = workloads.randcorr(n, rng)
    d = np.sqrt(rng.uniform(0.5, 3.0, n))
    return r * np.outer(d, d)


@pytest.mark.parametrize("k", [17, 18, 19, 20, 21, 22, 23, 24, 25, 29, 32])
def test_mid_orders_vs_oracle(oracle, k):
    """Orders 17..32 (the G-threads-per-unit kernels, KT = 20 / 24 / 32 with
    identity padding): index batches over 3 datasets with non-unit variances,
    with and without bias; log det / inverse-diagonal terms; and unranking
    mode (every order-k n-plet of N = k + 3 variables on engine 1)."""
    n, d, t = 40, 3, 900
    sig = np.stack([_random_cov(n, 100 + k + s) for s in range(d)])
    sig = 0.5 * (sig + sig.transpose(0, 2, 1))
    rng = np.random.default_rng(k)
    idx = np.sort(np.stack([rng.choice(n, k, replace=False) for _ in range(300)]), axis=1)
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=t) for s in sig])
    batch = hoi.NpletBatch(n, indices=idx)
    for bias in (False, True):
        h = hoi.compute_hoi_batch(covs, batch, bias_correct=bias)
        want = oracle.hoi_batch(sig, [t] * d, idx=idx, bias=bias)
        np.testing.assert_allclose(np.stack([h.tc, h.dtc, h.o, h.s]), np.stack(want[:4]),
                                   rtol=RTOL, atol=ATOL)
    terms = hoi.entropy_terms(covs, batch)
    xj, _, xl = oracle.terms_fixed(sig, [t] * d, idx)
    np.testing.assert_allclose(terms.excess_joint, xj, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(terms.excess_leave_one_out, xl, rtol=1e-12, atol=1e-12)
    m = k + 3
    small = hoi.CovSet([hoi.CovarianceMatrix(sig[0, :m, :m], n_samples_used=t)])
    dev = hoi.scan_device(small, k, k, bias_correct=True, engine=1)
    _, vals = oracle.scan(sig[:1, :m, :m], [t], k, k, oracle.CollectR(), bias=True)
    np.testing.assert_allclose(dev.out.cpu().numpy(), vals, rtol=RTOL, atol=ATOL)


def test_mixed_masks_high_orders_vs_oracle(oracle):
    """Mixed-order mask batches reaching orders 17..32 (compacted per order,
    rows scattered back, inverse diagonal scattered by variable id)."""
    n, t = 34, 700
    sig = _random_cov(n, 77)
    sig = 0.5 * (sig + sig.T)
    rng = np.random.default_rng(5)
    orders = rng.integers(2, 33, size=240)
    masks = np.zeros((orders.size, n), dtype=bool)
    for r, k in enumerate(orders):
        masks[r, rng.choice(n, int(k), replace=False)] = True
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig, n_samples_used=t)])
    batch = hoi.NpletBatch(n, masks=masks)
    for bias in (False, True):
        h = hoi.compute_hoi_batch(covs, batch, bias_correct=bias)
        want = oracle.hoi_batch(sig, [t], masks=masks, bias=bias)
        np.testing.assert_allclose(np.stack([h.tc, h.dtc, h.o, h.s]), np.stack(want[:4]),
                                   rtol=RTOL, atol=ATOL)
    terms = hoi.entropy_terms(covs, batch)
    xj, _, xl, _ = oracle.terms_mixed(sig[None], [t], masks)
    np.testing.assert_allclose(terms.excess_joint, xj, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(terms.excess_leave_one_out, xl, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("n,lo,hi", [(12, 1, 12), (13, 2, 13), (16, 3, 9)])
@pytest.mark.parametrize("bias", [False, True])
def test_lattice_engine_vs_oracle(oracle, n, lo, hi, bias, engine):
    """Exhaustive scans through the lattice (2) and the per-n-plet engine in
    unranking mode (1: per-thread unit chunks stepping the lexicographic
    successor), whole range and a rank sub-range, vs the oracle."""
    sig = _random_cov(n, n)
    sig = 0.5 * (sig + sig.T)
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig, n_samples_used=500)])
    dev = hoi.scan_device(covs, lo, hi, bias_correct=bias, engine=engine)
    _, vals = oracle.scan(sig, [500], lo, hi, oracle.CollectR(), bias=bias)
    np.testing.assert_allclose(dev.out.cpu().numpy(), vals, rtol=RTOL, atol=ATOL)
    # a sub-range of ranks lands at the same rows
    total = hoi.count_nplets(n, lo, hi)
    g0, g1 = total // 3, 2 * total // 3 + 1
    part = hoi.scan_device(covs, lo, hi, bias_correct=bias, engine=engine, g_begin=g0, g_end=g1)
    np.testing.assert_array_equal(part.out.cpu().numpy(), dev.out[:, g0:g1].cpu().numpy())


def test_lattice_matches_percell_engine_cfg3(golden):
    g = golden.npz("cfg3")
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"], n_samples_used=int(g["t"]))])
    for bias in (False, True):
        a = hoi.scan_device(covs, 3, 20, bias_correct=bias, engine=2).out
        b = hoi.scan_device(covs, 3, 20, bias_correct=bias, engine=1).out
        err = (a - b).abs() - 1e-9 * b.abs()
        assert float(err.max()) <= 1e-11
        assert bool((a[3] == a[0] + a[1]).all())


@pytest.mark.parametrize("bias", [True, False])
@pytest.mark.parametrize("n", [24, 25, 26, 28])
def test_lattice_column_pass_splits_vs_percell(n, bias):
    """Two-pass full output at the column pass's other splits (N = 24/25: 7
    low prefix bits, N = 26: 8, N = 28: 9; cfg4's 10 is the every-row test)
    against the per-n-plet engine on every row.  Without bias the whole-range
    scan takes the specialised pass-2 kernel (held ring job, block pairs over
    the lowest high prefix bit); with bias the general one."""
    rng = np.random.default_rng(100 + n)
    c = 0.7 * workloads.randcorr(n, rng) + 0.3 * np.eye(n)
    covs = hoi.CovSet([hoi.CovarianceMatrix(c, n_samples_used=1000)])
    a = hoi.scan_device(covs, 2, n, bias_correct=bias, engine=2).out
    b = hoi.scan_device(covs, 2, n, bias_correct=bias, engine=1).out
    err = (a - b).abs() - 1e-9 * b.abs()
    assert float(err.max()) <= 1e-11
    assert bool((a[3] == a[0] + a[1]).all())
    del a, b
    torch.cuda.empty_cache()


def test_lattice_multi_dataset(oracle):
    sigs = np.stack([_random_cov(14, s) for s in (1, 2, 3)])
    sigs = 0.5 * (sigs + sigs.transpose(0, 2, 1))
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=300) for s in sigs])
    dev = hoi.scan_device(covs, 2, 14, bias_correct=True, engine=2)
    _, vals = oracle.scan(sigs, [300] * 3, 2, 14, oracle.CollectR(), bias=True)
    np.testing.assert_allclose(dev.out.cpu().numpy(), vals, rtol=RTOL, atol=ATOL)


def test_lattice_dataset_stacks(oracle):
    """Multi-dataset lattice scans below N = 24 run as stacks (one table
    launch and one stencil launch per stack, claimed 4 datasets per block):
    D = 9 with per-dataset bias rows vs the oracle; D = 65 at N = 20 (two
    stacks of the 512 MB table budget) vs the per-n-plet engine."""
    sigs = np.stack([_random_cov(14, 40 + s) for s in range(9)])
    sigs = 0.5 * (sigs + sigs.transpose(0, 2, 1))
    ts = [200 + 17 * s for s in range(9)]
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=t) for s, t in zip(sigs, ts)])
    dev = hoi.scan_device(covs, 2, 14, bias_correct=True, engine=2)
    _, vals = oracle.scan(sigs, ts, 2, 14, oracle.CollectR(), bias=True)
    np.testing.assert_allclose(dev.out.cpu().numpy(), vals, rtol=RTOL, atol=ATOL)
    # shrunk towards I: a raw randcorr(20) can be so ill-conditioned at
    # order 20 that any two elimination orders differ beyond 1e-9
    big = hoi.CovSet([hoi.CovarianceMatrix(
        0.6 * workloads.randcorr(20, np.random.default_rng(s)) + 0.4 * np.eye(20),
        n_samples_used=500 + s) for s in range(65)])
    a = hoi.scan_device(big, 2, 20, bias_correct=True, engine=2).out
    b = hoi.scan_device(big, 2, 20, bias_correct=True, engine=1).out
    err = (a - b).abs() - 1e-9 * b.abs()
    assert float(err.max()) <= 1e-11
    assert bool((a[3] == a[0] + a[1]).all())
    del a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,d", [(12, 5), (23, 3)])
def test_lattice_dataset_stacks_at_the_size_limits(oracle, n, d):
    """Dataset stacks at the smallest lattice (N = 12: 4 blocks per dataset)
    and the largest stacked size (N = 23, just below the two-pass split):
    vs the oracle at N = 12, vs the per-n-plet engine at N = 23."""
    sigs = np.stack([0.7 * workloads.randcorr(n, np.random.default_rng(60 + s)) + 0.3 * np.eye(n)
                     for s in range(d)])
    ts = [300 + 11 * s for s in range(d)]
    covs = hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=t) for s, t in zip(sigs, ts)])
    lo = 2 if n == 12 else 18
    a = hoi.scan_device(covs, lo, n, bias_correct=True, engine=2).out
    if n == 12:
        _, vals = oracle.scan(sigs, ts, lo, n, oracle.CollectR(), bias=True)
        np.testing.assert_allclose(a.cpu().numpy(), vals, rtol=RTOL, atol=ATOL)
    else:
        b = hoi.scan_device(covs, lo, n, bias_correct=True, engine=1).out
        err = (a - b).abs() - 1e-9 * b.abs()
        assert float(err.max()) <= 1e-11
        del b
    del a
    torch.cuda.empty_cache()


def test_lattice_scans_are_deterministic():
    """Repeated multi-dataset lattice scans are bit-identical.  Regression:
    when consumers lagged (D >= 4, strided output stores) a ring slot could
    be refilled by TMA while shared loads of it were still in flight (fixed
    with a proxy fence before each slot release)."""
    for n, d in ((20, 8), (22, 4)):
        covs = hoi.CovSet([hoi.CovarianceMatrix(workloads.randcorr(n, np.random.default_rng(s)))
                           for s in range(d)])
        ref = hoi.scan_device(covs, 2, n, engine=2).out
        for _ in range(3):
            assert bool((hoi.scan_device(covs, 2, n, engine=2).out == ref).all())
        del ref
        torch.cuda.empty_cache()


def test_lattice_declines_singular_covariance(oracle):
    """A duplicated variable makes R singular: the lattice engine declines
    and the per-n-plet engine applies the reference's jitter rule."""
    sig = _random_cov(12, 7)
    sig[11, :] = sig[10, :]
    sig[:, 11] = sig[:, 10]
    covs = hoi.CovSet([hoi.CovarianceMatrix(sig)])
    dev = hoi.scan_device(covs, 2, 4)
    _, vals = oracle.scan(sig, [0], 2, 4, oracle.CollectR())
    got = dev.out.cpu().numpy()
    assert np.isfinite(got).all()
    rows = [c for k in range(2, 5) for c in itertools.combinations(range(12), k)]
    clean = np.array([not (10 in r and 11 in r) for r in rows])
    np.testing.assert_allclose(got[:, clean], vals[:, clean], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("measure,direction,k,bias", [("o", "min", 1000, False),
                                                      ("s", "max", 100, True),
                                                      ("tc", "max", 7, False)])
def test_filtered_topk_matches_full_output(measure, direction, k, bias):
    """The lattice engine's filtered TopK (sampled threshold, no full output)
    returns exactly what the full-output path returns (itself checked against
    the oracle above): N = 24 is the smallest size that takes the sampled
    branch (2^14 table blocks), orders 2..24, 16.8M n-plets."""
    from paper_2501_03381_b200 import scanner
    rng = np.random.default_rng(7)
    c = workloads.randcorr(24, rng)
    x = rng.standard_normal((3000, 24)) @ np.linalg.cholesky(c).T
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(x))])
    got = hoi.scan(covs, 2, 24, hoi.TopK(measure, direction, k), bias_correct=bias)[0]
    ctx = scanner._ScanCtx(covs, 2, 24, bias, 2)
    ref = hoi.TopK(measure, direction, k)
    total = hoi.count_nplets(24, 2, 24)
    out, _, _ = ctx.full(0, total)
    scanner._topk_plane(ctx, ref, out, 0, scanner.MEASURES.index(measure))
    want = ref.finalize()[0]
    assert [e.indices for e in got] == [e.indices for e in want]
    # the filtered pass sums the leave-one-out terms in one pass, the full
    # output in two (low bits, then high bits): last-bit differences only
    np.testing.assert_allclose([(e.tc, e.dtc, e.o, e.s) for e in got],
                               [(e.tc, e.dtc, e.o, e.s) for e in want], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("shard_bits", [1, 2])
def test_block_shards_reassemble_the_scan(shard_bits):
    """Multi-GPU block shards, run one after another on one GPU: each shard
    writes only its own rows (global positions), the shards' row sets are
    the host model's partition, their union is bit-identical to the
    single-GPU scan, and per-shard TopK lists merged with the reference key
    equal the single-GPU TopK."""
    from paper_2501_03381_b200 import scanner, sharding
    rng = np.random.default_rng(5)
    c = workloads.randcorr(24, rng)
    x = rng.standard_normal((2500, 24)) @ np.linalg.cholesky(c).T
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(x))])
    total = hoi.count_nplets(24, 2, 24)
    ctx = scanner._ScanCtx(covs, 2, 24, False, 2)
    want, _, _ = ctx.full(0, total)
    want = want.clone()
    got = torch.full((4, total, 1), float("nan"), dtype=torch.float64, device="cuda")
    # shard of every row: membership pattern over variables 24-10-sb .. 13
    # (the partition scanner.shard_rows models on the host)
    idx, _ = unrank_device(24, 2, 24, 0, total)
    lo_var = 24 - 10 - shard_bits
    pat = torch.zeros(total, dtype=torch.int64, device="cuda")
    for t in range(shard_bits):
        pat |= (idx == lo_var + t).any(dim=1).long() << t
    del idx
    for r in range(1 << shard_bits):
        before = torch.isnan(got[0, :, 0])
        ctx.full_shard(r, shard_bits, got)
        newly = before & ~torch.isnan(got[0, :, 0])
        assert torch.equal(newly, pat == r)
    assert torch.equal(got, want)
    parts = []
    for r in range(1 << shard_bits):
        red = hoi.TopK("o", "min", 500)
        cx = scanner._ScanCtx(covs, 2, 24, False, 2)
        assert scanner._topk_lattice(cx, red, 2, shard=r, shard_bits=shard_bits)
        parts.append(red._best)
    merged = sharding.merge_topk(parts, 500)
    single = hoi.scan(covs, 2, 24, hoi.TopK("o", "min", 500))[0]
    assert [e.indices for _, e in merged[0]] == [e.indices for e in single]


@pytest.mark.parametrize("world", [2, 4])
def test_block_shard_sets_reassemble_the_scan(world):
    """block_shard_plan's per-rank shard pairs, run one after another on one
    GPU: each rank's set writes exactly the rows of its shards, the union is
    bit-identical to the single-GPU scan, and the merged per-rank TopK
    lists equal the single-GPU TopK."""
    from paper_2501_03381_b200 import scanner, sharding
    rng = np.random.default_rng(11)
    c = workloads.randcorr(22, rng)
    x = rng.standard_normal((2000, 22)) @ np.linalg.cholesky(c).T
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(x))])
    total = hoi.count_nplets(22, 2, 22)
    ctx = scanner._ScanCtx(covs, 2, 22, False, 2)
    want, _, _ = ctx.full(0, total)
    want = want.clone()
    sb, masks = sharding.block_shard_plan(22, world)
    got = torch.full((4, total, 1), float("nan"), dtype=torch.float64, device="cuda")
    idx, _ = unrank_device(22, 2, 22, 0, total)
    lo_var = 22 - 10 - sb
    pat = torch.zeros(total, dtype=torch.int64, device="cuda")
    for t in range(sb):
        pat |= (idx == lo_var + t).any(dim=1).long() << t
    del idx
    for m in masks:
        before = torch.isnan(got[0, :, 0])
        ctx.full_shard_set(m, sb, got)
        newly = before & ~torch.isnan(got[0, :, 0])
        own = torch.zeros_like(newly)
        for cidx in range(1 << sb):
            if (m >> cidx) & 1:
                own |= pat == cidx
        assert torch.equal(newly, own)
    assert torch.equal(got, want)
    parts = []
    for m in masks:
        red = hoi.TopK("o", "min", 50)
        assert scanner._topk_lattice(scanner._ScanCtx(covs, 2, 22, False, 2), red, 2,
                                     shard_bits=sb, shard_mask=m)
        parts.append(red._best)
    merged = sharding.merge_topk(parts, 50)
    one = hoi.scan(covs, 2, 22, hoi.TopK("o", "min", 50))
    assert [[e.indices for _, e in per] for per in merged] == [[e.indices for e in per]
                                                               for per in one]
    del got, want
    torch.cuda.empty_cache()


def test_topk_bound_brackets_the_exact_key():
    """hoi_topk_bound: never below the exact k-th key (hoi_topk_threshold),
    tighter with more bits, equal to it at 64 bits."""
    import ctypes
    rng = np.random.default_rng(3)
    vals = torch.as_tensor(rng.standard_normal((50000, 5)), device="cuda")
    lib, s = _native.lib(), _native.stream_handle(torch)
    ws = torch.empty(4096 + 64, dtype=torch.int64, device="cuda")
    key = torch.empty(1, dtype=torch.int64, device="cuda")
    for sign, k in ((1.0, 1000), (-1.0, 7)):
        _native.check(lib.hoi_topk_threshold(vals.data_ptr(), 50000, 5, 2, sign, k,
                                             key.data_ptr(), ws.data_ptr(), s), "threshold")
        exact = int(key.item()) & (2 ** 64 - 1)
        prev = None
        for bits in (12, 24, 36, 64):
            _native.check(lib.hoi_topk_bound(vals.data_ptr(), 50000, 5, 2, sign, k, bits,
                                             key.data_ptr(), ws.data_ptr(), s), "bound")
            b = int(key.item()) & (2 ** 64 - 1)
            assert b >= exact and (prev is None or b <= prev)
            prev = b
        assert prev == exact


def test_topk_batch_matches_host_reducer():
    """Device batched TopK == the reference's TopK.update on the same
    HoiBatch (cfg5-style: 16 datasets, N = 400, order-10 random n-plets)."""
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(d)))
                       for d in range(16)])
    idx = workloads.cfg5_nplets(b=30000)
    batch = hoi.NpletBatch(400, indices=idx)
    for measure, direction, k in [("o", "min", 100), ("s", "max", 7)]:
        got = hoi.topk_batch(covs, batch, hoi.TopK(measure, direction, k)).finalize()
        ref = hoi.TopK(measure, direction, k)
        ref.update(batch, hoi.compute_hoi_batch(covs, batch))
        want = ref.finalize()
        for g, w in zip(got, want):
            assert [e.indices for e in g] == [e.indices for e in w]
            assert [(e.tc, e.dtc, e.o, e.s) for e in g] == [(e.tc, e.dtc, e.o, e.s) for e in w]


def test_device_features_match_host_replay():
    """The device feature reducer equals the reference accumulator fed the
    same device measures batch by batch (host replay, the generic Reducer
    path), on 3 datasets of N = 16 over orders 2..16 and a sub-range."""
    from paper_2501_03381_b200 import scanner
    rng = np.random.default_rng(21)
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(
        rng.standard_normal((600, 16)) @ np.linalg.cholesky(workloads.randcorr(16, rng)).T))
        for _ in range(3)])
    got = hoi.extract_features(covs)

    class Replay(hoi.FeatureAccumulator):
        pass                                   # not the exact type: takes the replay path

    want = hoi.scan(covs, 2, 16, Replay(16), batch_size=3000)
    for g, w in zip(got, want):
        for name in hoi.FEATURE_NAMES:
            assert getattr(g, name) == pytest.approx(getattr(w, name), rel=1e-11, abs=1e-12), name


def test_scan_file_round_trip(tmp_path, golden):
    """Binary scan format: cfg1's device output written in small chunks and
    read back through the host memmap reader equals the golden values."""
    g = golden.npz("cfg1")
    covs = hoi.CovSet([hoi.CovarianceMatrix(g["cov"])])
    dev = hoi.scan_device(covs, 3, 10)
    path = dev.save(tmp_path / "cfg1.hoiscan", chunk_rows=100)
    head, planes = hoi.read_scan(path)
    assert head["n"] == 10 and head["g_end"] - head["g_begin"] == 968 and head["datasets"] == 1
    np.testing.assert_array_equal(planes, dev.out.cpu().numpy())
    np.testing.assert_allclose(planes[:, :, 0], g["vals"], rtol=RTOL, atol=ATOL)


def test_topk_at_n32_largest_lattice():
    """N = 32, orders 2..32 (4.29e9 n-plets, 2^22 table blocks, 34 GB log-det
    table): the filtered TopK's entries are re-evaluated by the per-n-plet
    engine (values within the FP64 tolerance), and none of 200,000
    uniformly sampled n-plets beats the k-th entry."""
    rng = np.random.default_rng(32)
    c = workloads.randcorr(32, rng)
    x = rng.standard_normal((4000, 32)) @ np.linalg.cholesky(c).T
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(x))])
    k = 50
    top = hoi.scan(covs, 2, 32, hoi.TopK("o", "min", k))[0]
    assert len(top) == k
    vals = [e.o for e in top]
    assert vals == sorted(vals)
    for order in sorted({e.order for e in top}):
        sel = [e for e in top if e.order == order]
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(32, indices=np.array([e.indices for e in sel])))
        np.testing.assert_allclose(h.o[:, 0], [e.o for e in sel], rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(h.tc[:, 0], [e.tc for e in sel], rtol=RTOL, atol=ATOL)
    total = hoi.count_nplets(32, 2, 32)
    ranks = torch.as_tensor(np.sort(rng.choice(total, size=200_000, replace=False)), device="cuda")
    idx = torch.empty((ranks.numel(), 32), dtype=torch.int32, device="cuda")
    orders = torch.empty(ranks.numel(), dtype=torch.int32, device="cuda")
    _native.check(_native.lib().hoi_unrank_list(32, 2, 32, ranks.data_ptr(), ranks.numel(),
                                                idx.data_ptr(), orders.data_ptr(),
                                                _native.stream_handle(torch)), "unrank_list")
    idx, orders = idx.cpu().numpy(), orders.cpu().numpy()
    worst = vals[-1]
    for kk in np.unique(orders):
        rows = idx[orders == kk, :kk].astype(np.int64)
        h = hoi.compute_hoi_batch(covs, hoi.NpletBatch(32, indices=rows, check_unique=False))
        assert (h.o[:, 0] >= worst - 1e-9).all()


def test_chunked_replay_reuses_the_table(monkeypatch):
    """A Callback scan at N = 24 (two-pass lattice) replayed in forced small
    device chunks (partial rank ranges that reuse one log-det table through
    compacted block lists) returns exactly the one-shot device output, batch
    by batch in the reference's order."""
    from paper_2501_03381_b200 import scanner
    rng = np.random.default_rng(24)
    c = workloads.randcorr(24, rng)
    x = rng.standard_normal((1500, 24)) @ np.linalg.cholesky(c).T
    covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(x))])
    lo, hi = 6, 11
    full = hoi.scan_device(covs, lo, hi, engine=2).out[:, :, 0].cpu().numpy()
    monkeypatch.setattr(scanner, "_chunk_rows", lambda *a, **k: 700_000)
    got, sizes = [], []

    def keep(batch, h):
        sizes.append((batch.batch_size, int(h.order[0])))
        got.append(np.stack([h.tc[:, 0], h.dtc[:, 0], h.o[:, 0], h.s[:, 0]]))

    hoi.scan(covs, lo, hi, hoi.Callback(keep), batch_size=250_000)
    got = np.concatenate(got, axis=1)
    assert got.shape == full.shape
    np.testing.assert_array_equal(got, full)
    assert all(b <= 250_000 for b, _ in sizes)
    assert [k for _, k in sizes] == sorted(k for _, k in sizes)


@pytest.mark.parametrize("n,k,d", [(400, 10, 16), (30, 16, 1), (30, 6, 1), (30, 20, 1)])
def test_fp32_fast_path_within_1e4_nats(n, k, d):
    """precision='fp32' (FP32 factorisation, FP64 logs and epilogue) stays
    within the north star's 1e-4 nats of the FP64 path; orders above 16 run
    the FP64 kernels (identical)."""
    if n == 400:
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg5_data(i)))
                           for i in range(d)])
        idx = workloads.cfg5_nplets(b=50_000, n=n, k=k)
    else:
        covs = hoi.CovSet([hoi.estimate_covariance(hoi.copula_transform(workloads.cfg4()))])
        rng = np.random.default_rng(k)
        idx = np.sort(np.argsort(rng.random((20_000, n)), axis=1)[:, :k], axis=1)
    batch = hoi.NpletBatch(n, indices=idx, check_unique=False)
    for bias in (False, True):
        h64 = hoi.compute_hoi_batch(covs, batch, bias_correct=bias)
        h32 = hoi.compute_hoi_batch(covs, batch, bias_correct=bias, precision="fp32")
        for m in ("tc", "dtc", "o", "s"):
            err = np.abs(getattr(h32, m) - getattr(h64, m)).max()
            assert err < 1e-4, (m, err)
            if k > 16:
                assert err == 0.0
