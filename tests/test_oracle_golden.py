"""Pin the CPU oracle (oracle/hoi_oracle.py) to golden vectors produced by
the real reference (tests/golden/make_golden.py).  CPU only."""

import math
import os

import numpy as np
import pytest

from paper_2501_03381_b200 import workloads

RTOL, ATOL = 1e-9, 1e-11          # ref tests/test_acceptance.py:81


def test_copula_matches_golden(golden, oracle):
    g = golden.npz("copula")
    np.testing.assert_array_equal(oracle.ranks(g["x"]), g["ranks"])
    np.testing.assert_array_equal(oracle.copula(g["x"]), g["z"])
    np.testing.assert_array_equal(oracle.ranks(g["tie"]), g["tie_ranks"])
    assert g["tie_ranks"][:, 0].tolist() == [3, 1, 4, 2]
    np.testing.assert_allclose(oracle.covariance(oracle.copula(g["x"])), g["cov"], rtol=1e-12)
    for (n, t), v in zip(g["bias_pairs"], g["bias_vals"]):
        assert oracle.entropy_bias(int(n), int(t)) == pytest.approx(v, abs=1e-15)
    np.testing.assert_array_equal(oracle.bias_table(60, 12), g["bias_tab_60"])
    np.testing.assert_array_equal(oracle.bias_table(2000, 30), g["bias_tab_2000"])
    np.testing.assert_array_equal(oracle.bias_table(10000, 20), g["bias_tab_10000"])


def test_frozen_constants(golden, oracle):
    fz = golden.meta["frozen"]
    assert oracle.entropy_bias(1, 2) == pytest.approx(fz["BIAS_1_2"], abs=1e-15)
    assert fz["BIAS_1_2"] == pytest.approx(-0.6351814227307391, abs=1e-15)
    assert oracle.count(30, 3, 30) == fz["count_30_3_30"] == 1_073_741_358
    for key, want in golden.meta["edge"]["counts"].items():
        n, lo, hi = map(int, key.split(","))
        assert oracle.count(n, lo, hi) == want


def test_workload_inputs_unchanged(golden):
    import hashlib

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    assert sha(workloads.cfg1()) == golden.meta["cfg1"]["x_sha"]
    assert sha(workloads.cfg2()) == golden.meta["cfg2"]["x_sha"]
    assert sha(workloads.cfg3()) == golden.meta["cfg3"]["x_sha"]
    assert sha(workloads.cfg4()) == golden.meta["cfg4"]["x_sha"]


def test_cfg1_full_scan(golden, oracle):
    g = golden.npz("cfg1")
    cov = oracle.covariance(oracle.copula(g["x"]))
    np.testing.assert_allclose(cov, g["cov"], rtol=1e-12)
    r = oracle.CollectR()
    rows, vals = oracle.scan(g["cov"], [0], 3, 10, r)
    assert sum(len(b) for b in rows) == 968
    np.testing.assert_allclose(vals[:, :, 0], g["vals"], rtol=RTOL, atol=ATOL)


def test_cfg2_full_scan_bias(golden, oracle):
    g = golden.npz("cfg2")
    cov = oracle.covariance(oracle.copula(workloads.cfg2()))
    np.testing.assert_allclose(cov, g["cov"], rtol=1e-12)
    r = oracle.CollectR()
    _, vals = oracle.scan(g["cov"], [int(g["t"])], 3, 12, r, bias=True)
    np.testing.assert_allclose(vals[:, :, 0], g["vals"], rtol=RTOL, atol=ATOL)
    m = golden.meta["cfg2"]
    assert m["o_0123"] > 0          # redundant block
    assert abs(m["o_456"]) < 1e-6   # the copula cannot see product synergy


@pytest.mark.parametrize("cfg,lo,hi", [("cfg3", 3, 20), ("cfg4", 2, 30)])
def test_sampled_ranks(golden, oracle, cfg, lo, hi):
    g = golden.npz(cfg)
    n = g["cov"].shape[0]
    rows = [tuple(int(v) for v in r if v >= 0) for r in g["idx"]]
    # global rank -> tuple is the reference's order-major lexicographic order
    for gr, tup in list(zip(g["g"], rows))[:40]:
        k = len(tup)
        off = sum(math.comb(n, kk) for kk in range(lo, k))
        it = __import__("itertools").combinations(range(n), k)
        assert next(__import__("itertools").islice(it, int(gr) - off, None)) == tup
    for bias, key in ((False, "vals"), (True, "vals_bias")):
        by_k = {}
        for i, t in enumerate(rows):
            by_k.setdefault(len(t), []).append(i)
        got = np.empty_like(g[key])
        for k, sel in by_k.items():
            tc, dtc, o, s, _ = oracle.hoi_batch(g["cov"], [int(g["t"])],
                                                idx=np.array([rows[i] for i in sel]), bias=bias)
            got[:, sel, :] = np.stack([tc, dtc, o, s])
        np.testing.assert_allclose(got, g[key], rtol=RTOL, atol=ATOL)


def test_edge_cases(golden, oracle):
    e = golden.npz("edge")
    for k in (2, 3, 4, 6):
        idx = np.array(list(__import__("itertools").combinations(range(6), k)))
        tc, dtc, o, s, _ = oracle.hoi_batch(np.eye(6), [0], idx=idx)
        for got, want in zip((tc, dtc, o, s), e[f"ident{k}"]):
            np.testing.assert_array_equal(got, want)
            assert (got == 0.0).all()
    for m in (2, 3, 4):
        for kind, fn in (("r", oracle.r_system), ("s", oracle.s_system)):
            tc, dtc, o, s, _ = oracle.hoi_batch(fn(m, 1.0), [0], idx=np.arange(m + 1)[None])
            np.testing.assert_allclose([tc[0, 0], dtc[0, 0], o[0, 0], s[0, 0]],
                                       e[f"rs_{kind}{m}"], atol=1e-13)
    with pytest.raises(oracle.OracleNotPD) as err:
        oracle.logdet_invdiag(np.stack([np.eye(2), np.array([[1.0, 2.0], [2.0, 1.0]])])[:, None])
    assert [list(c) for c in err.value.coords] == golden.meta["edge"]["npd_coords"]
    ld, idg = oracle.logdet_invdiag((np.ones((3, 3)) + np.eye(3) * 1e-14)[None, None])
    np.testing.assert_allclose(ld, e["singular_ld"], rtol=1e-9)
    tc, dtc, o, s, _ = oracle.hoi_batch(e["mix_sigma"], [0], masks=e["mix_masks"])
    np.testing.assert_allclose(np.stack([tc, dtc, o, s]), e["mix_vals"], rtol=RTOL, atol=ATOL)
    xj, xs, xl = oracle.terms_fixed(e["t2_sig"], [60, 60], e["t2_idx"], bias=True)
    np.testing.assert_allclose(xj + 3 * oracle.H1, e["t2_hj"], rtol=1e-12)
    np.testing.assert_allclose(xl + 2 * oracle.H1, e["t2_hl"], rtol=1e-12)


def test_reducers_on_toy_covsets(golden, oracle):
    red = golden.meta["reducers"]
    sig = {k: np.array(v) for k, v in golden.meta["toy_sigmas"].items()}
    for direction in ("max", "min"):
        got = oracle.scan(sig["t1"], [0], 3, 5, oracle.TopKR("o", direction, 7))
        want = red[f"top_o_{direction}"]
        assert [list(e[0]) for e in got[0]] == [w[0] for w in want]
        np.testing.assert_allclose([e[1] for e in got[0]], [w[1] for w in want], rtol=RTOL)
    got = oracle.scan(sig["t2"], [0, 0], 3, 6, oracle.TopKR("s", "max", 9), batch_size=13,
                      workers=3)
    for per_got, per_want in zip(got, red["top_s_max_d2"]):
        assert [list(e[0]) for e in per_got] == [w[0] for w in per_want]
    got = oracle.scan(np.eye(5), [0], 3, 3, oracle.TopKR("o", "max", 4), batch_size=2)
    assert [list(e[0]) for e in got[0]] == red["top_tie"]
    _, c8 = oracle.scan(sig["t3"], [0, 0], 2, 4, oracle.HistR("tc", 8, 0.0, 0.5))
    assert c8.tolist() == red["hist_8"]
    _, c2 = oracle.scan(sig["t3"], [0, 0], 2, 4, oracle.HistR("tc", 2, 0.20, 0.21))
    assert c2.tolist() == red["hist_2"]
    feats = oracle.scan(sig["t7"], [0, 0, 0], 2, 6, oracle.FeaturesR(6))
    for f, w in zip(feats, red["features_t7"]):
        for name, v in w.items():
            assert f[name] == pytest.approx(v, abs=1e-12), name


def test_cfg3_topk_and_histogram(golden, oracle):
    g = golden.npz("cfg3")
    want = golden.meta["cfg3"]["top_o_min"]
    got = oracle.scan(g["cov"], [int(g["t"])], 3, 20, oracle.TopKR("o", "min", 10),
                      workers=os.cpu_count() or 1)
    assert [list(e[0]) for e in got[0]] == [w[0] for w in want]
    np.testing.assert_allclose([e[1] for e in got[0]], [w[1] for w in want], rtol=RTOL)
