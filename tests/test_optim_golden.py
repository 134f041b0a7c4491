"""Optimiser drop-in (ref:optimizers.py) against
results of the real reference
(tests/golden/make_golden_optim.py).  Host-only checks run on CPU; the
greedy / anneal runs evaluate every energy on the device (-m gpu)."""

import json
import warnings
from pathlib import Path

import numpy as np
import pytest

import paper_2501_03381_b200 as hoi

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "optim.json").read_text())
RTOL, ATOL = 1e-9, 1e-11


def _covs():
    z = np.load(Path(__file__).resolve().parent / "golden" / "optim.npz")
    return hoi.CovSet([hoi.CovarianceMatrix(s, n_samples_used=int(t))
                       for s, t in zip(z["sigma"], z["t"])])


SPECS = {
    "mean_o_max": hoi.ObjectiveSpec("o", "max"),
    "mean_s_min": hoi.ObjectiveSpec("s", "min"),
    "effect_tc_max": hoi.ObjectiveSpec("tc", "max", "effect", (0, 1), (2, 3)),
}


def test_objective_spec_validation():
    for kw in [dict(measure="q"), dict(direction="up"), dict(aggregator="median"),
               dict(aggregator="effect"), dict(aggregator="effect", cond_a=(0,), cond_b=(1,)),
               dict(aggregator="effect", cond_a=(0, 1), cond_b=(1, 2)),
               dict(aggregator="effect", cond_a=(0, 1, 2), cond_b=(3, 4))]:
        with pytest.raises(hoi.InvalidData):
            hoi.ObjectiveSpec(**kw)
    assert hoi.ObjectiveSpec("o", "min").value_of(2.0) == -2.0


def test_evaluate_objective_host_matches_reference(oracle):
    """The HoiBatch-level objective on the oracle's measures equals the
    reference's evaluate_objective (mean, paired Cohen's d, direction)."""
    covs = _covs()
    idx = np.array(GOLD["objective_idx"])
    tc, dtc, o, s, orders = oracle.hoi_batch(covs.stacked(), [c.n_samples_used for c in covs.covs],
                                             idx=idx)
    h = hoi.HoiBatch(tc=tc, dtc=dtc, o=o, s=s, order=orders)
    for name, sp in SPECS.items():
        np.testing.assert_allclose(hoi.evaluate_objective(h, sp), GOLD["objective"][name],
                                   rtol=1e-12)
    h2 = hoi.HoiBatch(tc=np.ones((2, 4)), dtc=tc[:2], o=o[:2], s=s[:2], order=orders[:2])
    with pytest.raises(hoi.DegenerateEffectSize):
        hoi.evaluate_objective(h2, SPECS["effect_tc_max"])


def test_optimizer_argument_validation():
    covs = _covs()
    with pytest.raises(hoi.InvalidOrderRange):
        hoi.greedy(covs, SPECS["mean_o_max"], 5, 3)
    with pytest.raises(hoi.InvalidData):
        hoi.greedy(covs, SPECS["mean_o_max"], 2, 3, kappa=0)
    with pytest.raises(hoi.InvalidOrderRange):
        hoi.anneal(covs, SPECS["mean_o_max"], hoi.AnnealSchedule(min_order=9, max_order=4))
    with pytest.raises(hoi.InvalidData):
        hoi.AnnealSchedule(alpha=1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SPECS))
@pytest.mark.parametrize("bias", [False, True])
def test_greedy_matches_reference(name, bias):
    covs = _covs()
    ev = []
    got = hoi.greedy(covs, SPECS[name], 3, 7, kappa=5, bias_correct=bias,
                     progress=lambda p: ev.append({k: p[k] for k in ("order", "batches", "nplets")}))
    want = GOLD["runs"][f"greedy_{name}_{int(bias)}"]
    assert [[e.order, list(e.indices)] for e in got.per_order] == [w[:2] for w in want["per_order"]]
    np.testing.assert_allclose([[e.energy, e.value] for e in got.per_order],
                               [w[2:] for w in want["per_order"]], rtol=RTOL, atol=ATOL)
    assert ev == want["progress"]


@pytest.mark.gpu
def test_greedy_restarts_matches_reference():
    got = hoi.greedy(_covs(), SPECS["mean_o_max"], 3, 6, kappa=4, seed=7, restarts=3, batch_size=50)
    want = GOLD["runs"]["greedy_restarts"]["per_order"]
    assert [[e.order, list(e.indices)] for e in got.per_order] == [w[:2] for w in want]
    np.testing.assert_allclose([e.energy for e in got.per_order], [w[2] for w in want], rtol=RTOL)


@pytest.mark.gpu
@pytest.mark.parametrize("name,sched", [
    ("anneal_across", hoi.AnnealSchedule(max_iters=80)),
    ("anneal_within", hoi.AnnealSchedule(temp0=0.05, mode="within-order", patience=15,
                                         max_iters=200, min_order=4, max_order=8))])
def test_anneal_matches_reference(name, sched):
    """Same per-chain random streams and draws as the reference: the same
    trajectory, final population and best solution."""
    st = hoi.anneal(_covs(), SPECS["mean_o_max"], sched, kappa=8, seed=3)
    want = GOLD["runs"][name]
    assert list(st.best_indices) == want["best_indices"]
    assert st.iterations == want["iterations"]
    np.testing.assert_array_equal(st.masks.astype(int), np.array(want["masks"]))
    np.testing.assert_allclose(st.energies, want["energies"], rtol=RTOL, atol=ATOL)
    assert st.best_energy == pytest.approx(want["best_energy"], rel=RTOL)
    assert st.temperature == pytest.approx(want["temperature"], rel=1e-12)


@pytest.mark.gpu
def test_device_objective_matches_reference():
    covs = _covs()
    idx = np.array(GOLD["objective_idx"])
    from paper_2501_03381_b200.optimizers import _batch_energies
    for name, sp in SPECS.items():
        e = _batch_energies(covs, hoi.NpletBatch(12, indices=idx), sp, False).cpu().numpy()
        np.testing.assert_allclose(e, GOLD["objective"][name], rtol=RTOL, atol=ATOL)


@pytest.mark.gpu
def test_greedy_kappa_clip_warns():
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        hoi.greedy(_covs(), SPECS["mean_o_max"], 1, 2, kappa=50)
    assert any("clipping" in str(x.message) for x in w)
