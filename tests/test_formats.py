"""Data formats either side of the path (paper_2501_03381_b200/formats.py)
against the REAL reference CLI's files (tests/golden/csv, written by
tests/golden/make_golden_csv.py).

CPU: the loader reads the data files exactly; its errors match the
reference's; every reference output file is reproduced byte for byte from
its own parsed values (repr floats, hex masks, quoting, line ends).
GPU: the whole pipeline from the same data files -- copula, covariance,
scan / features / greedy / anneal on the device -- formatted and compared
field by field: names, orders and masks exactly, floats within the FP64
bound (rtol 1e-9, atol 1e-11).
"""

import csv
import io
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2501_03381_b200 as hoi
from paper_2501_03381_b200 import formats
from paper_2501_03381_b200.errors import InvalidData
from paper_2501_03381_b200.scanner import FEATURE_NAMES, TopEntry

GOLD = Path(__file__).resolve().parent / "golden" / "csv"
IN, OUT = GOLD / "in", GOLD / "out"


def _rows(text):
    return list(csv.reader(io.StringIO(text)))


def _ref(name):
    return (OUT / f"{name}.csv").read_text(encoding="utf-8")


def _indices(mask_text):
    m = int(mask_text, 16)
    return tuple(i for i in range(m.bit_length()) if (m >> i) & 1)


# -------------------------------------------------------------- CPU ----

def test_load_datasets_reads_the_files_exactly():
    names, datas = formats.load_datasets(IN)
    assert names == ["ds_a", "ds_b", "ds_c"]
    for name, dm in zip(names, datas):
        raw = _rows((IN / f"{name}.csv").read_text())
        assert dm.column_names == raw[0]
        np.testing.assert_array_equal(dm.values, np.array(raw[1:], dtype=float))
    one_names, one = formats.load_datasets(IN / "ds_b.csv")
    assert one_names == ["ds_b"] and one[0].values.shape == (120, 9)


@pytest.mark.parametrize("text,msg", [
    ("a,b\n", "need a header row"),
    ("a,b\n1,2\n3\n", "row 3 has 1 fields, expected 2"),
    ("a,b\n1,2\n3,x\n", "non-numeric value in row 3"),
])
def test_read_csv_errors(tmp_path, text, msg):
    p = tmp_path / "d.csv"
    p.write_text(text)
    with pytest.raises(InvalidData, match=msg):
        formats.read_csv(p)


def test_loader_directory_errors(tmp_path):
    with pytest.raises(InvalidData, match="no .csv files"):
        formats.load_datasets(tmp_path)
    with pytest.raises(InvalidData, match="no such file"):
        formats.load_datasets(tmp_path / "missing")
    (tmp_path / "a.csv").write_text("x,y,z\n1,2,3\n2,1,3\n3,3,1\n")
    (tmp_path / "b.csv").write_text("x,y,w\n1,2,3\n2,1,3\n3,3,1\n")
    with pytest.raises(InvalidData, match="header differs"):
        formats.load_datasets(tmp_path)
    bad = tmp_path / "bad.csv"
    bad.write_bytes(b"x\n\xff\n")
    with pytest.raises(InvalidData, match="not valid UTF-8"):
        formats.read_csv(bad)


def test_mask_and_float_text():
    assert formats.mask_hex((0, 3, 4)) == "0x19"
    assert formats.mask_hex(()) == "0x0"
    assert formats.float_text(0.1) == "0.1"
    assert formats.float_text(np.float64(-2.5e-300)) == "-2.5e-300"


def _names():
    return formats.load_datasets(IN)[1][0].column_names


def test_topk_csv_reproduces_the_reference_bytes():
    text = _ref("top")
    rows = _rows(text)[1:]
    names = sorted({r[0] for r in rows})
    per = {n: [] for n in names}
    m_idx = ("tc", "dtc", "o", "s").index("o")
    for r in rows:
        idx = _indices(r[3])
        assert ",".join(_names()[i] for i in idx) == r[2] and len(idx) == int(r[1])
        v = [float(x) for x in r[4:8]]
        per[r[0]].append(TopEntry(idx, len(idx), v[m_idx], *v))
    assert formats.topk_csv([per[n] for n in names], names, _names()) == text


def test_histogram_csv_reproduces_the_reference_bytes():
    text = _ref("hist")
    rows = _rows(text)[1:]
    names = list(dict.fromkeys(r[0] for r in rows))
    bins = len(rows) // len(names)
    edges = np.array([float(r[1]) for r in rows[:bins]] + [float(rows[bins - 1][2])])
    counts = np.array([int(r[3]) for r in rows], dtype=np.int64).reshape(len(names), bins)
    assert formats.histogram_csv((edges, counts), names) == text


def test_features_csv_reproduces_the_reference_bytes():
    text = _ref("features")
    rows = _rows(text)
    assert tuple(rows[0][1:]) == FEATURE_NAMES
    fvs = [SimpleNamespace(as_dict=lambda r=r: dict(zip(FEATURE_NAMES, map(float, r[1:]))))
           for r in rows[1:]]
    assert formats.features_csv(fvs, [r[0] for r in rows[1:]]) == text


def test_greedy_and_anneal_csv_reproduce_the_reference_bytes():
    text = _ref("greedy")
    per = [SimpleNamespace(order=int(r[0]), indices=_indices(r[2]), value=float(r[3]))
           for r in _rows(text)[1:]]
    assert formats.greedy_csv(SimpleNamespace(per_order=per), _names()) == text
    text = _ref("anneal")
    rows = _rows(text)[1:]

    def mask(r):
        m = np.zeros(9, dtype=bool)
        m[list(_indices(r[3]))] = True
        return m

    state = SimpleNamespace(best_mask=mask(rows[0]), best_energy=float(rows[0][4]),
                            masks=np.stack([mask(r) for r in rows[1:]]),
                            energies=np.array([float(r[4]) for r in rows[1:]]))
    ident = SimpleNamespace(value_of=lambda e: e)
    assert formats.anneal_csv(state, ident, _names()) == text


# -------------------------------------------------------------- GPU ----

def _close(got_text, ref_text, float_cols):
    got, ref = _rows(got_text), _rows(ref_text)
    assert got[0] == ref[0] and len(got) == len(ref)
    for g, r in zip(got[1:], ref[1:]):
        for c, (a, b) in enumerate(zip(g, r)):
            if c in float_cols:
                assert float(a) == pytest.approx(float(b), rel=1e-9, abs=1e-11), (c, g, r)
            else:
                assert a == b, (c, g, r)


@pytest.mark.gpu
def test_pipeline_from_data_files_matches_the_reference_cli():
    names, datas = formats.load_datasets(IN)
    var = datas[0].column_names
    covs = formats.covset_from_data(datas)
    top = hoi.scan(covs, 3, 9, hoi.TopK("o", "min", 15), bias_correct=True)
    _close(formats.topk_csv(top, names, var), _ref("top"), {4, 5, 6, 7})
    hist = hoi.scan(covs, 2, 6, hoi.Histogram("tc", 12, 0.0, 2.0))
    _close(formats.histogram_csv(hist, names), _ref("hist"), {1, 2})
    feats = hoi.extract_features(covs)
    _close(formats.features_csv(feats, names), _ref("features"), set(range(1, 22)))
    spec = hoi.ObjectiveSpec(measure="o", direction="min")
    g = hoi.greedy(covs, spec, 3, 6, kappa=5, seed=0)
    _close(formats.greedy_csv(g, var), _ref("greedy"), {3})
    spec = hoi.ObjectiveSpec(measure="dtc", direction="max")
    sched = hoi.AnnealSchedule(temp0=None, alpha=0.99, max_iters=60, patience=0,
                               mode="across-orders", min_order=3, max_order=7)
    st = hoi.anneal(covs, spec, sched, kappa=6, seed=3)
    _close(formats.anneal_csv(st, spec, var), _ref("anneal"), {4})
