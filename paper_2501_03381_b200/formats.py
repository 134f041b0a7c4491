"""Data formats either side of the path.

Input: the reference CLI's data files -- UTF-8 CSV, a header row of
variable names, one sample per row; a directory of CSVs with identical
headers is one dataset per file, in filename order
(ref:cli.py:79-120).  Output: the CSV texts its subcommands write for
TopK / Histogram scans, feature fingerprints and the greedy / anneal
optimisers (ref:cli.py:52-62, 206-248, 272-279, 318-331, 355-359): floats
as Python's shortest round-trip repr, n-plets as comma-joined variable
names plus a hex bit mask (bit i = column i), "\\n" line ends.  The CLI
itself (argument parsing, exit codes) is out of scope; these are the
formats, so files written here diff cleanly against the reference's.

The full output of an exhaustive scan has no CSV form (34 GB at N = 30):
that is ``DeviceScan.save`` / ``read_scan``.
"""

from __future__ import annotations

import csv
import io
from pathlib import Path

import numpy as np

from .copula_core import CovSet, DataMatrix, copula_transform, estimate_covariance
from .errors import InvalidData

__all__ = ["read_csv", "load_datasets", "covset_from_data", "topk_csv", "histogram_csv",
           "features_csv", "greedy_csv", "anneal_csv", "float_text", "mask_hex"]


def float_text(x) -> str:
    """Shortest decimal that round-trips the float64 (ref:cli.py:52-54)."""
    return repr(float(x))


def mask_hex(indices) -> str:
    """Hex bit mask of an n-plet, bit i = variable i (ref:cli.py:57-62)."""
    return hex(sum(1 << int(i) for i in set(int(v) for v in indices)))


def _table(header, rows) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(header)
    w.writerows(rows)
    return buf.getvalue()


def _nplet_fields(indices, variable_names):
    return [",".join(variable_names[i] for i in indices), mask_hex(indices)]


# ------------------------------------------------------------------ input --

def read_csv(path) -> DataMatrix:
    """One data file -> DataMatrix with its header as column names
    (ref:cli.py:79-97: same errors for bad UTF-8, short files, ragged rows
    and non-numeric fields)."""
    path = Path(path)
    try:
        with open(path, newline="", encoding="utf-8") as fh:
            lines = list(csv.reader(fh))
    except UnicodeDecodeError as e:
        raise InvalidData(f"{path}: not valid UTF-8 ({e})") from None
    if len(lines) < 2:
        raise InvalidData(f"{path}: need a header row and at least one data row")
    names, body = lines[0], lines[1:]
    for r, row in enumerate(body):
        if len(row) != len(names):
            raise InvalidData(f"{path}: row {r + 2} has {len(row)} fields, expected {len(names)}")
    try:
        values = np.array([[float(x) for x in row] for row in body], dtype=np.float64)
    except ValueError:
        bad = next(r for r, row in enumerate(body) if not _numeric(row))
        raise InvalidData(f"{path}: non-numeric value in row {bad + 2}") from None
    return DataMatrix(values.reshape(len(body), len(names)), column_names=names)


def _numeric(row) -> bool:
    try:
        [float(x) for x in row]
    except ValueError:
        return False
    return True


def load_datasets(input_path):
    """(dataset names, [DataMatrix]) from a CSV file or a directory of CSVs
    with identical headers, files in name order (ref:cli.py:100-116)."""
    path = Path(input_path)
    if path.is_dir():
        files = sorted(path.glob("*.csv"), key=lambda p: p.name)
        if not files:
            raise InvalidData(f"{path}: no .csv files in directory")
    elif path.is_file():
        files = [path]
    else:
        raise InvalidData(f"{input_path}: no such file or directory")
    datas = [read_csv(f) for f in files]
    for f, dm in zip(files[1:], datas[1:]):
        if dm.column_names != datas[0].column_names:
            raise InvalidData(f"{f}: header differs from {files[0]}")
    return [f.stem for f in files], datas


def covset_from_data(datas) -> CovSet:
    """Raw data -> copula -> covariance per dataset (ref:cli.py:119-120)."""
    return CovSet([estimate_covariance(copula_transform(dm)) for dm in datas])


# ----------------------------------------------------------------- output --

def topk_csv(result, dataset_names, variable_names) -> str:
    """``scan(..., TopK)`` result (one entry list per dataset) as the scan
    subcommand's CSV (ref:cli.py:224-236)."""
    rows = [[name, e.order, *_nplet_fields(e.indices, variable_names),
             *(float_text(v) for v in (e.tc, e.dtc, e.o, e.s))]
            for name, entries in zip(dataset_names, result) for e in entries]
    return _table(["dataset", "order", "variables", "mask", "tc", "dtc", "o", "s"], rows)


def histogram_csv(result, dataset_names) -> str:
    """``scan(..., Histogram)`` result (edges, counts (D, bins)) as the scan
    subcommand's CSV (ref:cli.py:237-244)."""
    edges, counts = result
    rows = [[name, float_text(edges[b]), float_text(edges[b + 1]), int(counts[d, b])]
            for d, name in enumerate(dataset_names) for b in range(counts.shape[1])]
    return _table(["dataset", "bin_lo", "bin_hi", "count"], rows)


def features_csv(features, dataset_names) -> str:
    """``extract_features`` result as the features subcommand's CSV, one row
    per dataset in FEATURE_NAMES order (ref:cli.py:355-359)."""
    from .scanner import FEATURE_NAMES
    rows = [[name, *(float_text(fv.as_dict()[c]) for c in FEATURE_NAMES)]
            for name, fv in zip(dataset_names, features)]
    return _table(["dataset", *FEATURE_NAMES], rows)


def greedy_csv(result, variable_names) -> str:
    """``greedy`` result, one row per order (ref:cli.py:272-279)."""
    rows = [[e.order, *_nplet_fields(e.indices, variable_names), float_text(e.value)]
            for e in result.per_order]
    return _table(["order", "variables", "mask", "value"], rows)


def anneal_csv(state, spec, variable_names) -> str:
    """``anneal`` state: the best mask, then every chain's current mask,
    values in the objective's sign convention (ref:cli.py:318-331)."""
    def row(kind, mask, energy):
        idx = tuple(int(v) for v in np.flatnonzero(mask))
        return [kind, len(idx), *_nplet_fields(idx, variable_names),
                float_text(spec.value_of(energy))]

    rows = [row("best", state.best_mask, state.best_energy)]
    rows += [row(f"chain_{c}", state.masks[c], float(state.energies[c]))
             for c in range(state.masks.shape[0])]
    return _table(["kind", "order", "variables", "mask", "value"], rows)
