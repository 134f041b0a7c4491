"""CSV fixtures from the REAL reference CLI (ref:cli.py) for the data
formats either side of the path (paper_2501_03381_b200/formats.py).

Run in the build container only (imports /root/reference):

    python tests/golden/make_golden_csv.py

Writes tests/golden/csv/in/*.csv (three seeded datasets, 9 variables,
120 samples, written with repr floats) and tests/golden/csv/out/*.csv, the
reference CLI's own output for: a TopK scan, a Histogram scan, the feature
fingerprint, greedy and anneal.  The commands are recorded in
tests/golden/csv/commands.json.
"""

import json
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "csv"
sys.path.insert(0, "/root/reference/pkg/src")

from hoi import cli  # noqa: E402  (the reference)

NAMES = ["amyg_l", "amyg_r", "hipp_l", "hipp_r", "pfc_m", "pfc_l", "ins_a", "acc", "thal"]

COMMANDS = {
    "top": ["scan", "--orders", "3:all", "--reduce", "top:15:min:o", "--bias-correct"],
    "hist": ["scan", "--orders", "2:6", "--reduce", "hist:tc:12:0:2"],
    "features": ["features"],
    "greedy": ["greedy", "--measure", "o", "--direction", "min", "--start-order", "3",
               "--target-order", "6", "--kappa", "5"],
    "anneal": ["anneal", "--measure", "dtc", "--direction", "max", "--iters", "60",
               "--kappa", "6", "--seed", "3", "--max-order", "7"],
}


def write_inputs(d: Path):
    rng = np.random.default_rng(2025)
    for name in ("ds_a", "ds_b", "ds_c"):
        a = rng.standard_normal((9, 9))
        c = a @ a.T
        c /= np.sqrt(np.outer(np.diag(c), np.diag(c)))
        x = rng.standard_normal((120, 9)) @ np.linalg.cholesky(c).T
        x[:, 4] = np.exp(x[:, 4])                   # a skewed marginal (the copula matters)
        lines = [",".join(NAMES)] + [",".join(repr(float(v)) for v in row) for row in x]
        (d / f"{name}.csv").write_text("\n".join(lines) + "\n", encoding="utf-8")


def main():
    if HERE.exists():
        shutil.rmtree(HERE)
    (HERE / "in").mkdir(parents=True)
    (HERE / "out").mkdir()
    write_inputs(HERE / "in")
    for key, argv in COMMANDS.items():
        rc = cli.main([*argv, "--input", str(HERE / "in"), "--out", str(HERE / "out" / f"{key}.csv")])
        assert rc == 0, (key, rc)
    (HERE / "commands.json").write_text(json.dumps(COMMANDS, indent=1) + "\n")
    print("wrote", sorted(p.name for p in (HERE / "out").iterdir()))


if __name__ == "__main__":
    main()
