"""`import hoi` -> this repository's drop-in, for the reference's own tests.

The reference's conformance modules (installed unmodified into
oracle/_ref/tests by oracle/build_ref.py) import `hoi`, `hoi.nplet_engine`
and `hoi.cli`.  This shim registers:

* `hoi`, `hoi.copula_core`, `hoi.nplet_engine`, `hoi.measures`,
  `hoi.scanner`, `hoi.optimizers`, `hoi.errors` -> paper_2501_03381_b200
  (the product, whose numeric path is libhoib200.so on the GPU);
* the fixture generators the tests import from `hoi` (`r_system_cov`,
  `s_system_cov`, `block_concat`, `sample_gaussian`, `PgmBlock`, `PgmSpec`;
  ref synthetic.py, out of scope for the engine) -> the
  reference's own functions, with their containers converted to the
  product's `CovarianceMatrix` / `DataMatrix` at the boundary;
* `hoi.cli` -> a stub (the CLI is out of scope; the test that drives it,
  acceptance criterion 9, is not collected).

Test infrastructure only: nothing in the product imports this.
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF_TESTS = REPO / "oracle" / "_ref" / "tests"


def available() -> bool:
    return (REPO / "oracle" / "_ref" / "site" / "hoi" / "__init__.py").exists() and \
        (REF_TESTS / "reference.py").exists()


def install():
    if "hoi" in sys.modules and getattr(sys.modules["hoi"], "_is_b200_shim", False):
        return sys.modules["hoi"]
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "oracle"))
    import build_ref

    import paper_2501_03381_b200 as prod
    from paper_2501_03381_b200 import (copula_core, errors, measures, nplet_engine, optimizers,
                                       scanner)

    ref = build_ref.import_reference()
    rsyn = sys.modules["hoi_ref.synthetic"]
    rcc = sys.modules["hoi_ref.copula_core"]

    def to_prod_cov(c):
        if isinstance(c, copula_core.CovarianceMatrix):
            return c
        return copula_core.CovarianceMatrix(np.array(c.sigma, dtype=np.float64),
                                            n_samples_used=int(c.n_samples_used),
                                            block_slices=getattr(c, "block_slices", None))

    def to_ref_cov(c):
        if isinstance(c, rcc.CovarianceMatrix):
            return c
        if isinstance(c, copula_core.CovarianceMatrix):
            return rcc.CovarianceMatrix(np.array(c.sigma), n_samples_used=c.n_samples_used,
                                        block_slices=c.block_slices)
        return c

    def r_system_cov(n_sources, c):
        return to_prod_cov(rsyn.r_system_cov(n_sources, c))

    def s_system_cov(n_sources, c):
        return to_prod_cov(rsyn.s_system_cov(n_sources, c))

    def block_concat(blocks):
        return to_prod_cov(rsyn.block_concat([to_ref_cov(b) for b in blocks]))

    def sample_gaussian(cov, t, seed):
        return copula_core.DataMatrix(rsyn.sample_gaussian(to_ref_cov(cov), t, seed).values)

    class PgmBlock(rsyn.PgmBlock):
        def cov(self):
            return to_prod_cov(super().cov())

    class PgmSpec(rsyn.PgmSpec):
        def __post_init__(self):
            self.blocks = [b if isinstance(b, PgmBlock) else PgmBlock(b.kind, b.n_sources, b.c)
                           for b in self.blocks]
            super().__post_init__()

        def build(self):
            return to_prod_cov(rsyn.block_concat([rsyn.PgmBlock.cov(b) for b in self.blocks]))

        @classmethod
        def from_json(cls, text):
            return cls(rsyn.PgmSpec.from_json(text).blocks)

    hoi = types.ModuleType("hoi")
    hoi.__dict__.update({k: getattr(prod, k) for k in dir(prod) if not k.startswith("__")})
    fixtures = dict(r_system_cov=r_system_cov, s_system_cov=s_system_cov,
                    block_concat=block_concat, sample_gaussian=sample_gaussian,
                    PgmBlock=PgmBlock, PgmSpec=PgmSpec)
    hoi.__dict__.update(fixtures)
    hoi.__path__ = []
    hoi._is_b200_shim = True
    synthetic = types.ModuleType("hoi.synthetic")
    synthetic.__dict__.update(fixtures)
    synthetic.ground_truth_hoi = prod.ground_truth_hoi

    cli = types.ModuleType("hoi.cli")

    def main(argv=None):
        raise NotImplementedError("the reference CLI is out of scope for the B200 engine")

    cli.main = main
    sys.modules.update({
        "hoi": hoi, "hoi.copula_core": copula_core, "hoi.nplet_engine": nplet_engine,
        "hoi.measures": measures, "hoi.scanner": scanner, "hoi.optimizers": optimizers,
        "hoi.errors": errors, "hoi.synthetic": synthetic, "hoi.cli": cli,
    })
    for name in ("copula_core", "nplet_engine", "measures", "scanner", "optimizers", "errors",
                 "synthetic", "cli"):
        setattr(hoi, name, sys.modules[f"hoi.{name}"])
    if str(REF_TESTS) not in sys.path:
        sys.path.insert(0, str(REF_TESTS))
    return hoi
