"""Install the real reference into oracle/_ref/ (test infrastructure only).

The reference (`/root/reference/pkg`, the pure-Python `hoi` package) is the
checker for this repository's GPU path, never part of it.  This recipe
installs it, unmodified, with pip (no index, no dependencies resolved:
numpy and scipy are already in the image) into

    oracle/_ref/site/hoi/         the reference package (imported as `hoi_ref`
                                  by tests/ref_conformance and bench.py's
                                  reference arm)
    oracle/_ref/tests/            the reference's own test modules and its
                                  independent oracle `reference.py`, run
                                  against the drop-in by tests/ref_conformance

`oracle/_ref/` is git-ignored (no reference source enters the history) but
not gpurun-ignored, so the installed copy travels to the GPU box with the
snapshot, like the built libhoib200.so.  `/root/reference` itself is only
read here, in the build container.  The install runs from a copy under
/tmp because setuptools writes build metadata next to the sources and the
reference tree is read-only.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "_ref"


def available() -> bool:
    return (REF / "src" / "hoi" / "__init__.py").exists()


def installed() -> bool:
    return (OUT / "site" / "hoi" / "__init__.py").exists() and (OUT / "tests" / "reference.py").exists()


def build(force: bool = False) -> bool:
    """Install the reference and copy its tests; False when the reference
    tree is absent (the GPU box), True when oracle/_ref is ready."""
    if installed() and not force:
        return True
    if not available():
        return installed()
    site = OUT / "site"
    tests = OUT / "tests"
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF, src, ignore=shutil.ignore_patterns("__pycache__", "*.egg-info", "build"))
        stage = Path(tmp) / "site"
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(stage), str(src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}")
        if site.exists():
            shutil.rmtree(site)
        site.parent.mkdir(parents=True, exist_ok=True)
        shutil.copytree(stage, site)
    if tests.exists():
        shutil.rmtree(tests)
    tests.mkdir(parents=True)
    for f in sorted((REF / "tests").glob("*.py")):
        shutil.copy2(f, tests / f.name)
    (OUT / "SOURCE.txt").write_text(
        "Installed by oracle/build_ref.py from /root/reference/pkg (unmodified). "
        "Test infrastructure only; git-ignored.\n")
    return True


def import_reference():
    """The installed reference package as module `hoi_ref` (its own
    package-relative imports resolve inside it)."""
    import importlib.util

    if "hoi_ref" in sys.modules:
        return sys.modules["hoi_ref"]
    init = OUT / "site" / "hoi" / "__init__.py"
    if not init.exists():
        raise ImportError("oracle/_ref is not installed (run oracle/build_ref.py here)")
    spec = importlib.util.spec_from_file_location(
        "hoi_ref", init, submodule_search_locations=[str(init.parent)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["hoi_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    ok = build(force="--force" in sys.argv)
    print(f"oracle/_ref ready: {ok} ({OUT})")
