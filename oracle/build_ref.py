"""Install the REAL reference package into oracle/_ref (TEST INFRASTRUCTURE ONLY).

    python -m oracle.build_ref          # also run by __graft_entry__.build()

The reference (`qcldpc`, /root/reference/pkg) is pure Python/numpy: there is
nothing to compile, so "building" it means installing it.  The tree under
/root/reference is read-only, so it is copied to a temporary directory first
and installed from there (`pip install --no-index --no-build-isolation
--no-deps --target oracle/_ref/site`); its own test files are copied to
oracle/_ref/ref_tests.  oracle/_ref is git-ignored (reference sources never
enter this repository's history) but NOT gpurun-ignored, so it travels to the
GPU box next to the built library and serves:

* tests/test_ref_conformance.py -- the reference's own test suite run against
  paper_1204_0334_b200 aliased as `qcldpc`;
* bench.py --impl reference / cpu_baseline -- the reference's own CPU
  decoder timed on the host cores (kind "reference").

Nothing on a GPU box reads /root/reference: when oracle/_ref is missing the
conformance test skips and the bench falls back to the oracle port.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
OUT = os.path.join(HERE, "_ref")
SITE = os.path.join(OUT, "site")
TESTS = os.path.join(OUT, "ref_tests")


def available() -> bool:
    """True when the installed reference package is present."""
    return os.path.isfile(os.path.join(SITE, "qcldpc", "bp.py"))


def site_dir() -> str:
    return SITE


def build(force: bool = False) -> bool:
    """Install the reference into oracle/_ref; False when /root/reference is absent."""
    if not os.path.isdir(REF_PKG):
        return available()
    if available() and os.path.isdir(TESTS) and not force:
        return True
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("build", "*.egg-info", "__pycache__"))
        for root, dirs, files in os.walk(src):          # copies keep the read-only modes
            os.chmod(root, 0o755)
            for f in files:
                os.chmod(os.path.join(root, f), 0o644)
        if os.path.isdir(SITE):
            shutil.rmtree(SITE)
        r = subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                            "--no-build-isolation", "--no-deps", "--target", SITE, src],
                           capture_output=True, text=True, cwd=tmp)
        if r.returncode != 0:
            raise RuntimeError(f"installing the reference failed:\n{r.stdout}\n{r.stderr}")
        if os.path.isdir(TESTS):
            shutil.rmtree(TESTS)
        shutil.copytree(os.path.join(src, "tests"), TESTS,
                        ignore=shutil.ignore_patterns("__pycache__"))
    return available()


if __name__ == "__main__":
    print("oracle/_ref:", "ok" if build(force="-f" in sys.argv) else "reference not available")
