"""pytest plugin: run the reference's own test suite against paper_1204_0334_b200.

    python -m pytest oracle/_ref/ref_tests -p ref_suite_shim      (tests/ on PYTHONPATH)

Maps the reference package name `qcldpc` and its submodules onto the drop-in
(`qcldpc.bp` -> paper_1204_0334_b200.bp, ...), so the unmodified reference
tests (installed by oracle/build_ref.py into git-ignored oracle/_ref) exercise
the B200 path through exactly the imports a user of the reference writes.
Two names are test oracles the drop-in does not ship (qcldpc.reference:
exact_posterior_llr, reference_window_decoder); they map to oracle/reference.py.
`qcldpc.cli` is out of scope and is left unmapped.
QCLDPC_B200_PRECISION selects the float32 production path or the float64
conformance build of the block decoder.
"""

import importlib
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
for k in [k for k in sys.modules if k == "qcldpc" or k.startswith("qcldpc.")]:
    del sys.modules[k]

import paper_1204_0334_b200 as _pkg  # noqa: E402
from oracle import reference as _oref  # noqa: E402

sys.modules["qcldpc"] = _pkg
for _name in ("bp", "codes", "convolutional", "channel", "harness", "data"):
    sys.modules["qcldpc." + _name] = importlib.import_module("paper_1204_0334_b200." + _name)
sys.modules["qcldpc.reference"] = _oref
_pkg.reference = _oref
