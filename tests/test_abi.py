"""CPU: the C-ABI library builds/loads and exports exactly what include/*.h declares."""
import ctypes as C
import os
import re

import numpy as np
import pytest
from conftest import REPO

HEADER = os.path.join(REPO, "include", "qcldpc_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"QC_API\s+[\w\s\*]+?\b((?:qc64|qc|cc)_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 20
    for must in ("qc_plan_create_qc", "qc_cnu", "qc_vnu", "qc_decode", "qc_channel", "cc_slot"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1204_0334_b200 import _lib
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(declared())


def test_argument_errors_map_to_value_error():
    from paper_1204_0334_b200 import _lib
    lib = _lib.load()
    sh = np.array([[0, 1], [2, 9]], dtype=np.int64)
    h = C.c_void_p()
    rc = lib.qc_plan_create_qc(sh.ctypes.data_as(C.c_void_p), 2, 2, 5, C.byref(h))
    assert rc < 0 and b"shifts" in lib.qc_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
    rc = lib.cc_plan_create(sh.ctypes.data_as(C.c_void_p), 1, 3, 11, C.byref(h))
    assert rc < 0 and b"gcd" in lib.qc_last_error()
    assert lib.qc_decode_work_words(None, 64) == 64          # no plan: header words only
    assert lib.qc_cnu(None, 33, None, None, None) < 0          # gamma not a multiple of 32


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_1204_0334_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_1204_0334_b200 import _lib
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(_lib.LibraryMissing):
        _lib.load(str(tmp_path / "nope.so"))
