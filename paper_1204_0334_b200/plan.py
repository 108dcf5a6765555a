"""Device plans (immutable, shared) and small device-buffer helpers."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib

# Message precision of the block decoder API: "float32" (production: phi-form
# fp32 kernels) or "float64" (conformance build: the reference's tanh rule in
# float64, csrc/block64.cu).  Campaigns and the stream decoder are fp32.
_PRECISION = os.environ.get("QCLDPC_B200_PRECISION", "float32")


def set_precision(p: str) -> None:
    global _PRECISION
    if p not in ("float32", "float64"):
        raise ValueError("precision must be 'float32' or 'float64'")
    _PRECISION = p


def get_precision() -> str:
    return _PRECISION


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1204_0334_b200 needs a CUDA device (no CPU fallback)")
    _lib.load()
    return torch


def pad32(gamma: int) -> int:
    return max(32, (gamma + 31) // 32 * 32)


def np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class BlockPlan:
    """qc_plan handle for an EdgeLayout (codes.py EdgeLayout.plan())."""

    def __init__(self, layout):
        require_cuda()
        lib = _lib.load()
        h = C.c_void_p()
        exp = layout.qc
        if exp is not None and int((exp.shifts < 0).sum()) == 0:
            sh = np.ascontiguousarray(exp.shifts, dtype=np.int64)
            _lib.check(lib.qc_plan_create_qc(np_ptr(sh), sh.shape[0], sh.shape[1], int(exp.p),
                                             C.byref(h)))
        else:
            ptr = np.ascontiguousarray(layout.check_ptr, dtype=np.int64)
            ev = np.ascontiguousarray(layout.edge_var, dtype=np.int64)
            if ev.size == 0:
                ev = np.zeros(1, np.int64)
            _lib.check(lib.qc_plan_create_csr(layout.n_vars, layout.n_checks, np_ptr(ptr),
                                              np_ptr(ev), C.byref(h)))
        self.handle = h
        dims = np.zeros(6, np.int64)
        _lib.check(lib.qc_plan_dims(h, np_ptr(dims)))
        self.N, self.M, self.E, self.dc_max, self.dv_max, self.check_regular = (int(x) for x in dims)
        if self.E != layout.edge_count or self.N != layout.n_vars:
            raise RuntimeError("device plan does not match the edge layout")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib._LIB is not None:
            try:
                _lib._LIB.qc_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


class StreamPlan:
    """cc_plan handle of an LdpcccCode."""

    def __init__(self, exp):
        require_cuda()
        lib = _lib.load()
        sh = np.ascontiguousarray(exp.shifts, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(lib.cc_plan_create(np_ptr(sh), sh.shape[0], sh.shape[1], int(exp.p), C.byref(h)))
        self.handle = h
        d = np.zeros(8, np.int64)
        _lib.check(lib.cc_plan_dims(h, np_ptr(d)))
        self.lam, self.ms, self.c, self.cb, self.E, self.sj, self.sl, self.p = (int(x) for x in d)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib._LIB is not None:
            try:
                _lib._LIB.cc_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


def lane_words(active: np.ndarray | None, gamma_pad: int):
    """(gamma,) bool mask -> (gamma_pad/32,) uint32 words (padding lanes inactive)."""
    if active is None:
        return None
    a = np.zeros(gamma_pad, dtype=bool)
    a[: active.size] = np.asarray(active, dtype=bool)
    return np.packbits(a.reshape(-1, 32), axis=1, bitorder="little").view("<u4").reshape(-1).astype(np.uint32)


def unpack_planes(words: np.ndarray, gamma: int) -> np.ndarray:
    """(n, W) uint32 hard-bit planes -> (n, gamma) uint8 bits."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    bits = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :gamma].astype(np.uint8)
