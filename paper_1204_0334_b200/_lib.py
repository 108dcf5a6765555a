"""ctypes boundary to the CUDA library (include/qcldpc_b200.h).

There is no CPU fallback: if `lib/libqcldpc_b200.so` is missing or CUDA is not
available, every compute entry point raises.  Argument errors reported by the
library (negative return codes) become ValueError, runtime/CUDA errors
(positive codes) RuntimeError -- the same exception classes the reference
raises (bp.py:229-230, convolutional.py:192-195, 222-226).
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QCB_LIB_PATH") or os.path.join(HERE, "lib", "libqcldpc_b200.so")  # override: A/B builds

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_d = C.c_double

# name -> (restype, argtypes); mirrors include/qcldpc_b200.h
SIGNATURES = {
    "qc_last_error": (C.c_char_p, []),
    "qc_abi_version": (_i, []),
    "qc_plan_create_qc": (_i, [_p, _i, _i, _i, C.POINTER(_p)]),
    "qc_plan_create_csr": (_i, [_i, _i, _p, _p, C.POINTER(_p)]),
    "qc_plan_destroy": (None, [_p]),
    "qc_plan_dims": (_i, [_p, _p]),
    "qc_init": (_i, [_p, _i, _p, _p, _p]),
    "qc_cnu": (_i, [_p, _i, _p, _p, _p]),
    "qc_vnu": (_i, [_p, _i, _p, _p, _p, _p, _p, _p]),
    "qc_cnu_ex": (_i, [_p, _i, _i, _p, _p, _p, _p]),
    "qc_vnu_ex": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p]),
    "qc_syndrome": (_i, [_p, _i, _p, _p, _p]),
    "qc_hard_bits": (_i, [_p, _i, _p, _p, _p]),
    "qc_bit_errors": (_i, [_p, _i, _p, _p, _p]),
    "qc_decode_work_words": (C.c_size_t, [_p, _i]),
    "qc_decode_records_offset": (C.c_size_t, [_i]),
    "qc_decode": (_i, [_p, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "qc_decode_es": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "qc_decode_es_scratch_words": (C.c_size_t, [_p, _i]),
    "qc_decode_es_launches": (_i, [_p, _i, _i]),
    "qc_agg_check": (_i, [_p, _i, _i, _p, _p, _p, _p]),
    "qc_agg_var": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p]),
    "qc_agg_fused": (_i, [_p, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p]),
    "qc_decode_launches": (_i, [_p, _i, _i, _i]),
    "qc_lane_major_to_host": (_i, [_i, _i, _i, _p, _p, _p, _p, _p, _p]),
    "qc_llr_from_host": (_i, [_i, _i, _i, _p, _p, _d, _p, _p]),
    "qc_lane_major": (_i, [_i, _i, _i, _p, _p, _p, _p]),
    "qc_lane_major_f32": (_i, [_i, _i, _i, _p, _p, _p, _p]),
    "qc_llr_from_lane_major": (_i, [_i, _i, _i, _p, _d, _p, _p]),
    "qc_host_create": (_i, [_p, _i, _i, _i, _i, C.POINTER(_p)]),
    "qc_host_destroy": (None, [_p]),
    "qc_host_dims": (_i, [_p, _p]),
    "qc_host_is_pinned": (_i, [_p, C.c_size_t]),
    "qc_host_decode": (_i, [_p, _p, _i, _d, _p, _p, _p, _p]),
    "qc_rc_state_bytes": (C.c_size_t, [_i]),
    "qc_rc_init": (_i, [_i, _i64, _p, _p]),
    "qc_rc_ticks": (_i, [_p, _i, _i, _i, _i, _i, _i64, _i64, _u64, _u64, _u64, _d, _i, _p, _p, _p, _p, _p, _p]),
    "qc_rc_next_id": (_i, [_i, _p, _p, _p]),
    "qc64_init": (_i, [_p, _i, _p, _p, _p]),
    "qc64_cnu": (_i, [_p, _i, _p, _p, _p]),
    "qc64_vnu": (_i, [_p, _i, _p, _p, _p, _p, _p, _p]),
    "qc64_hard_bits": (_i, [_p, _i, _p, _p, _p]),
    "qc64_decode": (_i, [_p, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "qc64_lane_major": (_i, [_i, _i, _i, _p, _p, _p, _p]),
    "qc64_mu_from_lane_major": (_i, [_i, _i, _i, _p, _d, _i, _p, _p]),
    "qc_channel": (_i, [_u64, _u64, _u64, _u64, _i, _i, _d, _p, _p, _p, _p]),
    "qc_channel_dev": (_i, [_u64, _u64, _p, _u64, _i, _i, _d, _p, _p]),
    "qc_lane_advance": (_i, [_p, _u64, _p]),
    "qc_batch_counts": (_i, [_i, _i, _p, _p, _p]),
    "cc_plan_create": (_i, [_p, _i, _i, _i, C.POINTER(_p)]),
    "cc_plan_destroy": (None, [_p]),
    "cc_plan_dims": (_i, [_p, _p]),
    "cc_slot": (_i, [_p, _i, _i, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "cc_slot_part": (_i, [_p, _i, _i, _i64, _p, _p, _p, _p, _p, _p, _i, _i, _i, _p]),
    "cc_advance": (_i, [_p, _i64, _p]),
    "cc_fold": (_i, [_p, _i, _p]),
    "cc_channel": (_i, [_p, _u64, _u64, _u64, _p, _i64, _p, _i, _d, _p, _p]),
    "cc_channel_frames": (_i, [_p, _u64, _u64, _u64, _p, _i64, _i, _i, _d, _p, _p]),
    "cc_slot_ahead": (_i, [_p, _i, _i, _i64, _p, _p, _p, _p, _i, _p, _p, _p]),
}

_LIB = None


class LibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and bind the shared library; raises if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not built: run `python -m paper_1204_0334_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().qc_last_error().decode(errors="replace")
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    """Call an int-returning entry point and map its return code."""
    check(getattr(load(), name)(*args))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(device=None) -> int:
    """cudaStream_t of torch's current stream (on `device`, default the current
    device) -- the raw-stream query, without torch.cuda.current_stream()'s
    per-call device resolution (~13 us, a third of a small push_frame)."""
    import torch
    if device is None:
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream(device).cuda_stream
