"""Batched sum-product decoding of LDPC block codes on B200.

Drop-in for /root/reference/pkg/src/qcldpc/bp.py (same names, argument
meaning, shapes and exceptions).  Messages live on the GPU in the paper's
edge-major Gamma-codeword packages, fp32; every update is a hand-written
sm_100a kernel reached through the C ABI (include/qcldpc_b200.h).  There is
no CPU path: without the library or a GPU these functions raise.

Numerics: the check rule runs in the log (phi) domain in fp32 (see
csrc/phi.cuh); against the float64 reference a single update agrees to
|delta| <= 1e-4 * max(|ref|, 1), and decisions / syndromes / error counts of
full decodes are checked bit-exact by tests/test_gpu_block.py.

`decode_batch` / `decode_llr_batch` run on `HostDecoder`, the native
host-buffer pipeline (csrc/host_pipe.cu): lane chunks rotate over CUDA
streams so PCIe copies overlap the graph-replayed decode, page-locked arrays
are DMA'd in place.  `BlockDecoder` is the device-resident engine (inputs and
outputs in HBM) used by the campaign drivers and the float64 build.
"""

from __future__ import annotations

import dataclasses
import os
import threading

import numpy as np

from . import _lib
from .codes import EdgeLayout
from .plan import get_precision, lane_words, pad32, require_cuda, unpack_planes

__all__ = [
    "L_MAX", "TANH_CLAMP", "MessageBatch", "DecodeResult", "channel_llrs", "init_messages",
    "check_node_update", "variable_node_update", "hard_decision_and_syndrome",
    "decode_llr_batch", "decode_batch", "BlockDecoder", "HostDecoder", "host_array",
    "set_pinned_outputs", "release_pinned_cache",
]

L_MAX = 50.0
TANH_CLAMP = 1e-12


def channel_llrs(y: np.ndarray, sigma: float) -> np.ndarray:
    """Channel LLRs 2y/sigma^2 clipped at +-L_MAX (host helper, bp.py:54-56)."""
    return np.clip(2.0 * np.asarray(y, dtype=np.float64) / (sigma * sigma), -L_MAX, L_MAX)


def _stream():
    return _lib.stream_handle()


class MessageBatch:
    """Per-edge message packages of gamma lock-step codewords, resident on the GPU.

    `packages` behaves like the reference's writable (E, gamma) float64 view
    (bp.py:82-84): the first access copies the device store into a host
    mirror; later accesses return the same array (O(1), so per-edge loops such
    as test_acceptance.py:207 stay cheap).  While a mirror exists the updates
    are write-through: check_node_update / variable_node_update upload it
    first (caller writes take effect) and refresh it in place afterwards, so a
    held reference sees the new packages exactly as a numpy view would.
    `packages_device` is the live (E, gamma) device view (no copies).
    """

    def __init__(self, layout: EdgeLayout, mu: np.ndarray):
        torch = require_cuda()
        mu = np.asarray(mu, dtype=np.float64)
        if mu.ndim != 2 or mu.shape[0] != layout.n_vars:
            raise ValueError(f"mu must be (N={layout.n_vars}, gamma), got {mu.shape}")
        self.layout = layout
        self.gamma = mu.shape[1]
        self.mu = mu
        self._gp = pad32(self.gamma)
        self.fp64 = get_precision() == "float64"
        self._host = None
        dt = torch.float64 if self.fp64 else torch.float32
        dev = torch.device("cuda", torch.cuda.current_device())
        m = torch.full((layout.n_vars, self._gp), L_MAX, dtype=dt)
        m[:, : self.gamma] = torch.from_numpy(mu).to(dt)
        self._mu_dev = m.to(dev)
        self._msgs = torch.zeros((max(layout.edge_count, 1), self._gp), dtype=dt, device=dev)
        if layout.edge_count:
            _lib.call("qc64_init" if self.fp64 else "qc_init", layout.plan().handle, self._gp,
                      self._mu_dev.data_ptr(), self._msgs.data_ptr(), _stream())

    @property
    def packages_device(self):
        return self._msgs[: self.layout.edge_count, : self.gamma]

    @property
    def packages(self) -> np.ndarray:
        if self._host is None:
            self._host = self.packages_device.double().cpu().numpy()
        return self._host

    def _before_update(self):
        """Push caller writes made through the host mirror to the device."""
        if self._host is not None:
            import torch
            self.packages_device.copy_(torch.from_numpy(self._host))

    def _after_update(self):
        """Refresh the host mirror in place (view semantics)."""
        if self._host is not None:
            import torch
            torch.from_numpy(self._host).copy_(self.packages_device.double())


@dataclasses.dataclass
class DecodeResult:
    """hard_bits / posteriors lane-major (gamma, N); syndrome_ok, iterations_run (gamma,)."""

    hard_bits: np.ndarray
    posteriors: np.ndarray
    syndrome_ok: np.ndarray
    iterations_run: np.ndarray


def init_messages(layout: EdgeLayout, y: np.ndarray, sigma: float) -> MessageBatch:
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    if y.shape[1] != layout.n_vars:
        raise ValueError(f"y has {y.shape[1]} symbols, layout has {layout.n_vars}")
    return MessageBatch(layout, np.ascontiguousarray(channel_llrs(y, sigma).T))


def _active_dev(active, gp):
    if active is None:
        return None
    import torch
    w = lane_words(np.asarray(active, dtype=bool), gp)
    return torch.from_numpy(w.view(np.int32)).cuda()


def check_node_update(batch: MessageBatch, layout: EdgeLayout, active: np.ndarray | None = None) -> None:
    """Replace every package with its check-to-variable message, in place (bp.py:134-162)."""
    if layout.edge_count == 0:
        return
    act = _active_dev(active, batch._gp)
    batch._before_update()
    _lib.call("qc64_cnu" if batch.fp64 else "qc_cnu", layout.plan().handle, batch._gp,
              batch._msgs.data_ptr(), _lib.ptr(act), _stream())
    batch._after_update()


def variable_node_update(batch: MessageBatch, layout: EdgeLayout,
                         active: np.ndarray | None = None) -> np.ndarray:
    """Packages <- variable-to-check messages on active lanes; returns the
    posteriors clip(mu + sum alpha) of EVERY lane, frozen ones included
    (N, gamma) (bp.py:165-188)."""
    import torch
    act = _active_dev(active, batch._gp)
    post = torch.zeros((layout.n_vars, batch._gp), dtype=batch._msgs.dtype, device=batch._msgs.device)
    batch._before_update()
    _lib.call("qc64_vnu" if batch.fp64 else "qc_vnu", layout.plan().handle, batch._gp,
              batch._msgs.data_ptr(), batch._mu_dev.data_ptr(), post.data_ptr(), None,
              _lib.ptr(act), _stream())
    batch._after_update()
    return post[:, : batch.gamma].double().cpu().numpy()


def hard_decision_and_syndrome(layout: EdgeLayout, posteriors: np.ndarray):
    """bits (N, gamma) uint8 (1 iff LLR < 0) and ok (gamma,) bool (bp.py:191-210)."""
    torch = require_cuda()
    post = np.asarray(posteriors, dtype=np.float64)
    n, g = post.shape
    gp = pad32(g)
    fp64 = get_precision() == "float64"
    if fp64:
        dev = torch.zeros((n, gp), dtype=torch.float64)
        dev[:, :g] = torch.from_numpy(post)
    else:
        p32 = post.astype(np.float32)
        p32[(post < 0) & (p32 == 0)] = -1.0        # keep the sign of tiny negatives
        dev = torch.zeros((n, gp), dtype=torch.float32)
        dev[:, :g] = torch.from_numpy(p32)
    dev = dev.cuda()
    hb = torch.zeros((n, gp // 32), dtype=torch.int32, device=dev.device)
    bad = torch.zeros(gp // 32, dtype=torch.int32, device=dev.device)
    plan = layout.plan()
    _lib.call("qc64_hard_bits" if fp64 else "qc_hard_bits", plan.handle, gp, dev.data_ptr(),
              hb.data_ptr(), _stream())
    if layout.edge_count:
        _lib.call("qc_syndrome", plan.handle, gp, hb.data_ptr(), bad.data_ptr(), _stream())
    bits = unpack_planes(hb.cpu().numpy().view(np.uint32), g)
    badw = bad.cpu().numpy().view(np.uint32)
    ok = ((badw[np.arange(g) >> 5] >> (np.arange(g) & 31).astype(np.uint32)) & 1) == 0
    return bits, ok


class BlockDecoder:
    """Device engine for repeated batched decodes of one code at fixed gamma.

    Buffers (all on the GPU, sized once):
      mu (N, gamma_pad) fp32 variable-major channel LLRs,
      msgs (E, gamma_pad) fp32 edge-major packages,
      post (N, gamma_pad) fp32, hb (N, gamma_pad/32) hard-bit planes,
      ok / iters / lane_bits (gamma_pad,).
    `run()` launches init + `iterations` x (check, variable) + syndrome (+ per-lane
    bit counts); after the first call it is replayed as one CUDA graph.
    """

    def __init__(self, layout: EdgeLayout, gamma: int, iterations: int = 30,
                 early_stop: bool = False, graph: bool = True, count_bits: bool = True,
                 precision: str | None = None, compact: bool = True):
        torch = require_cuda()
        if iterations < 1:
            raise ValueError("need at least one iteration")
        self.layout, self.gamma, self.iterations = layout, gamma, iterations
        self.early_stop = bool(early_stop)
        self.gp = pad32(gamma)
        self.plan = layout.plan()
        self.fp64 = (precision or get_precision()) == "float64"
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        N, E, gp = layout.n_vars, max(layout.edge_count, 1), self.gp
        f32, i32 = (torch.float64 if self.fp64 else torch.float32), torch.int32
        self.mu = torch.full((N, gp), L_MAX, dtype=f32, device=dev)
        self.msgs = torch.zeros((E, gp), dtype=f32, device=dev)
        self.post = torch.zeros((N, gp), dtype=f32, device=dev)
        self.hb = torch.zeros((N, gp // 32), dtype=i32, device=dev)
        self.work = torch.zeros(int(_lib.load().qc_decode_work_words(self.plan.handle, gp)), dtype=i32, device=dev)
        # early stop with lane compaction (es_compact.cu): a second lane set
        nes = int(_lib.load().qc_decode_es_scratch_words(self.plan.handle, gp)) if (
            self.early_stop and not self.fp64 and compact) else 0
        self.es_scratch = torch.zeros(nes, dtype=i32, device=dev) if nes else None
        self.ok = torch.zeros(gp, dtype=torch.uint8, device=dev)
        self.iters = torch.zeros(gp, dtype=i32, device=dev)
        self.lane_bits = torch.zeros(gp, dtype=i32, device=dev) if count_bits else None
        self._use_graph = graph
        self._graph = None
        self._x = None          # lane-major fp64 staging (device)
        self._host = {}         # pinned host buffers
        self._lock = threading.Lock()

    # -- device work ------------------------------------------------------
    def _launch(self):
        if self.fp64:
            _lib.call("qc64_decode", self.plan.handle, self.gp, self.iterations, int(self.early_stop),
                      self.mu.data_ptr(), self.msgs.data_ptr(), self.post.data_ptr(),
                      self.hb.data_ptr(), self.work.data_ptr(), self.ok.data_ptr(),
                      self.iters.data_ptr(), _stream())
            if self.lane_bits is not None:
                _lib.call("qc_bit_errors", self.plan.handle, self.gp, self.hb.data_ptr(),
                          self.lane_bits.data_ptr(), _stream())
            return
        if self.es_scratch is not None:
            _lib.call("qc_decode_es", self.plan.handle, self.gp, self.iterations,
                      self.mu.data_ptr(), self.msgs.data_ptr(), self.post.data_ptr(),
                      self.hb.data_ptr(), self.work.data_ptr(), self.es_scratch.data_ptr(), self.ok.data_ptr(),
                      self.iters.data_ptr(), _lib.ptr(self.lane_bits), _stream())
            return
        _lib.call("qc_decode", self.plan.handle, self.gp, self.iterations, int(self.early_stop),
                  self.mu.data_ptr(), self.msgs.data_ptr(), self.post.data_ptr(),
                  self.hb.data_ptr(), self.work.data_ptr(), self.ok.data_ptr(),
                  self.iters.data_ptr(), _lib.ptr(self.lane_bits), _stream())

    def run(self):
        """Decode the LLRs currently in `self.mu` (on torch's current stream)."""
        if not self._use_graph:
            self._launch()
            return
        import torch
        if self._graph is None:
            self._launch()                       # eager warm-up (also validates arguments)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch()
            self._graph = g
        else:
            self._graph.replay()

    def kernel_launches_per_run(self) -> int:
        """Our kernels in one run() (for bench gpu_launches)."""
        if self.fp64:
            it = self.iterations
            n = (2 + 4 * it + 2) if self.early_stop else (1 + 2 * it + 2)
        elif self.es_scratch is not None:
            n = int(_lib.load().qc_decode_es_launches(self.plan.handle, self.gp, self.iterations))
        else:
            n = int(_lib.load().qc_decode_launches(self.plan.handle, self.gp, self.iterations,
                                                   int(self.early_stop)))
        if self.lane_bits is not None:
            n += 1
        return n

    # -- host <-> device ----------------------------------------------------
    def _pinned(self, key, shape, dtype):
        import torch
        t = self._host.get(key)
        if t is None or tuple(t.shape) != tuple(shape):
            t = torch.empty(shape, dtype=dtype, pin_memory=True)
            self._host[key] = t
        return t

    def load_lane_major(self, x: np.ndarray, sigma: float | None):
        """x (gamma_in, N) fp64: received values (sigma given) or LLRs (sigma None).

        Host side: one multi-threaded copy into a pinned staging buffer, then an
        async H2D; the LLR scale/clip/transpose runs on the GPU."""
        import torch
        x = np.asarray(x, dtype=np.float64)
        gi, n = x.shape
        if n != self.layout.n_vars or gi > self.gp:
            raise ValueError(f"input {x.shape} does not fit (<= {self.gp}, {self.layout.n_vars})")
        h = self._pinned("x", (gi, n), torch.float64)
        h.copy_(torch.from_numpy(np.ascontiguousarray(x)))
        if self._x is None or tuple(self._x.shape) != (gi, n):
            self._x = torch.empty((gi, n), dtype=torch.float64, device=self.device)
        self._x.copy_(h, non_blocking=True)
        if self.fp64:
            _lib.call("qc64_mu_from_lane_major", n, self.gp, gi, self._x.data_ptr(),
                      float(sigma) if sigma is not None else 0.0, 1, self.mu.data_ptr(), _stream())
            return
        _lib.call("qc_llr_from_lane_major", n, self.gp, gi, self._x.data_ptr(),
                  float(sigma) if sigma is not None else 0.0, self.mu.data_ptr(), _stream())

    def stage_result(self, gamma: int):
        """Queue the lane-major conversion and the device->host copies of the
        first `gamma` lanes (posteriors as fp32, the precision they were
        computed in; hard bits; syndrome flags; iteration counts)."""
        import torch
        n = self.layout.n_vars
        pdt = torch.float64 if self.fp64 else torch.float32
        if getattr(self, "_lm", None) is None or self._lm[0].shape[0] != gamma:
            self._lm = (torch.empty((gamma, n), dtype=pdt, device=self.device),
                        torch.empty((gamma, n), dtype=torch.uint8, device=self.device))
        post_d, bits_d = self._lm
        _lib.call("qc64_lane_major" if self.fp64 else "qc_lane_major_f32", n, self.gp, gamma,
                  self.post.data_ptr(), post_d.data_ptr(), bits_d.data_ptr(), _stream())
        hp = self._pinned("post", (gamma, n), pdt)
        hb = self._pinned("bits", (gamma, n), torch.uint8)
        hs = self._pinned("small", (2, self.gp), torch.int32)
        hp.copy_(post_d, non_blocking=True)
        hb.copy_(bits_d, non_blocking=True)
        hs[0].copy_(self.ok.to(torch.int32), non_blocking=True)
        hs[1].copy_(self.iters, non_blocking=True)
        self._done = torch.cuda.Event()
        self._done.record()

    def collect_result(self, gamma: int, post, bits, ok, its, at: int = 0):
        """Wait for stage_result and write lanes into host arrays at row `at`
        (multi-threaded copies; fp32 posteriors widen to float64)."""
        import torch
        self._done.synchronize()
        torch.from_numpy(post[at:at + gamma]).copy_(self._host["post"])
        torch.from_numpy(bits[at:at + gamma]).copy_(self._host["bits"])
        small = self._host["small"].numpy()
        ok[at:at + gamma] = small[0, :gamma].astype(bool)
        its[at:at + gamma] = small[1, :gamma]

    def result(self, gamma: int) -> DecodeResult:
        n = self.layout.n_vars
        post = np.empty((gamma, n), dtype=np.float64)
        bits = np.empty((gamma, n), dtype=np.uint8)
        ok = np.empty(gamma, dtype=bool)
        its = np.empty(gamma, dtype=np.int64)
        self.stage_result(gamma)
        self.collect_result(gamma, post, bits, ok, its)
        return DecodeResult(hard_bits=bits, posteriors=post, syndrome_ok=ok, iterations_run=its)


HOST_CHUNK = 512        # largest pipelined chunk of the host-buffer API (plan C/4, C/2, C.., C/2, C/4; tools/e2e_bench.py)
HOST_CHUNK_ES = 1024    # chunk of early-stop batches from 2048 lanes (lane compaction needs >= 1024)
HOST_SLOTS = 4          # CUDA streams (device buffer sets) the chunks rotate over, pageable input
HOST_SLOTS_PINNED = 3   # same for page-locked input (no host staging copy to hide; tools/e2e_bench.py)
PINNED_MIN_BYTES = 1 << 20
# pageable inputs up to this size are staged page-locked in one copy (1.1-1.7x
# at 32-1024 lanes of n18360; above it the pipeline's fp32 staging threads win)
STAGE_PAGEABLE_MAX_BYTES = 160 << 20


class HostDecoder:
    """Native host-buffer pipeline (qc_host_* in include/qcldpc_b200.h): chunks of
    `chunk` lanes rotate over `slots` streams, so the copy-in of chunk k+1 and
    the copy-out of chunk k-1 overlap the graph-replayed decode of chunk k."""

    def __init__(self, layout: EdgeLayout, chunk: int, slots: int, iterations: int, early_stop: bool):
        import ctypes
        require_cuda()
        self.layout = layout
        self.plan = layout.plan()          # must outlive the native decoder
        h = ctypes.c_void_p()
        _lib.call("qc_host_create", self.plan.handle, chunk, slots, iterations, int(early_stop),
                  ctypes.byref(h))
        self.handle = h.value
        self.chunk, self.slots = chunk, slots
        self._lock = threading.Lock()      # the native decoder serves one call at a time

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h and _lib._LIB is not None:
            _lib.load().qc_host_destroy(h)

    def decode(self, x: np.ndarray, sigma: float) -> DecodeResult:
        """x (gamma, N) fp64: received values (sigma > 0) or LLRs (sigma = 0)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        G, n = x.shape
        post = host_empty((G, n), np.float64)
        bits = host_empty((G, n), np.uint8)
        ok = np.empty(G, dtype=bool)
        its = np.empty(G, dtype=np.int64)
        with self._lock:
            _lib.call("qc_host_decode", self.handle, x.ctypes.data, G, float(sigma), bits.ctypes.data,
                      post.ctypes.data, ok.ctypes.data, its.ctypes.data)
        return DecodeResult(hard_bits=bits, posteriors=post, syndrome_ok=ok, iterations_run=its)


_PINNED_OUTPUTS = [os.environ.get("QCLDPC_B200_PINNED_OUTPUTS", "1") != "0"]


def set_pinned_outputs(on: bool) -> None:
    """Whether decode_batch / decode_llr_batch return large results in page-locked
    memory (default on: the device DMAs straight into them, ~10% faster e2e).
    Page-locked blocks come from torch's caching host allocator: a dropped
    result's block is reused by the next call but stays pinned for the life
    of the process; release_pinned_cache() returns the unused ones to the OS."""
    _PINNED_OUTPUTS[0] = bool(on)


def release_pinned_cache() -> None:
    """Free the cached page-locked blocks no live result array uses."""
    import torch
    torch._C._host_emptyCache()


def host_empty(shape, dtype, min_bytes: int | None = None) -> np.ndarray:
    """Output array for the host-buffer API: large ones come from torch's caching
    page-locked allocator (unless set_pinned_outputs(False)), so the decoder
    DMAs straight into them and a freed result's pages are reused by the next
    call (no fresh page faults)."""
    dtype = np.dtype(dtype)
    floor = PINNED_MIN_BYTES if min_bytes is None else min_bytes
    if not _PINNED_OUTPUTS[0] or int(np.prod(shape)) * dtype.itemsize < floor:
        return np.empty(shape, dtype=dtype)
    import torch
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8,
           np.dtype(np.float32): torch.float32}[dtype]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


def host_array(a: np.ndarray) -> np.ndarray:
    """Copy of `a` in page-locked host memory (inputs the decoder DMAs in place)."""
    out = host_empty(a.shape, a.dtype)
    np.copyto(out, a)
    return out


def _host_decoder(layout: EdgeLayout, gamma: int, iterations: int, early_stop: bool,
                  pinned_input: bool = False) -> HostDecoder:
    import torch
    # small batches: one chunk up to 64 lanes; above that at least two chunks,
    # so the copy-in of one overlaps the decode of another: 64-lane chunks up to
    # 128 lanes, 128-lane chunks below 256 (96 / 128 / 160 / 192 lanes: 15-25%
    # faster than one chunk since the small-batch passes got cheaper,
    # profiles/r02/e2e_chunk_sweep.jsonl); from 256 lanes about two chunks
    # (e.g. 512 lanes: 64 + 128 + 256 + 64 over chunk 256)
    if gamma <= 32:
        chunk = pad32(gamma)
    elif gamma <= 64:
        chunk = 64
    elif gamma <= 128:
        chunk = 64
    elif gamma < 256:
        chunk = 128
    else:
        chunk = min(HOST_CHUNK, max(128, ((gamma + 1) // 2 + 63) // 64 * 64))
    if early_stop and gamma >= 2 * HOST_CHUNK_ES:
        # early stop: chunks large enough for lane compaction (es_compact.cu,
        # from 1024 lanes) -- profiles/r02/es_compaction.md
        chunk = HOST_CHUNK_ES
    slots = (HOST_SLOTS_PINNED if pinned_input else HOST_SLOTS) if gamma > chunk else 1
    cache = layout.__dict__.setdefault("_host_decoders", {})
    key = (chunk, slots, iterations, bool(early_stop), torch.cuda.current_device())
    dec = cache.get(key)
    if dec is None:
        if len(cache) >= 12:
            cache.clear()
        dec = HostDecoder(layout, chunk, slots, iterations, early_stop)
        cache[key] = dec
    return dec


def _decoder(layout: EdgeLayout, gamma: int, iterations: int, early_stop: bool) -> BlockDecoder:
    """float64 conformance build: device engine at the batch's own gamma."""
    cache = layout.__dict__.setdefault("_decoders", {})
    import torch
    key = (pad32(gamma), iterations, bool(early_stop), get_precision(), torch.cuda.current_device())
    dec = cache.get(key)
    if dec is None:
        if len(cache) >= 8:
            cache.clear()
        dec = BlockDecoder(layout, pad32(gamma), iterations, early_stop, count_bits=False)
        cache[key] = dec
    return dec


def _decode_host(layout: EdgeLayout, x: np.ndarray, sigma: float | None, iterations: int,
                 early_stop: bool) -> DecodeResult:
    require_cuda()
    if get_precision() == "float64":
        dec = _decoder(layout, x.shape[0], iterations, early_stop)
        with dec._lock:                    # one call at a time per cached decoder (shared buffers)
            dec.load_lane_major(x, sigma)
            dec.run()
            return dec.result(x.shape[0])
    x = np.ascontiguousarray(x, dtype=np.float64)
    pinned = bool(x.size) and _lib.load().qc_host_is_pinned(x.ctypes.data, x.nbytes) == 1
    if not pinned and 0 < x.nbytes <= STAGE_PAGEABLE_MAX_BYTES:
        # ordinary numpy input of a small batch: one multi-threaded copy into
        # page-locked memory (torch's intra-op pool, no thread start-up) and the
        # page-locked path, instead of the pipeline's per-call staging threads
        # (profiles/r02/e2e_pageable_small.jsonl)
        import torch
        staged = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
        staged.copy_(torch.from_numpy(x))
        x, pinned = staged.numpy(), True
    return _host_decoder(layout, x.shape[0], iterations, early_stop, pinned).decode(x, sigma or 0.0)


def decode_llr_batch(layout: EdgeLayout, mu: np.ndarray, iterations: int,
                     early_stop: bool = False) -> DecodeResult:
    """Decode channel LLRs mu (gamma, N) (saturated internally) -- bp.py:213-265."""
    if iterations < 1:
        raise ValueError("need at least one iteration")
    mu = np.atleast_2d(np.asarray(mu, dtype=np.float64))
    if mu.shape[1] != layout.n_vars:
        raise ValueError(f"mu has {mu.shape[1]} symbols, layout has {layout.n_vars}")
    return _decode_host(layout, mu, None, iterations, early_stop)


def decode_batch(layout: EdgeLayout, y: np.ndarray, sigma: float, iterations: int,
                 early_stop: bool = False) -> DecodeResult:
    """Decode received values y (gamma, N) over AWGN with noise sigma -- bp.py:268-274."""
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    if y.shape[1] != layout.n_vars:
        raise ValueError(f"y has {y.shape[1]} symbols, layout has {layout.n_vars}")
    if iterations < 1:
        raise ValueError("need at least one iteration")
    s = abs(float(sigma))
    s = s if s > 0.0 else 1e-300
    return _decode_host(layout, y, s, iterations, early_stop)
