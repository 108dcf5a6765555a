"""LDPC convolutional codes unwrapped from QC-LDPC block codes, decoded on B200.

Drop-in for /root/reference/pkg/src/qcldpc/convolutional.py.  `LdpcccCode`
carries the same host attributes (lam, ms, c, cb, label_grid, lut_c, lut_v,
lut_sub, sub_offset, edge_count, period, rate_bound; convolutional.py:67-151);
`StreamDecoder` keeps its state on the GPU -- I processor groups of message
packages and the I*(m_s+1)-frame channel ring (circular window in HBM) -- and
advances one slot per `push_frame` with three sm_100a kernels (csrc/stream.cu).
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import _lib
from .codes import ExponentMatrix
from .plan import StreamPlan, pad32, require_cuda

__all__ = ["LdpcccCode", "DecodedFrame", "unwrap_qc", "StreamDecoder"]


class LdpcccCode:
    """Unwrapped (convolutional) form of a QC-LDPC block code."""

    def __init__(self, exp: ExponentMatrix):
        J, L = exp.block_rows, exp.block_cols
        lam = math.gcd(J, L)
        if lam < 2:
            raise ValueError(
                f"gcd(J, L) = {lam}: the shift grid cannot be partitioned into a square "
                "sub-block grid, so there is nothing to unwrap")
        self.exp = exp
        self.lam = lam
        self.ms = lam - 1
        self.p = exp.p
        self.sub_j = J // lam
        self.sub_l = L // lam
        self.c = self.sub_l * exp.p
        self.cb = self.sub_j * exp.p
        self.label_grid = np.arange(lam * lam, dtype=np.int64).reshape(lam, lam)
        k = np.arange(lam)
        # layer phase kappa couples frames kappa-ms..kappa; frame phase phi couples layers phi..phi+ms
        self.lut_c = self.label_grid[k[:, None], (k[:, None] + 1 + k[None, :]) % lam]
        self.lut_v = self.label_grid[(k[:, None] + k[None, :]) % lam, k[:, None]]
        sj, sl = self.sub_j, self.sub_l
        self.lut_sub = [exp.shifts[(b // lam) * sj:(b // lam + 1) * sj, (b % lam) * sl:(b % lam + 1) * sl]
                        for b in range(lam * lam)]
        self.sub_edge_count = np.array([int((g >= 0).sum()) * self.p for g in self.lut_sub],
                                       dtype=np.int64)
        self.sub_offset = np.concatenate([[0], np.cumsum(self.sub_edge_count)[:-1]]).astype(np.int64)
        self.edge_count = int(self.sub_edge_count.sum())
        self._plans = {}

    @property
    def period(self) -> int:
        return self.lam

    @property
    def rate_bound(self) -> float:
        return (self.c - self.cb) / self.c

    def plan(self) -> StreamPlan:
        """Device plan of the current CUDA device (created on first use, immutable)."""
        import torch
        dev = torch.cuda.current_device()
        if dev not in self._plans:
            pl = StreamPlan(self.exp)
            if pl.E != self.edge_count or pl.c != self.c or pl.lam != self.lam:
                raise RuntimeError("device LDPCCC plan does not match the host tables")
            self._plans[dev] = pl
        return self._plans[dev]


def unwrap_qc(exp: ExponentMatrix) -> LdpcccCode:
    """Unwrapped convolutional code of a QC grid; ValueError when gcd(J, L) < 2."""
    return LdpcccCode(exp)


@dataclasses.dataclass
class DecodedFrame:
    """Emitted frame: lane-major hard bits / posteriors; tail=True for flushed frames."""

    frame_index: int
    hard_bits: np.ndarray
    posteriors: np.ndarray
    tail: bool = False


class StreamDecoder:
    """Pipelined window decoder with I processors over gamma lanes (GPU-resident).

    Frame t pushed at slot t is emitted at slot t + I*(m_s+1) - 1 after I
    iterations; the first emission happens at slot I*(m_s+1) - 1.

    Emitted frames' arrays live in page-locked host memory (the copy-out is
    asynchronous); a caller that keeps very many frames alive can switch to
    ordinary arrays with `set_pinned_outputs(False)` (each push then waits for
    its copy-out) and return cached page-locked blocks with
    `release_pinned_cache()`.
    """

    def __init__(self, code: LdpcccCode, processors: int, gamma: int = 1):
        if processors < 1:
            raise ValueError("need at least one processor")
        if gamma < 1:
            raise ValueError("gamma must be positive")
        torch = require_cuda()
        self.code = code
        self.processors = processors
        self.gamma = gamma
        self.period = code.ms + 1
        self.window = processors * self.period
        self.t = 0
        self._flushed = False
        self._gp = pad32(gamma)
        self._plan = code.plan()
        dev = torch.device("cuda", torch.cuda.current_device())
        self._msg = torch.zeros((processors * code.edge_count, self._gp), dtype=torch.float32, device=dev)
        self._ring = torch.zeros((self.window, code.c, self._gp), dtype=torch.float32, device=dev)
        self._mu = torch.empty((code.c, self._gp), dtype=torch.float32, device=dev)
        self._post = torch.zeros((code.c, self._gp), dtype=torch.float32, device=dev)
        self._y = torch.empty((gamma, code.c), dtype=torch.float64, device=dev)
        self._y_host = None      # page-locked staging of pushed frames
        self._lm = None          # lane-major device outputs of emitted frames
        self._es = None          # side stream of the emitting processor (I >= 2)
        self._ev_rest = None     # end of the last slot's main-stream work
        self._kind = np.zeros((processors, code.lam * code.lam), dtype=np.int8)
        self._ring_live = np.zeros(self.window, dtype=bool)
        self._tracked = 0          # slots folded into _kind / _ring_live (brought up to date on access)

    # What each (processor group, sub-block label) block of the message store
    # holds in the REFERENCE's terms after the slots run so far (host-side
    # bookkeeping of convolutional.py:256-334, O(I*T) per slot): the device
    # keeps var->check messages in phi form and skips the emission-time clear
    # (convolutional.py:328-330), so message_memory / channel_memory translate.
    _ZERO, _BETA, _ALPHA = 0, 1, 2

    def _sync_track(self):
        """Bring the block-kind / ring-liveness tables up to slot self.t -- done
        when message_memory / channel_memory are read, not on every push (the
        per-slot bookkeeping is ~I*T table writes of host Python)."""
        for t in range(self._tracked, self.t):
            self._track(t)
        self._tracked = self.t

    def _track(self, t):
        code, T, I, kind = self.code, self.period, self.processors, self._kind
        ph = t % T
        for d in range(T):
            kind[(t // T) % I, code.lut_v[ph, d]] = self._BETA
        self._ring_live[t % self.window] = True
        for i in range(1, I + 1):
            s = t - (i - 1) * T
            if s < 0:
                break
            for d in range(T):
                f = s - code.ms + d
                if f >= 0:
                    kind[(f // T) % I, code.lut_c[ph, d]] = self._ALPHA
        for i in range(1, I + 1):
            j = t - i * T + 1
            if j < 0:
                break
            for d in range(T):
                kind[(j // T) % I, code.lut_v[j % T, d]] = self._BETA if i < I else self._ZERO
            if i == I:
                self._ring_live[j % self.window] = False

    @property
    def channel_memory(self) -> np.ndarray:
        """Channel LLR ring, (I*(m_s+1), c, gamma) float64 host copy; slots of
        emitted frames read 0.0 as in the reference (convolutional.py:331)."""
        import torch
        torch.cuda.synchronize()
        self._sync_track()
        ring = self._ring[:, :, : self.gamma].double().cpu().numpy()
        ring[~self._ring_live] = 0.0
        return ring

    @property
    def message_memory(self) -> np.ndarray:
        """Edge message packages, (I, base edge count, gamma) float64 host copy,
        in the reference's representation (convolutional.py:200-218): alpha on
        check->variable blocks, beta on variable->check blocks (converted from
        the device's phi form, beta = sign * phi(|psi| ln 2), within fp32
        rounding), 0.0 on never-written / emitted blocks."""
        import torch
        torch.cuda.synchronize()
        self._sync_track()
        code = self.code
        m = self._msg[:, : self.gamma].double().cpu().numpy()
        m = m.reshape(self.processors, code.edge_count, self.gamma)
        for g in range(self.processors):
            for lbl in range(code.lam * code.lam):
                sl = slice(int(code.sub_offset[lbl]), int(code.sub_offset[lbl] + code.sub_edge_count[lbl]))
                k = self._kind[g, lbl]
                if k == self._ZERO:
                    m[g, sl] = 0.0
                elif k == self._BETA:
                    psi = m[g, sl]
                    x = np.abs(psi) * math.log(2.0)
                    with np.errstate(divide="ignore", over="ignore"):
                        mag = -np.log(np.tanh(0.5 * x))          # phi is its own inverse
                    m[g, sl] = np.copysign(np.minimum(mag, 50.0), psi)
        return m

    def push_frame(self, y_frame: np.ndarray, sigma: float) -> DecodedFrame | None:
        """Feed one received frame (gamma, c); return the emitted frame or None.

        The frame emitted at slot t (t - I*T + 1) does not depend on frame t for
        I >= 2: the emitting processor's check and variable updates touch edges
        and ring slots disjoint from the entry of frame t and from the other
        processors' work (cc_slot_part).  So it runs first, on a side stream,
        and its copy-out overlaps the host staging of frame t, its copy-in and
        the other I - 1 processors, which keep running after this returns."""
        if self._flushed:
            raise RuntimeError("decoder already flushed; create a new one")
        y = np.atleast_2d(np.asarray(y_frame, dtype=np.float64))
        if y.shape != (self.gamma, self.code.c):
            raise ValueError(f"expected frame shape {(self.gamma, self.code.c)}, got {y.shape}")
        import torch
        em = self._emit_begin()
        # page-locked staging (torch's multi-threaded host copy), then one call:
        # asynchronous H2D + LLR conversion on the current stream
        if self._y_host is None:
            self._y_host = torch.empty((self.gamma, self.code.c), dtype=torch.float64, pin_memory=True)
            self._y_ev = torch.cuda.Event()
        else:
            self._y_ev.synchronize()     # the previous frame's copy has left the staging buffer
        self._y_host.copy_(torch.from_numpy(np.ascontiguousarray(y)))
        s = abs(float(sigma))
        st = _lib.stream_handle()
        _lib.call("qc_llr_from_host", self.code.c, self._gp, self.gamma, self._y_host.data_ptr(), self._y.data_ptr(),
                  s if s > 0.0 else 1e-300, self._mu.data_ptr(), st)
        self._y_ev.record()
        self._rest(self._mu, em is not None, st)
        return self._emit_end(em, tail=False)

    def push_llr_device(self, mu_dev) -> DecodedFrame | None:
        """B200 extension: push a frame of LLRs already on the device, (c, gamma_pad) fp32."""
        if self._flushed:
            raise RuntimeError("decoder already flushed; create a new one")
        import torch
        if (not isinstance(mu_dev, torch.Tensor) or mu_dev.dtype != torch.float32 or not mu_dev.is_cuda
                or mu_dev.device != self._msg.device or tuple(mu_dev.shape) != (self.code.c, self._gp)
                or not mu_dev.is_contiguous()):
            raise ValueError(f"mu_dev must be a contiguous float32 tensor of shape {(self.code.c, self._gp)} "
                             f"on {self._msg.device}")
        return self._advance(mu_dev, tail=False)

    def flush(self) -> list:
        """Push zero-LLR virtual frames until every real frame has left; frames flagged tail."""
        if self._flushed:
            raise RuntimeError("decoder already flushed")
        out = []
        for _ in range(self.window - 1):
            fr = self._advance(None, tail=True)
            if fr is not None:
                out.append(fr)
        self._flushed = True
        return out

    def _advance(self, mu_dev, tail: bool) -> DecodedFrame | None:
        em = self._emit_begin()
        self._rest(mu_dev, em is not None)
        return self._emit_end(em, tail)

    def _emit_begin(self):
        """Queue slot t's emitting processor (0-based I-1) on the side stream, then
        the lane-major conversion and the copy-out of the emitted frame."""
        t = self.t
        j = t - self.window + 1
        if j < 0 or self.processors < 2:
            return None
        import torch
        from .bp import host_empty
        if self._es is None:
            self._es = torch.cuda.Stream()
            self._es_ev = torch.cuda.Event()
            self._lm = (torch.empty((self.gamma, self.code.c), dtype=torch.float64, device=self._post.device),
                        torch.empty((self.gamma, self.code.c), dtype=torch.uint8, device=self._post.device))
        es = self._es
        if self._ev_rest is not None:
            es.wait_event(self._ev_rest)          # slot t-1 complete
        else:
            es.wait_stream(torch.cuda.current_stream())
        c, I = self.code.c, self.processors
        _lib.call("cc_slot_part", self._plan.handle, I, self._gp, t, None, self._msg.data_ptr(),
                  self._ring.data_ptr(), None, self._post.data_ptr(), None, I - 1, 1, 6, es.cuda_stream)
        # page-locked outputs whatever their size: a copy into pageable memory
        # would block this call until the emitting chain finished
        post = host_empty((self.gamma, c), np.float64, min_bytes=0)
        bits = host_empty((self.gamma, c), np.uint8, min_bytes=0)
        post_d, bits_d = self._lm
        _lib.call("qc_lane_major_to_host", c, self._gp, self.gamma, self._post.data_ptr(), post_d.data_ptr(),
                  bits_d.data_ptr(), post.ctypes.data, bits.ctypes.data, es.cuda_stream)
        ev = self._es_ev                          # recorded and waited for within this push
        ev.record(es)
        return j, post, bits, ev

    def _rest(self, mu_dev, split: bool, stream=None):
        """Queue the rest of slot t on the main stream: the entry of frame t and
        processors 0..I-2 (the whole slot when nothing was split off)."""
        import torch
        t = self.t
        I = self.processors
        j = t - self.window + 1
        post = self._post.data_ptr() if (j >= 0 and not split) else None
        _lib.call("cc_slot_part", self._plan.handle, I, self._gp, t, None, self._msg.data_ptr(),
                  self._ring.data_ptr(), _lib.ptr(mu_dev), post, None, 0, I - 1 if split else I, 7,
                  stream if stream is not None else _lib.stream_handle())
        if self._ev_rest is None:
            self._ev_rest = torch.cuda.Event()
        self._ev_rest.record()
        self.t = t + 1

    def _emit_end(self, em, tail: bool) -> DecodedFrame | None:
        j = self.t - self.window                  # the frame slot t (= self.t - 1) emits
        if em is None:
            if j < 0:
                return None
            return self._emit_sync(j, tail)       # I = 1: emitted by the whole slot on the main stream
        jj, post, bits, ev = em
        ev.synchronize()
        return DecodedFrame(frame_index=jj, hard_bits=bits, posteriors=post, tail=tail)

    def _emit_sync(self, j: int, tail: bool) -> DecodedFrame:
        import torch
        from .bp import host_empty
        c = self.code.c
        if self._lm is None:
            self._lm = (torch.empty((self.gamma, c), dtype=torch.float64, device=self._post.device),
                        torch.empty((self.gamma, c), dtype=torch.uint8, device=self._post.device))
        post_d, bits_d = self._lm
        post = host_empty((self.gamma, c), np.float64, min_bytes=0)
        bits = host_empty((self.gamma, c), np.uint8, min_bytes=0)
        _lib.call("qc_lane_major_to_host", c, self._gp, self.gamma, self._post.data_ptr(), post_d.data_ptr(),
                  bits_d.data_ptr(), post.ctypes.data, bits.ctypes.data, _lib.stream_handle())
        torch.cuda.current_stream().synchronize()
        return DecodedFrame(frame_index=j, hard_bits=bits, posteriors=post, tail=tail)
