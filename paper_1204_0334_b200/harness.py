"""Monte-Carlo BER/FER campaigns and throughput benchmarks on B200 GPUs.

Drop-in for /root/reference/pkg/src/qcldpc/harness.py (same config, result
rows, CSV/JSONL formats, stop rule and lane addressing), with the work moved
to the device:

* block mode (harness.py:140-204): one launch decodes B reference batches of
  gamma lanes at once (gamma_kernel = B * gamma).  Channel (Philox + inverse
  CDF) -> fused init -> 30 flooding iterations -> per-lane bit counts -> per-
  batch (frames, bit_errors, frame_errors) all run inside one CUDA graph; the
  host only reads the counter array.  Batch b of point pi draws lanes
  (pi << 32) + b*gamma + g exactly as the reference, so counts are identical.
* stream mode (harness.py:212-286): S independent segments decoded side by
  side (gamma_kernel = S * gamma lanes), every push slot (channel + entry +
  I check layers + I frames + counting) captured once as a graph.
* multi-GPU: with a torch.distributed group, round k gives rank r the batches
  [k*W*B + r*B, k*W*B + (r+1)*B); one all_reduce(SUM) of the int64 per-batch
  counter array per round; every rank then applies the ordered stop rule.
  `workers` is accepted for compatibility and ignored (GPUs replace processes).
"""

from __future__ import annotations

import dataclasses
import json
import math
import multiprocessing
import time

import numpy as np

from . import _lib
from .bp import BlockDecoder
from .channel import ebn0_to_sigma, seed_words
from .codes import EdgeLayout
from .convolutional import LdpcccCode
from .dist import ordered_prefix, sum_counts, world
from .plan import pad32, require_cuda

__all__ = [
    "SimulationConfig", "PointResult", "CSV_COLUMNS", "run_block_simulation",
    "run_stream_simulation", "bench_throughput", "write_csv", "write_jsonl",
    "BlockCampaign", "StreamCampaign", "RecycleCampaign",
]

CSV_COLUMNS = [
    "code_id", "mode", "ebn0_db", "iters_or_I", "gamma", "frames",
    "bit_errors", "frame_errors", "ber", "fer", "seconds", "frames_per_sec",
    "info_bits_per_sec",
]
TIMING_COLUMNS = ("seconds", "frames_per_sec", "info_bits_per_sec")


@dataclasses.dataclass
class SimulationConfig:
    """Campaign settings shared by block and stream simulations (harness.py:49-73)."""

    code_id: str
    ebn0_db: object
    iterations: int = 30
    processors: int = 20
    gamma: int = 32
    stop_block_errors: int = 100
    max_frames: int = 1_000_000
    seed: int = 0
    workers: int = 1
    early_stop: bool = False
    stream_segment_frames: int | None = None

    def points(self) -> list:
        e = self.ebn0_db
        return [float(x) for x in (e if isinstance(e, (list, tuple, np.ndarray)) else [e])]


@dataclasses.dataclass
class PointResult:
    """One CSV row of a campaign."""

    code_id: str
    mode: str
    ebn0_db: float
    iters_or_i: int
    gamma: int
    frames: int
    bit_errors: int
    frame_errors: int
    ber: float
    fer: float
    seconds: float
    frames_per_sec: float
    info_bits_per_sec: float

    def row(self) -> list:
        return [
            self.code_id, self.mode, f"{self.ebn0_db:g}", self.iters_or_i,
            self.gamma, self.frames, self.bit_errors, self.frame_errors,
            f"{self.ber:.8g}", f"{self.fer:.8g}", f"{self.seconds:.3f}",
            f"{self.frames_per_sec:.3f}", f"{self.info_bits_per_sec:.3f}",
        ]


def write_csv(results, out) -> None:
    import csv

    def emit(fh):
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for r in results:
            w.writerow(r.row())

    if hasattr(out, "write"):
        emit(out)
    else:
        with open(out, "w", newline="") as fh:
            emit(fh)


def write_jsonl(records, out) -> None:
    def emit(fh):
        for r in records:
            fh.write(json.dumps(r, sort_keys=True) + "\n")

    if hasattr(out, "write"):
        emit(out)
    else:
        with open(out, "w") as fh:
            emit(fh)


def _kernel_units(gref: int, target_lanes: int, max_units: int) -> int:
    """Reference batches per launch: a multiple of 32/gcd(gref, 32), ~target_lanes lanes."""
    step = 32 // math.gcd(gref, 32)
    want = max(1, min(max_units, -(-target_lanes // gref)))
    return max(step, -(-want // step) * step)


def _round_buffers(units: int, W: int):
    """Page-locked counter buffers for _run_rounds (a ring of 3: at most two
    rounds are in flight), allocated before a point's clock starts -- a
    first-time page-locked allocation inside it costs about a millisecond."""
    import torch
    return [torch.empty((W * units, 3), dtype=torch.int64, pin_memory=True) for _ in range(3)]


def _run_rounds(step, counts_of, units: int, frames_per_unit: int, rank: int, W: int, group,
                stop: int, max_frames: int, host_bufs=None):
    """Drive rounds of a campaign engine until the reference's ordered stop rule
    holds (harness.py:173-192); returns (frames, bit_errors, frame_errors).

    Round k: `step(k)` decodes this rank's `units` reference batches, their
    counters land in rank's slice of a (W * units, 3) array, one all_reduce(SUM)
    merges the ranks (NCCL on GPUs), and the array is copied to page-locked
    memory behind an event -- all stream-ordered, nothing blocks the host.
    Round k + 1 is queued BEFORE round k's counters are read, so the device
    never idles while the host applies the stop rule.  The look-ahead round is
    only queued while the frame budget is not already exhausted by the rounds in
    flight; when a frame-error stop lands, its (uncounted) work is discarded --
    the counts are those of the ordered prefix, as with the reference's pool.
    """
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    per_round = W * units * frames_per_unit
    bufs = host_bufs or _round_buffers(units, W)

    def launch(rnd):
        step(rnd)
        allc = torch.zeros((W * units, 3), dtype=torch.int64, device=dev)
        allc[rank * units:(rank + 1) * units] = counts_of()
        sum_counts(allc, group)
        host = bufs[rnd % 3]
        host.copy_(allc, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return host, ev

    tot, rnd = (0, 0, 0), 0
    cur = launch(0)
    while True:
        # rounds 0..rnd are queued; speculate on rnd + 1 unless the budget ends earlier
        nxt = launch(rnd + 1) if (rnd + 1) * per_round < max_frames else None
        host, ev = cur
        ev.synchronize()
        tot, done, _ = ordered_prefix(host.numpy(), stop, max_frames, tot)
        if done:
            return tot
        rnd += 1
        cur = nxt if nxt is not None else launch(rnd)


class BlockCampaign:
    """Device-resident block campaign engine for one code / gamma_kernel / iteration count."""

    def __init__(self, layout: EdgeLayout, gamma_ref: int, units: int, iterations: int,
                 early_stop: bool, seed: int, graph: bool = True):
        torch = require_cuda()
        self.layout, self.gref, self.units = layout, gamma_ref, units
        self.gk = gamma_ref * units             # counted lanes; the kernels run pad32(gk)
        self.k0, self.k1 = seed_words(seed)
        # campaigns run the fp32 production kernels (the channel writes fp32 LLRs)
        self.dec = BlockDecoder(layout, self.gk, iterations, early_stop, graph=False, count_bits=True,
                                precision="float32")
        dev = self.dec.device
        self.lane0 = torch.zeros(1, dtype=torch.int64, device=dev)
        self.counts = torch.zeros((units, 3), dtype=torch.int64, device=dev)
        self.sigma = None
        self._graph = None
        self._use_graph = graph

    def _launch(self):
        n = self.layout.n_vars
        self.counts.zero_()
        _lib.call("qc_channel_dev", self.k0, self.k1, self.lane0.data_ptr(), 0, n, self.dec.gp,
                  float(self.sigma), self.dec.mu.data_ptr(), _lib.stream_handle())
        self.dec._launch()
        _lib.call("qc_batch_counts", self.gk, self.gref, self.dec.lane_bits.data_ptr(),
                  self.counts.data_ptr(), _lib.stream_handle())

    def kernel_launches_per_step(self) -> int:
        return 1 + self.dec.kernel_launches_per_run() + 1

    def step(self, lane0: int, sigma: float):
        """Decode lanes lane0 .. lane0 + gamma_kernel - 1; counts -> self.counts (device).
        (When gamma_kernel is not a multiple of 32 the padding lanes decode the
        next lane ids too, but only the first gamma_kernel lanes are counted.)"""
        import torch
        self.lane0.fill_(int(lane0))
        if self.sigma != sigma:
            self.sigma, self._graph = sigma, None
        if not self._use_graph:
            self._launch()
            return
        if self._graph is None:
            self._launch()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch()
            self._graph = g
            return
        self._graph.replay()


class RecycleCampaign:
    """Lane-recycling early-stop engine (csrc/recycle.cu) for regular (J, 24) QC codes.

    gamma_kernel lanes ("slots") decode codewords continuously: a slot whose
    codeword froze (syndrome clean) or reached the iteration cap takes the next
    codeword id at once, so the GPU always works on dense lanes.  Codeword k of
    rank r is lane lane_base + b*gref + k % gref of reference batch
    b = (k // gref) * W + r; per-batch counters are exactly the reference's
    early-stop counts (harness.py:144-154 with early_stop=True).
    """

    TICKS = 16

    def __init__(self, layout: EdgeLayout, gamma_ref: int, gamma_kernel: int, iterations: int, seed: int,
                 rank: int, world_size: int):
        torch = require_cuda()
        self.layout, self.gref, self.gk, self.iters = layout, gamma_ref, gamma_kernel, iterations
        self.rank, self.W = rank, world_size
        self.k0, self.k1 = seed_words(seed)
        self.plan = layout.plan()
        dev = torch.device("cuda", torch.cuda.current_device())
        N, E = layout.n_vars, layout.edge_count
        self.mu = torch.zeros((N, self.gk), dtype=torch.float32, device=dev)
        self.msgs = torch.zeros((E, self.gk), dtype=torch.float32, device=dev)
        self.hb = torch.zeros((N, self.gk // 32), dtype=torch.int32, device=dev)
        nbytes = int(_lib.load().qc_rc_state_bytes(self.gk))
        self.state = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        self._graph = None

    @staticmethod
    def supports(layout: EdgeLayout) -> bool:
        """All-live QC grids (kernels address edges by shift arithmetic)."""
        return layout.qc is not None and bool((layout.qc.shifts >= 0).all())

    def _ticks(self, sigma, lane_base, id_limit, n_batches, counts):
        _lib.call("qc_rc_ticks", self.plan.handle, self.gk, self.gref, self.W, self.rank, self.iters,
                  int(id_limit), int(n_batches), self.k0, self.k1, int(lane_base), float(sigma), self.TICKS,
                  self.mu.data_ptr(), self.msgs.data_ptr(), self.hb.data_ptr(), self.state.data_ptr(),
                  counts.data_ptr(), _lib.stream_handle())

    def run_point(self, sigma: float, lane_base: int, stop: int, max_frames: int, group=None):
        """Decode until the ordered stop rule is met; returns (frames, bit_errors, frame_errors)."""
        import torch
        W, gref = self.W, self.gref
        n_batches = -(-max_frames // gref)                 # global batch rows
        local_batches = -(-n_batches // W) if n_batches > self.rank else 0
        id_limit = max(0, min(local_batches, -(-(n_batches - self.rank) // W))) * gref
        counts = torch.zeros((n_batches + W, 3), dtype=torch.int64, device=self.mu.device)
        _lib.call("qc_rc_init", self.gk, int(id_limit), self.state.data_ptr(), _lib.stream_handle())
        self._graph = None
        # only a window of batches after the consumed prefix can be in flight: a
        # graph of TICKS ticks completes at most TICKS lane generations (a codeword
        # takes >= 1 tick) and the read window lags one round behind the consumed
        # prefix (the look-ahead round is queued before the current one is read)
        win = 2 * self.TICKS * (self.gk // gref + 1) * W + 64

        def launch(lo):
            """Queue one graph of ticks, then the reduced rows [lo, lo + win) to
            page-locked memory behind an event (stream-ordered, host not blocked)."""
            if self._graph is None:
                self._ticks(sigma, lane_base, id_limit, n_batches, counts)      # eager first round
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._ticks(sigma, lane_base, id_limit, n_batches, counts)
                self._graph = g
            else:
                self._graph.replay()
            hi = min(n_batches, lo + win)
            red = counts[lo:hi].clone()
            sum_counts(red, group)
            host = torch.empty(tuple(red.shape), dtype=torch.int64, pin_memory=True)
            host.copy_(red, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            return lo, host, ev

        tot, done, scan = (0, 0, 0), False, 0
        cur = launch(0)
        while True:
            nxt = launch(scan)      # look-ahead round, queued before this one is read
            lo, host, ev = cur
            ev.synchronize()
            rows = host.numpy()[scan - lo:]
            # consume the prefix of complete batches in order (harness.py:173-192)
            hi = 0
            while hi < rows.shape[0] and rows[hi, 0] == gref:
                hi += 1
            tot, done, used = ordered_prefix(rows[:hi], stop, max_frames, tot)
            scan += used
            if done or scan >= n_batches:
                break
            cur = nxt
        torch.cuda.synchronize()
        return tot


def run_block_simulation(layout: EdgeLayout, config: SimulationConfig, *,
                         gamma_kernel: int | None = None, group=None, recycle: bool | None = None,
                         batches_per_launch: int | None = None) -> list:
    """Sweep the Eb/N0 points with the GPU block decoder (harness.py:157-204).

    early_stop campaigns on regular (J, 24) QC codes use lane recycling
    (`RecycleCampaign`, identical counts) unless recycle=False."""
    torch = require_cuda()
    rank, W, g = world() if group is None else (torch.distributed.get_rank(group),
                                                 torch.distributed.get_world_size(group), group)
    if config.early_stop and (recycle if recycle is not None else RecycleCampaign.supports(layout)):
        return _run_block_recycled(layout, config, gamma_kernel, rank, W, g)
    rate = 1.0 - layout.n_checks / layout.n_vars
    info_bits = layout.n_vars - layout.n_checks
    gref = config.gamma
    max_units = max(1, -(-config.max_frames // (gref * W)))
    units = batches_per_launch or _kernel_units(gref, gamma_kernel or 2048, max_units)
    eng = BlockCampaign(layout, gref, units, config.iterations, config.early_stop, config.seed)
    results = []
    for pi, db in enumerate(config.points()):
        sigma = ebn0_to_sigma(db, rate)
        lane_base = pi << 32
        # the point's first step runs eagerly and captures its CUDA graph: do it
        # before the clock starts (counts are per step, so it changes nothing)
        eng.step(lane_base, sigma)
        bufs = _round_buffers(units, W)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tot = _run_rounds(lambda rnd: eng.step(lane_base + ((rnd * W + rank) * units) * gref, sigma),
                          lambda: eng.counts, units, gref, rank, W, g, config.stop_block_errors,
                          config.max_frames, bufs)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        frames, be, fe = tot
        results.append(PointResult(
            code_id=config.code_id, mode="block", ebn0_db=db, iters_or_i=config.iterations,
            gamma=gref, frames=frames, bit_errors=be, frame_errors=fe,
            ber=be / (frames * layout.n_vars) if frames else 0.0,
            fer=fe / frames if frames else 0.0, seconds=dt,
            frames_per_sec=frames / dt if dt else 0.0,
            info_bits_per_sec=frames * info_bits / dt if dt else 0.0))
    return results


def _run_block_recycled(layout, config, gamma_kernel, rank, W, g):
    import torch
    rate = 1.0 - layout.n_checks / layout.n_vars
    info_bits = layout.n_vars - layout.n_checks
    gk = max(128, (gamma_kernel or 4096) // 128 * 128)
    eng = RecycleCampaign(layout, config.gamma, gk, config.iterations, config.seed, rank, W)
    results = []
    for pi, db in enumerate(config.points()):
        sigma = ebn0_to_sigma(db, rate)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        frames, be, fe = eng.run_point(sigma, pi << 32, config.stop_block_errors, config.max_frames, g)
        dt = time.perf_counter() - t0
        results.append(PointResult(
            code_id=config.code_id, mode="block", ebn0_db=db, iters_or_i=config.iterations,
            gamma=config.gamma, frames=frames, bit_errors=be, frame_errors=fe,
            ber=be / (frames * layout.n_vars) if frames else 0.0,
            fer=fe / frames if frames else 0.0, seconds=dt,
            frames_per_sec=frames / dt if dt else 0.0,
            info_bits_per_sec=frames * info_bits / dt if dt else 0.0))
    return results


class StreamCampaign:
    """Device-resident stream-segment engine: S segments of gamma_ref lanes side by side."""

    def __init__(self, code: LdpcccCode, gamma_ref: int, segments: int, processors: int,
                 pushes: int, seed: int, graph: bool = True):
        torch = require_cuda()
        self.code, self.gref, self.S, self.I, self.pushes = code, gamma_ref, segments, processors, pushes
        self.gk = gamma_ref * segments          # counted lanes
        self.gp = pad32(self.gk)                 # lanes the kernels run
        self.window = processors * (code.ms + 1)
        self.k0, self.k1 = seed_words(seed)
        self.plan = code.plan()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.msg = torch.zeros((processors * code.edge_count, self.gp), dtype=torch.float32, device=dev)
        self.ring = torch.zeros((self.window, code.c, self.gp), dtype=torch.float32, device=dev)
        # channel LLRs of K frames per launch (cc_channel_frames): one launch of
        # ~8M normals fills the machine where a single small frame is latency-bound
        # (running the batches on a side stream beside the slot kernels measured
        # no faster, profiles/r02/sbench_lookahead.md)
        self.K = max(1, min(pushes, 16, (8 << 20) // max(1, code.c * self.gp)))
        self.mu = torch.zeros((self.K, code.c, self.gp), dtype=torch.float32, device=dev)
        self.cnt = torch.zeros((3, self.gp), dtype=torch.int32, device=dev)
        self.lane0 = torch.zeros(1, dtype=torch.int64, device=dev)
        self.sigma = None
        self._graph = None
        self._use_graph = graph

    def _channel(self, b, s):
        t = b * self.K
        _lib.call("cc_channel_frames", self.plan.handle, self.k0, self.k1, 0, self.lane0.data_ptr(), t,
                  min(self.K, self.pushes - t), self.gp, float(self.sigma), self.mu.data_ptr(), s)

    def _frame(self, t):
        return self.mu[t % self.K].data_ptr()

    def _launch(self):
        # frame 0: channel batch + entry; then per slot t the look-ahead slot
        # (check phase, variable phase entering frame t + 1: two launches) with
        # the channel in batches of K frames -- the same results as
        # channel + cc_slot per slot (tests/test_gpu_stream.py)
        s = _lib.stream_handle()
        self.cnt.zero_()
        self._channel(0, s)
        _lib.call("cc_slot_part", self.plan.handle, self.I, self.gp, 0, None, self.msg.data_ptr(),
                  self.ring.data_ptr(), self._frame(0), None, self.cnt.data_ptr(), 0, 0, 1, s)
        for t in range(self.pushes):
            nxt = t + 1 < self.pushes
            if nxt and (t + 1) % self.K == 0:
                self._channel((t + 1) // self.K, s)     # after the slot that entered frame t (last of its batch)
            _lib.call("cc_slot_ahead", self.plan.handle, self.I, self.gp, t, None, self.msg.data_ptr(),
                      self.ring.data_ptr(), self._frame(t + 1) if nxt else None, int(nxt), None,
                      self.cnt.data_ptr(), s)
        _lib.call("cc_fold", self.cnt.data_ptr(), self.gp, s)

    def kernel_launches_per_step(self) -> int:
        # channel batches, entry of frame 0, (check, variable + next entry) per slot, final fold
        return -(-self.pushes // self.K) + 1 + 2 * self.pushes + 1

    def step(self, lane0: int, sigma: float):
        import torch
        self.lane0.fill_(int(lane0))
        if self.sigma != sigma:
            self.sigma, self._graph = sigma, None
        if not self._use_graph:
            self._launch()
            return
        if self._graph is None:
            self._launch()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch()
            self._graph = g
            return
        self._graph.replay()

    def segment_counts(self):
        """(S, 3) int64 (frames, bit_errors, frame_errors) per segment (device)."""
        import torch
        emitted = max(0, self.pushes - self.window + 1)
        c = self.cnt[:, : self.gk].reshape(3, self.S, self.gref).to(torch.int64).sum(dim=2)
        out = torch.empty((self.S, 3), dtype=torch.int64, device=self.cnt.device)
        out[:, 0] = emitted * self.gref
        out[:, 1] = c[1]
        out[:, 2] = c[2]
        return out


def run_stream_simulation(code: LdpcccCode, config: SimulationConfig, *,
                          gamma_kernel: int | None = None, group=None,
                          batches_per_launch: int | None = None) -> list:
    """Sweep the Eb/N0 points with the GPU pipelined stream decoder (harness.py:236-286)."""
    torch = require_cuda()
    rank, W, g = world() if group is None else (torch.distributed.get_rank(group),
                                                 torch.distributed.get_world_size(group), group)
    window = config.processors * (code.ms + 1)
    counted = config.stream_segment_frames or max(2 * (window - 1), 64)
    pushes = counted + window - 1
    info_bits = code.c - code.cb
    gref = config.gamma
    per_seg = counted * gref
    max_units = max(1, -(-config.max_frames // (per_seg * W)))
    units = batches_per_launch or _kernel_units(gref, gamma_kernel or 256, max_units)
    eng = StreamCampaign(code, gref, units, config.processors, pushes, config.seed)
    results = []
    for pi, db in enumerate(config.points()):
        sigma = ebn0_to_sigma(db, code.rate_bound)
        lane_base = pi << 32
        eng.step(lane_base, sigma)                 # eager run + graph capture, outside the clock
        bufs = _round_buffers(units, W)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tot = _run_rounds(lambda rnd: eng.step(lane_base + ((rnd * W + rank) * units) * gref, sigma),
                          eng.segment_counts, units, per_seg, rank, W, g, config.stop_block_errors,
                          config.max_frames, bufs)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        frames, be, fe = tot
        results.append(PointResult(
            code_id=config.code_id, mode="stream", ebn0_db=db, iters_or_i=config.processors,
            gamma=gref, frames=frames, bit_errors=be, frame_errors=fe,
            ber=be / (frames * code.c) if frames else 0.0,
            fer=fe / frames if frames else 0.0, seconds=dt,
            frames_per_sec=frames / dt if dt else 0.0,
            info_bits_per_sec=frames * info_bits / dt if dt else 0.0))
    return results


def bench_throughput(layout: EdgeLayout | None, config: SimulationConfig,
                     code: LdpcccCode | None = None, frames: int = 256) -> list:
    """Decoded-frames/s records for gamma in {1, config.gamma} x workers in
    {1, cpu_count} (harness.py:294-331), same keys as the reference.

    The reference's `workers` are processes that each decode one gamma-lane
    batch at a time, so `workers` batches are in flight at once.  On the GPU
    the same concurrency is one kernel launch over `workers` reference batches
    side by side (gamma_kernel = workers x gamma lanes, padded to a multiple of
    32; padding lanes are not counted): workers = 1 decodes one batch per
    launch, workers = cores decodes cores batches per launch.  Each record
    adds `batches_per_launch` and `lanes_per_launch` to say so."""
    cores = multiprocessing.cpu_count()
    records = []
    db = config.points()[0]
    for gamma in sorted({1, config.gamma}):
        for workers in sorted({1, cores}):
            cfg = dataclasses.replace(config, gamma=gamma, workers=workers, stop_block_errors=2**62,
                                      max_frames=frames, ebn0_db=db)
            if code is not None:
                per_unit = (config.stream_segment_frames or
                            max(2 * (config.processors * (code.ms + 1) - 1), 64)) * gamma
                units = min(workers, max(1, -(-frames // per_unit)))
                res = run_stream_simulation(code, cfg, batches_per_launch=units)[0]
                meta = dict(mode="stream", n=code.c, m=code.cb, edge_count=code.edge_count,
                            iters_or_I=config.processors)
            else:
                units = min(workers, max(1, -(-frames // gamma)))
                res = run_block_simulation(layout, cfg, batches_per_launch=units, recycle=False)[0]
                meta = dict(mode="block", n=layout.n_vars, m=layout.n_checks,
                            edge_count=layout.edge_count, iters_or_I=config.iterations)
            records.append(dict(
                code_id=config.code_id, gamma=gamma, workers=workers, physical_cores=cores,
                frames=res.frames, seconds=round(res.seconds, 4),
                frames_per_sec=round(res.frames_per_sec, 3),
                info_bits_per_sec=round(res.info_bits_per_sec, 1),
                per_frame_ms=round(1000 * res.seconds / res.frames, 4) if res.frames else None,
                batches_per_launch=units, lanes_per_launch=pad32(units * gamma),
                **meta))
    return records
