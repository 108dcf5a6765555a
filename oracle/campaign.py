"""Monte-Carlo campaign restatement (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/qcldpc/harness.py:
* block task: batch b of point pi draws lanes (pi<<32) + b*gamma + g at
  positions 0..N-1, decodes, returns (gamma, bit errors, frame errors)
  (harness.py:140-154);
* ordered accumulation with the stop rule "frame_errors >= stop or frames >=
  max_frames" checked after every batch (harness.py:157-204);
* stream task: segment s draws lanes (pi<<32) + s*gamma + g, frame t at
  position t*c, pushes = counted + window - 1, counting push-emitted frames
  only (harness.py:212-286).
`workers > 1` runs tasks on a multiprocessing pool and consumes results in
order exactly as harness.py:183-193 does; this is the CPU baseline bench.py
times beside the GPU.
"""

from __future__ import annotations

import itertools
import multiprocessing

import numpy as np

from . import bp, channel
from .stream import StreamOracle

_W = {}


def _init(**kw):
    _W.clear()
    _W.update(kw)


def block_task(b: int):
    lay, seed, sigma, gamma, iters, lane0 = (_W[k] for k in
                                             ("lay", "seed", "sigma", "gamma", "iters", "lane0"))
    y = channel.received(seed, sigma, lane0 + b * gamma, gamma, lay.n_vars)
    bits, _, _, _ = bp.decode_llr(lay, bp.channel_llrs(y, sigma), iters, _W.get("early", False))
    return gamma, int(bits.sum()), int(bits.any(axis=1).sum())


def stream_task(s: int):
    code, seed, sigma, gamma, I, pushes, lane0 = (_W[k] for k in (
        "code", "seed", "sigma", "gamma", "I", "pushes", "lane0"))
    dec = StreamOracle(code, I, gamma)
    fr = be = fe = 0
    for t in range(pushes):
        y = channel.received(seed, sigma, lane0 + s * gamma, gamma, code.c, start=t * code.c)
        out = dec.push(y, sigma)
        if out is not None:
            fr += gamma
            be += int(out.hard_bits.sum())
            fe += int(out.hard_bits.any(axis=1).sum())
    return fr, be, fe


def ping(_):
    """No-op task: brings a pool's workers up outside a timed region."""
    return 0


def _run(task, init_kw, stop, max_frames, workers, start_method="fork"):
    fr = be = fe = 0
    if workers <= 1:
        _init(**init_kw)
        for b in itertools.count():
            if fe >= stop or fr >= max_frames:
                break
            f, e1, e2 = task(b)
            fr += f; be += e1; fe += e2
    else:
        # "spawn" from processes that initialised CUDA or thread pools (a forked
        # child of such a process can abort in its after-fork hooks)
        with multiprocessing.get_context(start_method).Pool(
                workers, initializer=_set_ctx, initargs=(init_kw,)) as pool:
            for f, e1, e2 in pool.imap(task, itertools.count()):
                fr += f; be += e1; fe += e2
                if fe >= stop or fr >= max_frames:
                    break
            pool.terminate()
    return fr, be, fe


def _set_ctx(kw):
    _init(**kw)


def block_point(lay, ebn0_db, point_index=0, *, iters=30, gamma=32, seed=0,
                stop=100, max_frames=1_000_000, workers=1, early_stop=False, start_method="fork"):
    rate = 1.0 - lay.n_checks / lay.n_vars
    sigma = channel.ebn0_to_sigma(ebn0_db, rate)
    kw = dict(lay=lay, seed=seed, sigma=sigma, gamma=gamma, iters=iters,
              lane0=point_index << 32, early=early_stop)
    return _run(block_task, kw, stop, max_frames, workers, start_method)


def stream_point(code, ebn0_db, point_index=0, *, processors=20, gamma=32, seed=0,
                 stop=100, max_frames=1_000_000, workers=1, segment_frames=None, start_method="fork"):
    window = processors * (code.ms + 1)
    counted = segment_frames or max(2 * (window - 1), 64)
    sigma = channel.ebn0_to_sigma(ebn0_db, (code.c - code.cb) / code.c)
    kw = dict(code=code, seed=seed, sigma=sigma, gamma=gamma, I=processors,
              pushes=counted + window - 1, lane0=point_index << 32)
    return _run(stream_task, kw, stop, max_frames, workers, start_method)


def sum_counts(rows):
    return tuple(int(x) for x in np.sum(np.asarray(rows, dtype=np.int64), axis=0))
