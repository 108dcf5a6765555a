"""Test oracles of the reference's `qcldpc.reference` module (TEST INFRASTRUCTURE ONLY).

The product package deliberately does not ship these two names (they are
oracles, not decoders: one enumerates 2^N codewords on the CPU, the other
replays the stream schedule on the CPU).  The reference-suite conformance
run (tests/test_ref_conformance.py) maps `qcldpc.reference` here.

* exact_posterior_llr -- /root/reference/pkg/src/qcldpc/reference.py:25-60:
  bitwise posterior LLR ln P(c_n=0|y)/P(c_n=1|y) by enumerating every word of
  length N <= 20 that satisfies all checks, with word weight exp(-sum c_n mu_n).
* reference_window_decoder -- reference.py:79-182: decode one finite stream
  (gamma = 1) through the pipelined slot schedule, including the zero-LLR tail
  padding of flush.  Restated with oracle.stream.StreamOracle, the float64
  restatement of StreamDecoder (convolutional.py:180-357), which the reference
  itself proves bit-identical to its direct replay (test_convolutional.py:
  135-153) and which tests/test_oracle.py pins to the reference's goldens.
"""

from __future__ import annotations

import numpy as np

from . import qc
from .stream import StreamOracle


def exact_posterior_llr(h, mu) -> np.ndarray:
    """h: object with `.n` and `.rows` (lists of column indices); mu (N,)."""
    mu = np.asarray(mu, dtype=np.float64)
    n = mu.size
    if n > 20:
        raise ValueError("enumeration over 2^N words is limited to N <= 20")
    ids = np.arange(1 << n, dtype=np.int64)
    bits = ((ids[:, None] >> np.arange(n)) & 1).astype(bool)         # (2^N, N)
    ok = np.ones(1 << n, dtype=bool)
    for cols in h.rows:
        ok &= (np.count_nonzero(bits[:, list(cols)], axis=1) % 2) == 0
    words = bits[ok]
    logw = -(words.astype(np.float64) @ mu)                           # log weight up to a constant
    out = np.empty(n)
    for i in range(n):
        zero, one = logw[~words[:, i]], logw[words[:, i]]
        lz = np.logaddexp.reduce(zero) if zero.size else -np.inf
        lo = np.logaddexp.reduce(one) if one.size else -np.inf
        with np.errstate(invalid="ignore"):
            out[i] = lz - lo
    return out


def reference_window_decoder(code, processors: int, llr_frames):
    """(bits, posteriors): one entry per pushed frame (uint8 bits, float64 LLRs)."""
    u = qc.unwrap(np.asarray(code.exp.shifts), int(code.exp.p))
    dec = StreamOracle(u, processors, 1)
    k = len(llr_frames)
    bits, posts = [None] * k, [None] * k
    frames = []
    for f in llr_frames:
        fr = dec.push_llr(np.asarray(f, dtype=np.float64).reshape(-1, 1))
        if fr is not None:
            frames.append(fr)
    for _ in range(dec.window - 1):
        fr = dec.push_llr(None, tail=True)
        if fr is not None:
            frames.append(fr)
    for fr in frames:
        if fr.frame_index < k:
            posts[fr.frame_index] = fr.posteriors[0]
            bits[fr.frame_index] = fr.hard_bits[0]
    return bits, posts
