"""CPU oracle for the qcldpc hot path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference's algorithms on
the decoding hot path (`/root/reference/pkg/src/qcldpc/{codes,bp,channel,
convolutional,harness}.py`).  Every function cites the reference file:line it
follows.  It exists to *check* the B200 path, never to *be* it:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
  leg and `--impl reference` arm) may import it;
* the product package `paper_1204_0334_b200` never imports it and fails loudly
  when its CUDA library is missing.

Parity pinning: the oracle is pinned against golden vectors produced by the
real reference (imported from /root/reference in the build container) by
`tests/golden/make_golden.py`; the fixtures are committed under
`tests/golden/` and checked by `tests/test_oracle.py` (CPU).  Known-answer
values from the reference's own tests (`test_bp.py:15-22`,
`test_channel.py:10-13`, `test_convolutional.py:12-13`) and the recorded
campaign counts (`pkg/test_output.txt:27,30`) are restated there too.
"""

from . import bp, campaign, channel, qc, stream  # noqa: F401
