"""Oracle port vs the real reference on one core: same batches, same outputs.

    python tools/port_vs_reference.py [--batches 6] > profiles/r02/port_vs_reference.json

Times `oracle.campaign.block_task` (the numpy float64 restatement bench.py
falls back to) against the reference's own `qcldpc.harness._block_task`
(installed in oracle/_ref by oracle/build_ref.py) on n18360, gamma 32, 30
iterations, 3.2 dB, alternating which goes first; checks the per-batch counts
and the full decode outputs are bit-identical.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from oracle import build_ref  # noqa: E402

sys.path.insert(0, build_ref.site_dir())
import qcldpc  # noqa: E402
from qcldpc.harness import _block_task, _init_block  # noqa: E402

from oracle import bp, campaign, channel, qc  # noqa: E402
from paper_1204_0334_b200 import codes as pc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=6)
    a = ap.parse_args()
    _, exp = pc.load_code(pc.bundled_code_path("n18360"))
    lay = qc.qc_layout(exp.shifts, exp.p)
    rlay = qcldpc.build_edge_layout(qcldpc.expand_qc(qcldpc.ExponentMatrix(exp.shifts, exp.p)))
    sigma = channel.ebn0_to_sigma(3.2, 1 - lay.n_checks / lay.n_vars)
    _init_block(rlay, qcldpc.SimulationConfig("n18360", [3.2], iterations=30, gamma=32), sigma, 0)
    campaign._init(lay=lay, seed=0, sigma=sigma, gamma=32, iters=30, lane0=0)
    tr, tp = [], []
    for b in range(a.batches):
        order = [("ref", _block_task), ("port", campaign.block_task)]
        if b % 2:
            order.reverse()
        got = {}
        for name, fn in order:
            t0 = time.perf_counter()
            got[name] = fn(b)
            (tr if name == "ref" else tp).append(time.perf_counter() - t0)
        assert got["ref"] == got["port"], (b, got)
    # full outputs (bits, posteriors, ok) of one batch, bit for bit
    y = channel.received(0, sigma, 0, 32, lay.n_vars)
    r = qcldpc.decode_batch(rlay, y, sigma, 30)
    bits, post, ok, _ = bp.decode_llr(lay, bp.channel_llrs(y, sigma), 30)
    same = bool(np.array_equal(r.hard_bits, bits) and np.array_equal(r.posteriors, post)
                and np.array_equal(r.syndrome_ok, ok))
    med = lambda x: sorted(x)[len(x) // 2]
    print(json.dumps({"workload": "n18360 gamma 32, 30 it, 3.2 dB, 1 core", "batches": a.batches,
                      "reference_s_per_batch": [round(x, 3) for x in tr],
                      "port_s_per_batch": [round(x, 3) for x in tp],
                      "median_ratio_port_over_reference": round(med(tp) / med(tr), 3),
                      "outputs_bit_identical": same}))


if __name__ == "__main__":
    main()
