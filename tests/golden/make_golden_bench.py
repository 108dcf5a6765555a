"""Golden campaign counts at the bench configurations, from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_bench.py

Runs the reference harness (`qcldpc.harness.run_block_simulation` /
`run_stream_simulation`, harness.py:157-286) on the configurations bench.py
measures, sized to finish in a few CPU minutes:
* n18360, 3.0 dB, 30 iterations, gamma 32, 1024 frames (32 reference batches),
* 18360' (the unwrapped n18360 grid), 3.1 dB, I = 20, gamma 32, one stream
  segment (158 counted frames x 32 lanes = 5056 frames).
The GPU tests replay them at the bench's kernel batch sizes (gamma 1024 block,
gamma 512 stream) and must reproduce every count.
"""

import json
import os
import sys
import time

import qcldpc
from qcldpc.harness import SimulationConfig, run_block_simulation, run_stream_simulation

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def main():
    _, exp_n = qcldpc.load_code(os.path.join(REPO, "paper_1204_0334_b200", "data", "n18360.qc"))
    out = {}
    t0 = time.time()
    lay = qcldpc.build_edge_layout(qcldpc.expand_qc(exp_n))
    cfg = SimulationConfig(code_id="n18360", ebn0_db=[3.0], iterations=30, gamma=32,
                           stop_block_errors=2**62, max_frames=1024, seed=0)
    out["n18360_block_3.0dB_30it_1024"] = [r.row()[:10] for r in run_block_simulation(lay, cfg)]
    print("block", time.time() - t0, out, flush=True)
    code = qcldpc.unwrap_qc(exp_n)
    cfg = SimulationConfig(code_id="n18360p", ebn0_db=[3.1], processors=20, gamma=32,
                           stop_block_errors=2**62, max_frames=5056, seed=0)
    out["n18360p_stream_3.1dB_I20_5056"] = [r.row()[:10] for r in run_stream_simulation(code, cfg)]
    print("stream", time.time() - t0, out, flush=True)
    with open(os.path.join(HERE, "campaigns_bench.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    sys.exit(main())
