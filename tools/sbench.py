#!/usr/bin/env python
"""LDPCCC slot micro-benchmark: one StreamCampaign segment group (18360' or A'),
per-slot time and algorithmic GB/s.  Used for ncu captures of the stream kernels.

  python tools/sbench.py --gamma 256 --I 20 [--code n18360|code_a --steps 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gamma", type=int, default=256)
    ap.add_argument("--I", type=int, default=20)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--code", default="n18360")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1204_0334_b200 as q
    if args.code == "code_a":
        d = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "codes.npz"))
        exp = q.ExponentMatrix(d["code_a_shifts"], int(d["code_a_p"]))
    else:
        _, exp = q.load_code(q.codes.bundled_code_path(args.code))
    code = q.unwrap_qc(exp)
    window = args.I * (code.ms + 1)
    counted = max(2 * (window - 1), 64)
    pushes = counted + window - 1
    G = args.gamma
    eng = q.StreamCampaign(code, 32, G // 32, args.I, pushes, seed=0, graph=not args.no_graph)
    sigma = q.ebn0_to_sigma(3.1, code.rate_bound)
    eng.step(0, sigma)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in range(args.steps):
        eng.step((s + 1) * G, sigma)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    slot = 4 * (4 * args.I * code.edge_count // code.lam + (args.I + 1) * code.c)
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    gbs = slot * G * pushes / (ms / 1e3) / 1e9
    print(json.dumps({"K": eng.K, "code": args.code, "I": args.I, "gamma": G, "pushes": pushes, "ms_per_segment": round(ms, 3),
                      "us_per_slot": round(ms * 1e3 / pushes, 2), "alg_gbs": round(gbs, 1),
                      "frac": round(gbs / peak, 4),
                      "mbit_s": round(counted * G * (code.c - code.cb) / (ms / 1e3) / 1e6, 1),
                      # a frame is decoded I*T slots after it is pushed
                      "latency_ms": round(window * ms / pushes, 3)}), flush=True)


if __name__ == "__main__":
    main()
