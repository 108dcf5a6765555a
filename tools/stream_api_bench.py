#!/usr/bin/env python
"""LDPCCC through the public API: StreamDecoder.push_frame throughput and
per-frame latency (convolutional.py:220-246 drop-in), next to the
device-resident StreamCampaign on the same code / I / gamma.

    python tools/stream_api_bench.py [--code n18360] [--I 20] [--gammas 32 512] [--frames 400]

push_frame: host numpy y (gamma, c) in, DecodedFrame (fp64 posteriors, u8
bits) out per emitted frame.  Latency = wall time of one push_frame call in
steady state (the emitted frame is frame t - I*T + 1: pipeline depth I*T
slots); throughput = info bits of emitted frames / wall time.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="n18360")
    ap.add_argument("--I", type=int, default=20)
    ap.add_argument("--gammas", type=int, nargs="+", default=[32, 512])
    ap.add_argument("--frames", type=int, default=400)
    ap.add_argument("--ebn0", type=float, default=3.1)
    a = ap.parse_args()
    import torch
    import paper_1204_0334_b200 as q
    h, exp = q.load_code(q.codes.bundled_code_path(a.code))
    code = q.unwrap_qc(exp)
    sigma = q.ebn0_to_sigma(a.ebn0, code.rate_bound)
    info = code.c - code.cb
    for G in a.gammas:
        rng = np.random.default_rng(0)
        ys = [1.0 + sigma * rng.standard_normal((G, code.c)) for _ in range(8)]
        dec = q.StreamDecoder(code, a.I, gamma=G)
        warm = dec.window + 8
        for t in range(warm):
            dec.push_frame(ys[t % 8], sigma)
        torch.cuda.synchronize()
        lat = []
        t0 = time.perf_counter()
        for t in range(a.frames):
            s = time.perf_counter()
            fr = dec.push_frame(ys[t % 8], sigma)
            lat.append(time.perf_counter() - s)
            assert fr is not None
        dt = time.perf_counter() - t0
        lat.sort()
        # device-resident engine on the same shape: one segment step of `pushes` slots
        window = a.I * (code.ms + 1)
        counted = max(2 * (window - 1), 64)
        pushes = counted + window - 1
        S = max(1, G // 32)
        eng = q.StreamCampaign(code, min(G, 32), S, a.I, pushes, seed=0)
        eng.step(0, sigma)
        eng.step(G, sigma)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step(2 * G, sigma)
        e1.record()
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1)
        dev_rate = counted * min(G, 32) * S * info / (dev_ms / 1e3) / 1e6
        print(json.dumps({
            "code": a.code + "'", "I": a.I, "gamma": G, "frames": a.frames,
            "push_frame_mbit_s": round(a.frames * G * info / dt / 1e6, 2),
            "push_frame_ms_per_slot": round(dt / a.frames * 1e3, 4),
            "latency_ms_p50": round(lat[len(lat) // 2] * 1e3, 4),
            "latency_ms_p99": round(lat[int(len(lat) * 0.99)] * 1e3, 4),
            "latency_ms_mean": round(sum(lat) / len(lat) * 1e3, 4), "latency_ms_max": round(lat[-1] * 1e3, 3),
            "frame_latency_ms_p50": round(lat[len(lat) // 2] * 1e3 * window, 2),
            "device_resident_mbit_s": round(dev_rate, 2),
            "device_ms_per_slot": round(dev_ms / pushes, 4),
        }), flush=True)
        del dec, eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
