#!/usr/bin/env python
"""BASELINE configs[4]: LDPCCC throughput / latency sweep over the window size
(processors I) and gamma on the GPU, next to the reference CPU path (oracle
port of StreamDecoder, numpy float64) timed on the host's cores.

GPU: harness segments (counted = 2(window-1), pushes = counted + window - 1),
every slot on the device, one CUDA graph per segment group.
CPU: steady-state slot time of StreamOracle with gamma = 32 lanes, one
independent decoder per core in parallel (bounded sample: window + 8 slots).
Latency = I*T slots (a frame leaves the pipeline I*T - 1 slots after entry).

  python tools/ldpccc_sweep.py --I 5 10 20 30 --gammas 32 512 --cpu
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def _cpu_slot_time(args):
    """Steady-state slot time of the reference's own StreamDecoder (qcldpc from
    oracle/_ref, unmodified) when installed, else the oracle port."""
    code_name, I, G, seed = args
    import numpy as np
    from oracle import build_ref, qc, stream
    import paper_1204_0334_b200 as q
    _, exp = q.load_code(q.codes.bundled_code_path(code_name))
    if build_ref.available():
        sys.path.insert(0, build_ref.site_dir())
        import qcldpc
        code = qcldpc.unwrap_qc(qcldpc.ExponentMatrix(exp.shifts, exp.p))
        dec = qcldpc.StreamDecoder(code, I, gamma=G)
        push, c, window = dec.push_frame, code.c, I * (code.ms + 1)
    else:
        U = qc.unwrap(exp.shifts, exp.p)
        dec = stream.StreamOracle(U, I, G)
        push, c, window = dec.push, U.c, I * (U.ms + 1)
    rng = np.random.default_rng(seed)
    sigma = 0.55
    for _ in range(window):
        push(rng.normal(1.0, sigma, size=(G, c)), sigma)
    t0 = time.perf_counter()
    n = 8
    for _ in range(n):
        push(rng.normal(1.0, sigma, size=(G, c)), sigma)
    return (time.perf_counter() - t0) / n


def _ref_available():
    from oracle import build_ref
    return build_ref.available()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="n18360")
    ap.add_argument("--I", type=int, nargs="+", default=[5, 10, 20, 30])
    ap.add_argument("--gammas", type=int, nargs="+", default=[32, 512])
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--cpu-I", type=int, nargs="+", default=[5, 20])
    args = ap.parse_args()
    import torch
    import paper_1204_0334_b200 as q
    _, exp = q.load_code(q.codes.bundled_code_path(args.code))
    code = q.unwrap_qc(exp)
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    b = code.c - code.cb
    for I in args.I:
        window = I * (code.ms + 1)
        counted = max(2 * (window - 1), 64)
        pushes = counted + window - 1
        slot_bytes = 4 * (4 * I * code.edge_count // code.lam + (I + 1) * code.c)
        for G in args.gammas:
            eng = q.StreamCampaign(code, 32, G // 32, I, pushes, seed=0)
            sigma = q.ebn0_to_sigma(3.1, code.rate_bound)
            eng.step(0, sigma)
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eng.step(G, sigma)
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e)
            us_slot = ms * 1e3 / pushes
            print(json.dumps({"side": "gpu", "code": args.code, "I": I, "gamma": G,
                              "us_per_slot": round(us_slot, 2),
                              "steady_mbit_s": round(G * b / us_slot, 1),
                              "segment_mbit_s": round(counted * G * b / (ms * 1e3), 1),
                              "frac": round(slot_bytes * G / (us_slot * 1e-6) / 1e9 / peak, 4),
                              "latency_ms": round(window * us_slot / 1e3, 3)}), flush=True)
            del eng
            torch.cuda.empty_cache()
    if args.cpu:
        cores = len(os.sched_getaffinity(0))
        for I in args.cpu_I:
            with mp.get_context("spawn").Pool(cores) as pool:   # this process initialised CUDA
                ts = pool.map(_cpu_slot_time, [(args.code, I, 32, k) for k in range(cores)])
            t = sorted(ts)[len(ts) // 2]
            window = I * (code.ms + 1)
            print(json.dumps({"side": "cpu", "code": args.code, "I": I, "gamma": 32, "cores": cores,
                              "us_per_slot": round(t * 1e6, 1),
                              "steady_mbit_s": round(cores * 32 * b / (t * 1e6), 3),
                              "latency_ms": round(window * t * 1e3, 1),
                              "impl": ("qcldpc.StreamDecoder (the reference, unmodified, oracle/_ref)"
                                       if _ref_available() else "oracle port of StreamDecoder (numpy float64)")
                                      + ", one decoder per core"}),
                  flush=True)


if __name__ == "__main__":
    main()
