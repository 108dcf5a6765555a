#!/usr/bin/env python
"""GPU campaign counts vs the float64 oracle campaign on the same seeds, at an
Eb/N0 where many frames fail (so bit-error counts inside failed frames are
exercised, not just converged frames).  Oracle on all host cores.

  python tools/campaign_parity.py --ebn0 3.0 --frames 2048 [--code n18360]
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="n18360")
    ap.add_argument("--ebn0", type=float, nargs="+", default=[3.0])
    ap.add_argument("--frames", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--stream", type=int, default=0, help="LDPCCC campaign with this many processors I")
    args = ap.parse_args()
    import paper_1204_0334_b200 as q
    from oracle import campaign, qc
    h, exp = q.load_code(q.codes.bundled_code_path(args.code))
    lay = q.build_edge_layout(h)
    olay = qc.qc_layout(exp.shifts, exp.p)
    workers = len(os.sched_getaffinity(0))
    if args.stream:
        code = q.unwrap_qc(exp)
        ocode = qc.unwrap(exp.shifts, exp.p)
        for db in args.ebn0:
            cfg = q.SimulationConfig(args.code, [db], processors=args.stream, gamma=32, stop_block_errors=2**62,
                                     max_frames=args.frames, seed=0)
            g = q.run_stream_simulation(code, cfg)[0]
            t0 = time.time()
            o = campaign.stream_point(ocode, db, 0, processors=args.stream, gamma=32, seed=0, stop=2**62,
                                      max_frames=args.frames, workers=workers, start_method="spawn")
            print(json.dumps({"code": args.code + "'", "I": args.stream, "ebn0_db": db,
                              "gpu": [g.frames, g.bit_errors, g.frame_errors], "oracle_f64": list(o),
                              "identical": [g.frames, g.bit_errors, g.frame_errors] == list(o),
                              "oracle_s": round(time.time() - t0, 1)}), flush=True)
        return
    for pi, db in enumerate(args.ebn0):
        cfg = q.SimulationConfig(args.code, [db], iterations=args.iters, gamma=32, stop_block_errors=2**62,
                                 max_frames=args.frames, seed=0)
        g = q.run_block_simulation(lay, cfg)[0]
        t0 = time.time()
        o = campaign.block_point(olay, db, 0, iters=args.iters, gamma=32, seed=0, stop=2**62,
                                 max_frames=args.frames, workers=workers, start_method="spawn")
        print(json.dumps({"code": args.code, "ebn0_db": db, "gpu": [g.frames, g.bit_errors, g.frame_errors],
                          "oracle_f64": list(o), "identical": [g.frames, g.bit_errors, g.frame_errors] == list(o),
                          "oracle_s": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
