#!/usr/bin/env python
"""Early-stop campaign throughput on n18360 (30-iteration cap): lane recycling
vs plain batched early stop vs fixed 30 iterations, fixed frame budget per point.

  python tools/es_bench.py --ebn0 3.0 3.2 3.4 3.6 --frames 65536
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ebn0", type=float, nargs="+", default=[3.0, 3.2, 3.4, 3.6])
    ap.add_argument("--frames", type=int, default=65536)
    ap.add_argument("--gamma-kernel", type=int, default=4096)
    ap.add_argument("--modes", nargs="+", default=["fixed30", "early_stop", "recycled"])
    ap.add_argument("--repeat", type=int, default=3)
    args = ap.parse_args()
    import paper_1204_0334_b200 as q
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    for db in args.ebn0:
        row = {"ebn0_db": db, "frames": args.frames}
        for name, es, rec in (("fixed30", False, None), ("early_stop", True, False), ("recycled", True, True)):
            if name not in args.modes:
                continue
            cfg = q.SimulationConfig("n18360", [db], iterations=30, gamma=32, stop_block_errors=2**62,
                                     max_frames=args.frames, seed=0, early_stop=es)
            q.run_block_simulation(lay, cfg, gamma_kernel=args.gamma_kernel, recycle=rec)   # warm-up
            runs = [q.run_block_simulation(lay, cfg, gamma_kernel=args.gamma_kernel, recycle=rec)[0]
                    for _ in range(args.repeat)]
            r = max(runs, key=lambda x: x.info_bits_per_sec)      # wall-clock campaign: best of repeats
            row[name] = {"mbit_s": round(r.info_bits_per_sec / 1e6, 1), "frame_errors": r.frame_errors,
                         "bit_errors": r.bit_errors}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
