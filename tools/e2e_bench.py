#!/usr/bin/env python
"""Host-buffer API sweep: decode_batch Mbit/s for n18360 at 30 it over the
pipeline's chunk / slot settings, with page-locked and pageable inputs.

  python tools/e2e_bench.py [--gamma 4096] [--chunks 256,512,1024] [--slots 2,3,4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gamma", type=int, default=4096)
    ap.add_argument("--chunks", default="256,512,1024")
    ap.add_argument("--slots", default="2,3,4")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--early-stop", action="store_true")
    ap.add_argument("--ebn0", type=float, default=3.2)
    ap.add_argument("--pinned-only", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import bp as qbp
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    N, K = lay.n_vars, lay.n_vars - lay.n_checks
    sigma = q.ebn0_to_sigma(args.ebn0, K / N)
    y_pg = 1.0 + sigma * np.random.default_rng(0).standard_normal((args.gamma, N))
    y_pin = q.host_array(y_pg)
    for c in map(int, args.chunks.split(",")):
        for s in map(int, args.slots.split(",")):
            qbp.HOST_CHUNK, qbp.HOST_SLOTS, qbp.HOST_SLOTS_PINNED = c, s, s
            lay.__dict__.pop("_host_decoders", None)
            torch.cuda.empty_cache()
            rec = {"chunk": c, "slots": s, "early_stop": args.early_stop, "ebn0_db": args.ebn0, "gamma": args.gamma}
            for name, y in ((("pinned", y_pin),) if args.pinned_only else (("pinned", y_pin), ("pageable", y_pg))):
                for _ in range(2):
                    r = q.decode_batch(lay, y, sigma, 30, early_stop=args.early_stop)
                del r
                t0 = time.perf_counter()
                for _ in range(args.steps):
                    r = q.decode_batch(lay, y, sigma, 30, early_stop=args.early_stop)
                    del r
                dt = (time.perf_counter() - t0) / args.steps
                rec[name + "_mbit_s"] = round(args.gamma * K / dt / 1e6, 1)
                rec[name + "_ms"] = round(dt * 1e3, 2)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
