#!/usr/bin/env python
"""BASELINE configs[3]: BER/FER Monte-Carlo Eb/N0 sweep of the n=18360 code at
30 flooding iterations, stop at `--stop` frame errors per point (PAPER.md:
1349-1351 uses 100), until BER <= 1e-6 -- through the drop-in harness API
(`run_block_simulation`), optionally sharded over GPUs with torchrun.

  python tools/ber_sweep.py --ebn0 2.6 2.8 3.0 3.2 3.4 3.6 --stop 100 --out profiles/r01/ber_n18360.csv
  python tools/ber_sweep.py --stream 20 --ebn0 ... # LDPCCC (unwrapped code, I = 20 window decoder)
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="n18360")
    ap.add_argument("--ebn0", type=float, nargs="+", default=[2.6, 2.8, 3.0, 3.2, 3.4, 3.6])
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--stop", type=int, default=100)
    ap.add_argument("--max-frames", type=int, default=20_000_000)
    ap.add_argument("--gamma-kernel", type=int, default=4096)
    ap.add_argument("--out", default=None)
    ap.add_argument("--stream", type=int, default=0, help="LDPCCC sweep with this many processors I")
    args = ap.parse_args()
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200.dist import init_from_env
    rank, W, _ = init_from_env()
    h, exp = q.load_code(q.codes.bundled_code_path(args.code))
    lay = q.build_edge_layout(h)
    rows = []
    t0 = time.time()
    for db in args.ebn0:
        if args.stream:
            cfg = q.SimulationConfig(code_id=args.code + "'", ebn0_db=[db], processors=args.stream, gamma=32,
                                     stop_block_errors=args.stop, max_frames=args.max_frames, seed=0)
            r = q.run_stream_simulation(q.unwrap_qc(exp), cfg, gamma_kernel=min(args.gamma_kernel, 512))[0]
        else:
            cfg = q.SimulationConfig(code_id=args.code, ebn0_db=[db], iterations=args.iters, gamma=32,
                                     stop_block_errors=args.stop, max_frames=args.max_frames, seed=0)
            r = q.run_block_simulation(lay, cfg, gamma_kernel=args.gamma_kernel)[0]
        rows.append(r)
        if rank == 0:
            print(",".join(str(x) for x in r.row()), flush=True)
        if r.ber <= 1e-6 and r.frame_errors >= args.stop:
            break
    if rank == 0:
        print(f"# {W} GPU(s), {time.time() - t0:.1f} s wall", flush=True)
        if args.out:
            q.write_csv(rows, args.out)


if __name__ == "__main__":
    main()
