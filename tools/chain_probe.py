#!/usr/bin/env python
"""Do two independent decode chains on two CUDA streams fill each other's
launch tails?  Times K decodes of gamma lanes on one stream vs the same work
split over two streams (two BlockDecoders, graph-replayed)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import _lib
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    K = 8
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    N, Kb = lay.n_vars, lay.n_vars - lay.n_checks
    sigma = q.ebn0_to_sigma(3.2, Kb / N)
    decs = [q.BlockDecoder(lay, G, 30) for _ in range(2)]
    for d in decs:
        _lib.call("qc_channel", 0, 0, 0, 0, N, G, sigma, d.mu.data_ptr(), None, None, 0)
        d.run()
        d.run()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    def serial():
        for _ in range(K):
            decs[0].run()
            decs[1].run()

    def parallel():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            for _ in range(K):
                decs[0].run()
        with torch.cuda.stream(s2):
            for _ in range(K):
                decs[1].run()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    ts, tp = timed(serial), timed(parallel)
    mb = lambda t: round(2 * K * G * Kb / (t / 1e3) / 1e6, 1)
    print(json.dumps({"gamma_per_chain": G, "serial_ms": round(ts, 3), "parallel_ms": round(tp, 3),
                      "serial_mbit_s": mb(ts), "parallel_mbit_s": mb(tp)}))


if __name__ == "__main__":
    main()
