#!/usr/bin/env python
"""Does PCIe DMA traffic slow the decode kernels?  Times K graph-replayed
decodes of one chunk (device-resident) alone, then while a side stream keeps
H2D and D2H copies of chunk-sized page-locked buffers running (what the host
pipeline does between decodes).

  python tools/dma_interference.py [--gamma 512]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gamma", type=int, default=512)
    ap.add_argument("--k", type=int, default=8)
    args = ap.parse_args()
    import torch
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import _lib
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    N, K = lay.n_vars, lay.n_vars - lay.n_checks
    G = args.gamma
    dec = q.BlockDecoder(lay, G, 30)
    _lib.call("qc_channel", 0, 0, 0, 0, N, G, q.ebn0_to_sigma(3.2, K / N), dec.mu.data_ptr(), None, None, 0)
    dec.run()
    torch.cuda.synchronize()
    nb = G * N * 8
    h_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(with_dma):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if with_dma:
            with torch.cuda.stream(s_in):
                for _ in range(3 * args.k):
                    d_in.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(s_out):
                for _ in range(3 * args.k):
                    h_out.copy_(d_out, non_blocking=True)
        a.record()
        for _ in range(args.k):
            dec.run()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.k

    timed(False)
    alone = [timed(False) for _ in range(3)]
    dma = [timed(True) for _ in range(3)]
    print(json.dumps({"gamma": G, "decode_ms_alone": [round(x, 4) for x in alone],
                      "decode_ms_with_dma": [round(x, 4) for x in dma],
                      "dma_bytes_each_way_per_copy": nb}))


if __name__ == "__main__":
    main()
