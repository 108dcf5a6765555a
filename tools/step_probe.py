#!/usr/bin/env python
"""Split of the bench step (BlockCampaign, n18360, 30 it): whole step vs the
decode loop alone vs the channel alone, CUDA events over K graph replays.

  python tools/step_probe.py [--gamma 1024] [--k 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gamma", type=int, default=1024)
    ap.add_argument("--k", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import _lib
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    N, M = lay.n_vars, lay.n_checks
    sigma = q.ebn0_to_sigma(3.2, 1 - M / N)
    eng = q.BlockCampaign(lay, 32, args.gamma // 32, 30, False, seed=0)
    for s in range(3):
        eng.step(s * args.gamma, sigma)
    torch.cuda.synchronize()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.k):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        return round(a.elapsed_time(b) / args.k, 4)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            fn()
        return g

    g_dec = capture(eng.dec._launch)
    g_ch = capture(lambda: _lib.call("qc_channel_dev", eng.k0, eng.k1, eng.lane0.data_ptr(), 0, N, eng.gk,
                                     float(sigma), eng.dec.mu.data_ptr(), _lib.stream_handle()))
    out = {"gamma": args.gamma,
           "step_ms": timed(lambda i=0: eng.step((10 + i) * args.gamma, sigma)),
           "step_graph_only_ms": timed(lambda i=0: eng._graph.replay()),
           "decode_graph_ms": timed(lambda i=0: g_dec.replay()),
           "channel_graph_ms": timed(lambda i=0: g_ch.replay()),
           "decode_eager_ms": timed(lambda i=0: eng.dec._launch()),
           "decode_launches": eng.dec.kernel_launches_per_run(),
           "pdl": os.environ.get("QCB_PDL", "1")}
    # same decoder, LLRs from the stand-alone channel entry point (as tools/kbench.py)
    _lib.call("qc_channel", 0, 0, 0, 0, N, eng.gk, sigma, eng.dec.mu.data_ptr(), None, None, 0)
    out["decode_eager_kbench_llrs_ms"] = timed(lambda i=0: eng.dec._launch())
    out["decode_graph_kbench_llrs_ms"] = timed(lambda i=0: g_dec.replay())
    mu = eng.dec.mu
    out["mu_abs_mean"] = round(float(mu.abs().mean()), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
