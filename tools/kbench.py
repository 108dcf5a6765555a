#!/usr/bin/env python
"""Kernel micro-benchmark: per-pass CUDA-event times of the decode-loop kernels
(check pass in phi form, variable pass in phi form) and whole-decode time, for
a list of gamma values.  One JSON line per gamma.  QCB_AGG=0 times the
two-pass reference schedule instead of the compact one.

  python tools/kbench.py --gammas 256 1024 2048 --reps 20
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gammas", type=int, nargs="+", default=[1024])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--code", default="n18360")
    ap.add_argument("--early-stop", action="store_true", help="time the early-stop decode (per-lane freeze)")
    ap.add_argument("--ebn0", type=float, default=3.2)
    ap.add_argument("--graph", action="store_true", help="time the decode as a CUDA-graph replay")
    ap.add_argument("--decode-only", action="store_true", help="skip the per-pass timings")
    args = ap.parse_args()
    import torch
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import _lib
    h, exp = q.load_code(q.codes.bundled_code_path(args.code))
    lay = q.build_edge_layout(h)
    N, E = lay.n_vars, lay.edge_count
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    for G in args.gammas:
        dec = q.BlockDecoder(lay, G, 30, early_stop=args.early_stop, graph=args.graph)
        sigma = q.ebn0_to_sigma(args.ebn0, 1 - lay.n_checks / N)
        _lib.call("qc_channel", 0, 0, 0, 0, N, G, sigma, dec.mu.data_ptr(), None, None, 0)
        st = _lib.stream_handle()
        p = dec.plan.handle

        def timeit(fn, reps=args.reps):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        # realistic message contents: run one decode first
        dec.run()
        if args.decode_only:
            dec_ms = timeit(dec.run, max(3, args.reps // 4))
            print(json.dumps({"gamma": G, "graph": args.graph, "early_stop": args.early_stop, "ebn0_db": args.ebn0,
                              "decode_ms": round(dec_ms, 4),
                              "mbit_s": round(G * (N - lay.n_checks) / dec_ms / 1e3, 1),
                              "mean_iterations": round(float(dec.iters[:G].float().mean().item()), 2)}), flush=True)
            del dec
            torch.cuda.empty_cache()
            continue
        cnu_phi = timeit(lambda: _lib.call("qc_cnu_ex", p, G, 2, dec.msgs.data_ptr(), dec.mu.data_ptr(), None, st))
        cnu_mu = timeit(lambda: _lib.call("qc_cnu_ex", p, G, 1, dec.msgs.data_ptr(), dec.mu.data_ptr(), None, st))
        vnu_phi = timeit(lambda: _lib.call("qc_vnu_ex", p, G, 1, dec.msgs.data_ptr(), dec.mu.data_ptr(), None,
                                           None, None, st))
        agg_ms = {}
        W = G // 32
        agg_ptr = dec.work.data_ptr() + int(_lib.load().qc_decode_records_offset(G)) * 4
        if os.environ.get("QCB_AGG", "1") != "0" and lay.check_regular:
            agg_ms["agg_check_ms"] = timeit(lambda: _lib.call("qc_agg_check", p, G, 0, dec.msgs.data_ptr(),
                                                              dec.mu.data_ptr(), agg_ptr, st))
            agg_ms["agg_var_ms"] = timeit(lambda: _lib.call("qc_agg_var", p, G, 0, dec.msgs.data_ptr(),
                                                            dec.mu.data_ptr(), agg_ptr, None, None, st))
            if G % 256 == 0:
                H = G // 2
                agg_ms["agg_fused_half_ms"] = timeit(lambda: _lib.call(
                    "qc_agg_fused", p, G, H, 0, 0, H, 0, dec.msgs.data_ptr(), dec.mu.data_ptr(), agg_ptr,
                    None, None, st))
            M = lay.n_checks
            agg_ms["agg_check_gbs"] = (E + 2 * M) * G * 4 / agg_ms["agg_check_ms"] / 1e6
            agg_ms["agg_var_gbs"] = (2 * E + N + M) * G * 4 / agg_ms["agg_var_ms"] / 1e6
        dec_ms = timeit(dec.run, max(3, args.reps // 4))
        mean_it = float(dec.iters[:G].float().mean().item())
        cb, vb = 2 * E * G * 4, (2 * E + N) * G * 4
        alg = 4 * (30 * (4 * E + N) + (N + E)) * G
        print(json.dumps({
            "gamma": G,
            "cnu_phi_ms": round(cnu_phi, 4), "cnu_phi_gbs": round(cb / cnu_phi / 1e6, 1),
            "cnu_from_mu_ms": round(cnu_mu, 4),
            "vnu_phi_ms": round(vnu_phi, 4), "vnu_phi_gbs": round(vb / vnu_phi / 1e6, 1),
            "decode_ms": round(dec_ms, 3), "decode_alg_gbs": round(alg / dec_ms / 1e6, 1),
            "decode_frac": round(alg / dec_ms / 1e6 / peak, 4),
            "mbit_s": round(G * (N - lay.n_checks) / dec_ms / 1e3, 1),
            **{k: round(v, 4) for k, v in agg_ms.items()},
            "agg_env": os.environ.get("QCB_AGG", "1"),
            "early_stop": args.early_stop, "ebn0_db": args.ebn0, "mean_iterations": round(mean_it, 2)}), flush=True)
        del dec
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
