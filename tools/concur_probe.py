#!/usr/bin/env python
"""Does a memory-only check pass (compact records) overlap a compute-heavy
variable pass when the two run on different lane halves on two streams?
Times agg_check(B) and agg_var(A) alone, back to back, and concurrently."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import _lib
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    N, M, E = lay.n_vars, lay.n_checks, lay.edge_count
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    p = lay.plan().handle
    halves = []
    for _ in range(2):
        mu = torch.empty((N, G), dtype=torch.float32, device="cuda")
        _lib.call("qc_channel", 1, 0, 0, 0, N, G, 0.55, mu.data_ptr(), None, None, 0)
        msgs = torch.zeros((E, G), dtype=torch.float32, device="cuda")
        agg = torch.zeros((M, 3, G), dtype=torch.float32, device="cuda")
        _lib.call("qc_agg_check", p, G, 1, msgs.data_ptr(), mu.data_ptr(), agg.data_ptr(), 0)
        _lib.call("qc_agg_var", p, G, 1, msgs.data_ptr(), mu.data_ptr(), agg.data_ptr(), None, None, 0)
        halves.append((mu, msgs, agg))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def chk(hh, st):
        mu, msgs, agg = hh
        _lib.call("qc_agg_check", p, G, 0, msgs.data_ptr(), mu.data_ptr(), agg.data_ptr(), st.cuda_stream)

    def var(hh, st):
        mu, msgs, agg = hh
        _lib.call("qc_agg_var", p, G, 0, msgs.data_ptr(), mu.data_ptr(), agg.data_ptr(), None, None,
                  st.cuda_stream)

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for _ in range(reps):
            fn()
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        b.record(cur)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    out = {"gamma_per_half": G}
    out["check_ms"] = timeit(lambda: chk(halves[1], s1))
    out["var_ms"] = timeit(lambda: var(halves[0], s1))
    out["serial_pair_ms"] = timeit(lambda: (chk(halves[1], s1), var(halves[0], s1)))

    def conc():
        chk(halves[1], s1)
        var(halves[0], s2)
        s1.wait_stream(s2)
        s2.wait_stream(s1)
    out["concurrent_pair_ms"] = timeit(conc)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
