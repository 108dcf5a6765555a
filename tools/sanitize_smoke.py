#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): channel, fused compact decode, early-stop decodes
(plain and with lane compaction), host pipeline with ragged chunks, LDPCCC
slots (public API and look-ahead campaign slots), recycling campaign.

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import paper_1204_0334_b200 as q
    from paper_1204_0334_b200 import bp as qbp
    qbp.HOST_CHUNK = 256
    exp = q.multiplicative_shifts(4, 24, 31)            # (4, 24) grid: fused compact kernels
    lay = q.build_edge_layout(q.expand_qc(exp))
    cfg = q.ChannelConfig(2.5, 5 / 6, seed=3, gamma=700)
    y = q.simulate_block(cfg, lay.n_vars)                 # on-device channel
    r = q.decode_batch(lay, y, cfg.sigma, 6)              # host pipeline: 64,128,256,124,128,64 (pageable: host LLRs)
    q.decode_batch(lay, q.host_array(y), cfg.sigma, 6)    # page-locked input: device LLR conversion
    r2 = q.decode_batch(lay, y[:100], cfg.sigma, 6, early_stop=True)
    assert r.hard_bits.shape == y.shape and r2.iterations_run.max() <= 6
    toy = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))
    q.decode_batch(toy, np.random.default_rng(1).normal(1, 0.8, (70, toy.n_vars)), 0.8, 5)
    # small batches: several rows per warp (block passes 2 / 4 lanes per thread)
    for G, es in ((32, False), (64, False), (32, True)):
        q.decode_batch(lay, y[:G], cfg.sigma, 5, early_stop=es)
    d96 = q.BlockDecoder(lay, 96, 5, early_stop=False, graph=False)
    d96.load_lane_major(y[:96], cfg.sigma)
    d96.run()
    d96.result(96)
    code = q.unwrap_qc(q.multiplicative_shifts(4, 24, 11))
    dec = q.StreamDecoder(code, 2, gamma=3)
    for t in range(12):
        dec.push_frame(np.random.default_rng(t).normal(1, 0.8, (3, code.c)), 0.8)
    dec.flush()
    sim = q.SimulationConfig("t", [2.8], iterations=8, gamma=32, stop_block_errors=10**9, max_frames=256,
                             seed=1, early_stop=True)
    q.run_block_simulation(lay, sim, gamma_kernel=128, recycle=True)
    # round 2: early stop with lane compaction (device engine and host pipeline),
    # LDPCCC look-ahead slots with batched channel frames
    ycmp = q.simulate_block(q.ChannelConfig(3.0, 5 / 6, seed=5, gamma=2048), lay.n_vars)
    r3 = q.decode_batch(lay, ycmp, q.ebn0_to_sigma(3.0, 5 / 6), 24, early_stop=True)   # 1024-lane chunks
    dec_es = q.BlockDecoder(lay, 1024, 30, early_stop=True, graph=False)
    assert dec_es.es_scratch is not None
    dec_es.load_lane_major(ycmp[:1024], q.ebn0_to_sigma(3.0, 5 / 6))
    dec_es.run()
    dec_es.result(1024)
    assert r3.iterations_run.min() < r3.iterations_run.max()
    scode = q.unwrap_qc(q.multiplicative_shifts(4, 24, 11))
    scfg = q.SimulationConfig("s", [2.6], iterations=3, gamma=32, stop_block_errors=10**9, max_frames=128,
                              seed=2, processors=3, stream_segment_frames=12)
    q.run_stream_simulation(scode, scfg)
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
