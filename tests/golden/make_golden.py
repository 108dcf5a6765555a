"""Generate golden fixtures from the REAL reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Needs /root/reference (read-only, not present on GPU boxes); the outputs are
committed so the GPU-side tests never touch the reference.  Every array here
is produced by calling the reference's public API (`qcldpc.*`), so the
fixtures pin both the oracle (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py).
"""

import json
import os
import sys

import numpy as np

import qcldpc
from qcldpc import channel as rch

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrs.items()})


def packbits_lane_major(bits):
    return np.packbits(np.asarray(bits, np.uint8), axis=1)


def main():
    # ---------------- codes
    _, exp_a = qcldpc.load_code(os.path.join(os.path.dirname(qcldpc.__file__), "data", "code_a.qc"))
    _, exp_n = qcldpc.load_code(os.path.join(REPO, "paper_1204_0334_b200", "data", "n18360.qc"))
    save("codes.npz", code_a_shifts=exp_a.shifts, code_a_p=np.int64(exp_a.p),
         n18360_shifts=exp_n.shifts, n18360_p=np.int64(exp_n.p))

    # ---------------- channel: raw words via numpy Philox as the reference keys it,
    # and reference lane_normals / simulate_block outputs
    cases = [(0, 0, 0, 64), (7, 3, 50, 100), (123, 2**32 + 5, 13, 77), (2**40 + 9, 31, 4096, 40)]
    ch = {}
    for i, (seed, lane, start, count) in enumerate(cases):
        ch[f"normals_{i}"] = rch.lane_normals(seed, lane, start, count)
        first, off = divmod(start, 4)
        bg = np.random.Philox(key=seed, counter=(lane << 64) + first)
        ch[f"words_{i}"] = np.random.Generator(bg).integers(0, 2**64, dtype=np.uint64,
                                                             size=off + count)[off:]
    cfg = rch.ChannelConfig(3.2, 5 / 6, seed=11, gamma=5)
    ch["block_y"] = rch.simulate_block(cfg, 300, lane_offset=(1 << 32) + 64, start=20)
    ch["block_sigma"] = np.float64(cfg.sigma)
    save("channel.npz", **ch)
    with open(os.path.join(HERE, "channel_cases.json"), "w") as fh:
        json.dump(cases, fh)

    # ---------------- toy block code (demo shape: multiplicative_shifts(2,4,8), 3.0 dB, seed 7)
    exp = qcldpc.multiplicative_shifts(2, 4, 8)
    lay = qcldpc.build_edge_layout(qcldpc.expand_qc(exp))
    st = qcldpc.code_stats(qcldpc.expand_qc(exp))
    cfg = rch.ChannelConfig(3.0, st.rate_bound, seed=7, gamma=32)
    y = rch.simulate_block(cfg, lay.n_vars)
    mu = qcldpc.channel_llrs(y, cfg.sigma)
    batch = qcldpc.MessageBatch(lay, np.ascontiguousarray(mu.T))
    qcldpc.check_node_update(batch, lay)
    cnu1 = batch.packages.copy()
    post1 = qcldpc.variable_node_update(batch, lay)
    vnu1 = batch.packages.copy()
    r30 = qcldpc.decode_batch(lay, y, cfg.sigma, 30)
    res = qcldpc.decode_batch(lay, y, cfg.sigma, 30, early_stop=True)
    save("block_toy.npz", y=y, sigma=np.float64(cfg.sigma), cnu1=cnu1, vnu1=vnu1, post1=post1,
         bits30=r30.hard_bits, post30=r30.posteriors, ok30=r30.syndrome_ok,
         bits_es=res.hard_bits, post_es=res.posteriors, ok_es=res.syndrome_ok,
         iters_es=res.iterations_run)

    # ---------------- code A, gamma=32, lanes 0..31 of point 0, 3.2 dB, 30 iterations
    for name, e in (("code_a", exp_a), ("n18360", exp_n)):
        lay = qcldpc.build_edge_layout(qcldpc.expand_qc(e))
        rate = 1.0 - lay.n_checks / lay.n_vars
        sigma = rch.ebn0_to_sigma(3.2 if name == "code_a" else 3.0, rate)
        G = 32
        y = np.stack([1.0 + sigma * rch.lane_normals(0, g, 0, lay.n_vars) for g in range(G)])
        mu = qcldpc.channel_llrs(y, sigma)
        batch = qcldpc.MessageBatch(lay, np.ascontiguousarray(mu.T))
        qcldpc.check_node_update(batch, lay)
        cnu1 = batch.packages[:6144, :4].astype(np.float32)
        r = qcldpc.decode_batch(lay, y, sigma, 30)
        save(f"block_{name}.npz", sigma=np.float64(sigma), bits=packbits_lane_major(r.hard_bits),
             ok=r.syndrome_ok, post8=r.posteriors[:8].astype(np.float32), cnu1_lanes0_3=cnu1,
             bit_errors=r.hard_bits.sum(axis=1), n=np.int64(lay.n_vars))

    # ---------------- stream decoder: small array code, I=2 and I=3, gamma=3
    code = qcldpc.unwrap_qc(qcldpc.multiplicative_shifts(4, 24, 8))
    rng = np.random.default_rng(4242)
    out = {}
    for I, K in ((2, 20), (3, 30)):
        sigma = 0.85
        ys = rng.normal(1.0, sigma, size=(K, 3, code.c))
        dec = qcldpc.StreamDecoder(code, I, gamma=3)
        frames = [f for f in (dec.push_frame(y, sigma) for y in ys) if f is not None]
        frames += dec.flush()
        out[f"I{I}_ys"] = ys
        out[f"I{I}_sigma"] = np.float64(sigma)
        out[f"I{I}_index"] = np.array([f.frame_index for f in frames])
        out[f"I{I}_tail"] = np.array([f.tail for f in frames])
        out[f"I{I}_bits"] = np.stack([f.hard_bits for f in frames])
        out[f"I{I}_post"] = np.stack([f.posteriors for f in frames])
    save("stream_small.npz", **out)

    # ---------------- stream on code A' (I=4, gamma=2, 3.1 dB, harness addressing)
    code = qcldpc.unwrap_qc(exp_a)
    sigma = rch.ebn0_to_sigma(3.1, code.rate_bound)
    I, K, G = 4, 40, 2
    dec = qcldpc.StreamDecoder(code, I, gamma=G)
    frames = []
    for t in range(K):
        y = np.stack([1.0 + sigma * rch.lane_normals(0, g, t * code.c, code.c) for g in range(G)])
        f = dec.push_frame(y, sigma)
        if f is not None:
            frames.append(f)
    frames += dec.flush()
    save("stream_code_a.npz", sigma=np.float64(sigma), I=np.int64(I), K=np.int64(K),
         index=np.array([f.frame_index for f in frames]), tail=np.array([f.tail for f in frames]),
         bits=np.stack([packbits_lane_major(f.hard_bits) for f in frames]),
         post0=np.stack([f.posteriors[0].astype(np.float32) for f in frames]))

    # ---------------- campaigns (small, reference harness) + recorded large ones
    from qcldpc.harness import SimulationConfig, run_block_simulation, run_stream_simulation
    toy_lay = qcldpc.build_edge_layout(qcldpc.expand_qc(qcldpc.multiplicative_shifts(2, 4, 8)))
    toy_code = qcldpc.unwrap_qc(qcldpc.multiplicative_shifts(2, 4, 8))
    camp = {}
    cfg = SimulationConfig(code_id="toy", ebn0_db=[2.0, 3.0], iterations=8, processors=2, gamma=8,
                           stop_block_errors=15, max_frames=2000, seed=5)
    camp["toy_block"] = [r.row()[:10] for r in run_block_simulation(toy_lay, cfg)]
    cfg2 = SimulationConfig(code_id="toy", ebn0_db=[2.0], iterations=8, processors=2, gamma=8,
                            stop_block_errors=10, max_frames=500, seed=5, stream_segment_frames=6)
    camp["toy_stream"] = [r.row()[:10] for r in run_stream_simulation(toy_code, cfg2)]
    cfg3 = SimulationConfig(code_id="code-a", ebn0_db=[3.2], iterations=30, gamma=32,
                            stop_block_errors=2**62, max_frames=256, seed=0)
    camp["code_a_block_256"] = [r.row()[:10] for r in run_block_simulation(
        qcldpc.build_edge_layout(qcldpc.expand_qc(exp_a)), cfg3)]
    # recorded by the reference run, pkg/test_output.txt:27,30 (seed 0, gamma 32)
    camp["recorded"] = {
        "code_a_block_3.2dB_30it_stop300": {"frames": 10912, "bit_errors": 45450, "frame_errors": 300},
        "code_a_stream_3.1dB_I20_stop300": {"frames": 15168, "bit_errors": 4627, "frame_errors": 435},
    }
    with open(os.path.join(HERE, "campaigns.json"), "w") as fh:
        json.dump(camp, fh, indent=1)
    print(json.dumps(camp, indent=1))


if __name__ == "__main__":
    sys.exit(main())
