"""GPU campaigns: counts identical to the reference harness (goldens)."""
import dataclasses
import io
import json
import os

import numpy as np
import pytest
from conftest import GOLDEN

from oracle import channel as och

pytestmark = pytest.mark.gpu
CAMP = json.load(open(os.path.join(GOLDEN, "campaigns.json")))


def toy_cfg(q, **kw):
    base = dict(code_id="toy", ebn0_db=[2.0, 3.0], iterations=8, processors=2, gamma=8,
                stop_block_errors=15, max_frames=2000, seed=5)
    base.update(kw)
    return q.SimulationConfig(**base)


def test_toy_block_campaign(gpu):
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))
    res = q.run_block_simulation(lay, toy_cfg(q))
    assert [r.row()[:10] for r in res] == CAMP["toy_block"]
    for gk in (32, 256):
        res = q.run_block_simulation(lay, toy_cfg(q), gamma_kernel=gk)
        assert [r.row()[:10] for r in res] == CAMP["toy_block"]
    buf = io.StringIO()
    q.write_csv(res, buf)
    assert buf.getvalue().splitlines()[0].split(",") == q.CSV_COLUMNS
    r = q.run_block_simulation(lay, toy_cfg(q, stop_block_errors=10**9, max_frames=24))[0]
    assert r.frames == 24


def test_toy_stream_campaign(gpu):
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(2, 4, 8))
    cfg = toy_cfg(q, ebn0_db=[2.0], stop_block_errors=10, max_frames=500, stream_segment_frames=6)
    res = q.run_stream_simulation(code, cfg)
    assert [r.row()[:10] for r in res] == CAMP["toy_stream"]


def test_code_a_block_256(gpu, codes_npz):
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(q.ExponentMatrix(codes_npz["code_a_shifts"],
                                                          int(codes_npz["code_a_p"]))))
    cfg = q.SimulationConfig("code-a", [3.2], iterations=30, gamma=32, stop_block_errors=2**62,
                             max_frames=256, seed=0)
    assert [r.row()[:10] for r in q.run_block_simulation(lay, cfg)] == CAMP["code_a_block_256"]


def test_recorded_block_campaign(gpu, codes_npz):
    """pkg/test_output.txt:27 -- 10912 frames / 45450 bit errors / 300 frame errors."""
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(q.ExponentMatrix(codes_npz["code_a_shifts"],
                                                          int(codes_npz["code_a_p"]))))
    cfg = q.SimulationConfig("code-a", [3.2], iterations=30, gamma=32, stop_block_errors=300,
                             max_frames=60_000, seed=0)
    r = q.run_block_simulation(lay, cfg)[0]
    want = CAMP["recorded"]["code_a_block_3.2dB_30it_stop300"]
    assert (r.frames, r.bit_errors, r.frame_errors) == (want["frames"], want["bit_errors"],
                                                        want["frame_errors"])


def test_recorded_stream_campaign(gpu, codes_npz):
    """pkg/test_output.txt:30 -- 15168 frames / 4627 bit errors / 435 frame errors."""
    q = gpu
    code = q.unwrap_qc(q.ExponentMatrix(codes_npz["code_a_shifts"], int(codes_npz["code_a_p"])))
    cfg = q.SimulationConfig("code-a-stream", [3.1], processors=20, gamma=32,
                             stop_block_errors=300, max_frames=60_000, seed=0)
    r = q.run_stream_simulation(code, cfg)[0]
    want = CAMP["recorded"]["code_a_stream_3.1dB_I20_stop300"]
    assert (r.frames, r.bit_errors, r.frame_errors) == (want["frames"], want["bit_errors"],
                                                        want["frame_errors"])


def test_bench_records(gpu):
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))
    recs = q.bench_throughput(lay, toy_cfg(q, ebn0_db=3.0), frames=16)
    assert {r["gamma"] for r in recs} == {1, 8}
    assert all(r["frames"] == 16 and r["mode"] == "block" for r in recs)
    # workers = concurrent reference batches per launch: the same codewords
    # decoded with different batching -- identical per-gamma results
    import multiprocessing
    cores = multiprocessing.cpu_count()
    for g in (1, 8):
        rs = [r for r in recs if r["gamma"] == g]
        assert {r["workers"] for r in rs} == {1, cores}
        one = next(r for r in rs if r["workers"] == 1)
        many = next(r for r in rs if r["workers"] == cores)
        assert one["batches_per_launch"] == 1
        assert many["batches_per_launch"] == min(cores, -(-16 // g))
    buf = io.StringIO()
    q.write_jsonl(recs, buf)
    assert [json.loads(l) for l in buf.getvalue().splitlines()] == recs


def test_stream_campaign_unaligned_frames_vs_oracle(gpu):
    """c = 18 (not a multiple of 4): frame starts t*c split Philox blocks."""
    from oracle import campaign, qc as oqc
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(2, 4, 9))
    assert code.c % 4 == 2
    cfg = q.SimulationConfig("u", [2.5], processors=3, gamma=8, stop_block_errors=12,
                             max_frames=400, seed=3, stream_segment_frames=7)
    r = q.run_stream_simulation(code, cfg)[0]
    U = oqc.unwrap(oqc.array_code_shifts(2, 4, 9), 9)
    want = campaign.stream_point(U, 2.5, 0, processors=3, gamma=8, seed=3, stop=12, max_frames=400,
                                 segment_frames=7)
    assert (r.frames, r.bit_errors, r.frame_errors) == want


def test_block_campaign_odd_n_vs_oracle(gpu):
    from oracle import campaign, qc as oqc
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(3, 7, 11)))
    assert lay.n_vars % 4 == 1
    cfg = q.SimulationConfig("o", [2.0], iterations=10, gamma=16, stop_block_errors=20, max_frames=3000,
                             seed=11)
    r = q.run_block_simulation(lay, cfg)[0]
    want = campaign.block_point(oqc.qc_layout(oqc.array_code_shifts(3, 7, 11), 11), 2.0, 0, iters=10,
                                gamma=16, seed=11, stop=20, max_frames=3000)
    assert (r.frames, r.bit_errors, r.frame_errors) == want


def test_recycled_early_stop_campaign_matches_oracle(gpu, codes_npz):
    """Lane recycling (early_stop campaigns) gives the reference's early-stop counts."""
    from oracle import campaign, qc as oqc
    q = gpu
    sh, p = codes_npz["code_a_shifts"], int(codes_npz["code_a_p"])
    lay = q.build_edge_layout(q.expand_qc(q.ExponentMatrix(sh, p)))
    assert q.RecycleCampaign.supports(lay)
    cfg = q.SimulationConfig("code-a", [3.0], iterations=30, gamma=32, stop_block_errors=4,
                             max_frames=640, seed=3, early_stop=True)
    r = q.run_block_simulation(lay, cfg, gamma_kernel=128)[0]
    want = campaign.block_point(oqc.qc_layout(sh, p), 3.0, 0, iters=30, gamma=32, seed=3, stop=4,
                                max_frames=640, early_stop=True)
    assert (r.frames, r.bit_errors, r.frame_errors) == want
    # the non-recycled early-stop path agrees too
    r2 = q.run_block_simulation(lay, cfg, gamma_kernel=128, recycle=False)[0]
    assert (r2.frames, r2.bit_errors, r2.frame_errors) == want


def test_n18360_failing_frames_match_oracle_f64(gpu):
    """Bit errors inside FAILED frames are the most fragile fp32 quantity (the
    decoder never converges there); on n18360 at 2.9 dB (FER ~0.7) the GPU
    campaign's frame / bit / frame-error counts equal the float64 oracle's
    (profiles/r01/campaign_parity_n18360.jsonl: also 2048 frames at 2.8/3.0/3.2 dB)."""
    q = gpu
    from oracle import campaign, qc
    h, exp = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    cfg = q.SimulationConfig("n18360", [2.9], iterations=30, gamma=32, stop_block_errors=2**62,
                             max_frames=128, seed=0)
    g = q.run_block_simulation(lay, cfg)[0]
    # serial oracle: never fork a process that has initialised CUDA / thread pools
    o = campaign.block_point(qc.qc_layout(exp.shifts, exp.p), 2.9, 0, iters=30, gamma=32, seed=0,
                             stop=2**62, max_frames=128, workers=1)
    assert (g.frames, g.bit_errors, g.frame_errors) == tuple(o)
    assert g.frame_errors > 32


def test_multiple_points_use_disjoint_noise(gpu):
    """test_harness.py:78-84: the same operating point twice draws fresh lanes
    per point (lane base = point index << 32)."""
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))
    res = q.run_block_simulation(lay, toy_cfg(q, ebn0_db=[2.0, 2.0]))
    assert res[0].frames > 0 and res[1].frames > 0
    assert (res[0].bit_errors, res[0].frame_errors) != (res[1].bit_errors, res[1].frame_errors)


def test_stream_counts_match_manual_replay(gpu):
    """test_harness.py:94-116 through this package's own public API: the device
    stream campaign counts exactly the push-emitted frames a StreamDecoder fed
    by lane_normals would count."""
    import numpy as np
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(2, 4, 8))
    cfg = toy_cfg(q, gamma=2, processors=2, stream_segment_frames=5, stop_block_errors=10**9,
                  max_frames=20, seed=9)
    res = q.run_stream_simulation(code, cfg)[0]
    window = 2 * (code.ms + 1)
    pushes = 5 + window - 1
    sigma = q.ebn0_to_sigma(2.0, code.rate_bound)
    frames = bit_errors = frame_errors = 0
    for seg in range(2):                      # max_frames consumes exactly two segments
        dec = q.StreamDecoder(code, 2, gamma=2)
        for t in range(pushes):
            y = np.stack([1.0 + sigma * q.lane_normals(9, seg * 2 + g, t * code.c, code.c) for g in range(2)])
            fr = dec.push_frame(y, sigma)
            if fr is not None:
                frames += 2
                bit_errors += int(fr.hard_bits.sum())
                frame_errors += int(fr.hard_bits.any(axis=1).sum())
    assert (res.frames, res.bit_errors, res.frame_errors) == (frames, bit_errors, frame_errors)
    assert res.iters_or_i == 2


BENCH = json.load(open(os.path.join(GOLDEN, "campaigns_bench.json")))


def _n18360(q, codes_npz):
    return q.ExponentMatrix(codes_npz["n18360_shifts"], int(codes_npz["n18360_p"]))


def test_bench_config_block_campaign(gpu, codes_npz):
    """bench.py's block configuration (n18360, 30 it, gamma_kernel 1024 lanes per
    launch = 32 reference batches) reproduces the reference harness's counts
    (tests/golden/make_golden_bench.py: 1024 frames at 3.0 dB)."""
    q = gpu
    lay = q.build_edge_layout(q.expand_qc(_n18360(q, codes_npz)))
    cfg = q.SimulationConfig("n18360", [3.0], iterations=30, gamma=32, stop_block_errors=2**62,
                             max_frames=1024, seed=0)
    res = q.run_block_simulation(lay, cfg, batches_per_launch=32)        # 1024 lanes per launch
    assert [r.row()[:10] for r in res] == BENCH["n18360_block_3.0dB_30it_1024"]


def test_decode_batch_gamma_1024_replicated_golden(gpu, codes_npz):
    """decode_batch at gamma 1024 (the host pipeline's 512-lane chunks, fused
    compact-schedule kernels) on the 32 golden n18360 lanes replicated 32 times:
    every copy's bits and syndrome flag equal the reference's."""
    q = gpu
    from conftest import golden
    g = golden("block_n18360.npz")
    lay = q.build_edge_layout(q.expand_qc(_n18360(q, codes_npz)))
    sigma = float(g["sigma"])
    y = och.received(0, sigma, 0, 32, lay.n_vars)
    yy = np.ascontiguousarray(np.tile(y, (32, 1)))
    r = q.decode_batch(lay, yy, sigma, 30)
    bits = np.packbits(r.hard_bits, axis=1).reshape(32, 32, -1)
    assert all(np.array_equal(bits[k], g["bits"]) for k in range(32))
    assert np.array_equal(r.syndrome_ok, np.tile(g["ok"], 32))
    assert np.array_equal(r.hard_bits.sum(axis=1), np.tile(g["bit_errors"], 32))


@pytest.mark.slow
def test_bench_config_stream_campaign(gpu, codes_npz):
    """bench.py's LDPCCC configuration (18360' = the n18360 grid unwrapped,
    I = 20, gamma_kernel 512 = 16 reference segments side by side) reproduces the
    reference harness's counts for its first segment (5056 frames at 3.1 dB)."""
    q = gpu
    code = q.unwrap_qc(_n18360(q, codes_npz))
    cfg = q.SimulationConfig("n18360p", [3.1], processors=20, gamma=32, stop_block_errors=2**62,
                             max_frames=5056, seed=0)
    res = q.run_stream_simulation(code, cfg, batches_per_launch=16)      # 512 lanes per launch
    assert [r.row()[:10] for r in res] == BENCH["n18360p_stream_3.1dB_I20_5056"]
