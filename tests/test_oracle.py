"""CPU: the oracle against golden vectors produced by the real reference.

Fixtures come from tests/golden/make_golden.py (run against /root/reference);
known-answer values are restated from the reference's own tests.
"""
import json
import os

import numpy as np
import pytest
from conftest import GOLDEN, golden

from oracle import bp, campaign, channel, qc, stream

# test_bp.py:15-22 (mpmath-frozen)
ALPHA_EXCLUSIVE = [-0.22733629380264572863, +0.37747645630979721384, -0.73532566405551922471]
ALPHA_DEGREE1 = 28.324190418452803892
# test_channel.py:10-13
SIGMA_R56 = {3.2: 0.53588996575190975146, 3.1: 0.5420952790986725772}
# test_convolutional.py:12-13
LUT_C_LAM4 = [[1, 2, 3, 0], [6, 7, 4, 5], [11, 8, 9, 10], [12, 13, 14, 15]]
LUT_V_LAM4 = [[0, 4, 8, 12], [5, 9, 13, 1], [10, 14, 2, 6], [15, 3, 7, 11]]


def _single(n):
    return qc.layout_from_rows(n, [list(range(n))])


def test_kat_check_update():
    lay = _single(3)
    buf = bp.init_buffer(lay, np.array([[2.0], [-1.0], [0.5]]))
    bp.check_update(buf, lay)
    assert np.allclose(buf[:3, 0], ALPHA_EXCLUSIVE, atol=1e-12, rtol=0)
    lay1 = _single(1)
    b1 = bp.init_buffer(lay1, np.array([[3.0]]))
    bp.check_update(b1, lay1)
    assert abs(b1[0, 0] - ALPHA_DEGREE1) < 1e-12


def test_kat_sigma():
    for db, s in SIGMA_R56.items():
        assert abs(channel.ebn0_to_sigma(db, 5 / 6) - s) < 1e-15


def test_philox_restatement_matches_numpy_words():
    cases = json.load(open(os.path.join(GOLDEN, "channel_cases.json")))
    g = golden("channel.npz")
    for i, (seed, lane, start, count) in enumerate(cases):
        want = g[f"words_{i}"]
        assert np.array_equal(channel.lane_words(seed, lane, start, count), want)
        k = min(count, 9)
        assert channel.lane_words_slow(seed, lane, start, k) == [int(x) for x in want[:k]]


def test_lane_normals_match_reference():
    cases = json.load(open(os.path.join(GOLDEN, "channel_cases.json")))
    g = golden("channel.npz")
    for i, (seed, lane, start, count) in enumerate(cases):
        assert np.array_equal(channel.lane_normals(seed, lane, start, count), g[f"normals_{i}"])
    y = channel.received(11, float(g["block_sigma"]), (1 << 32) + 64, 5, 300, start=20)
    assert np.array_equal(y, g["block_y"])


def test_ndtri_restatement_bit_exact():
    from scipy.special import ndtri
    rng = np.random.default_rng(3)
    w = rng.integers(0, 2**64, size=20000, dtype=np.uint64)
    u = channel.words_to_uniform(w)
    u = np.concatenate([u, [2.0**-54, 0.5, channel._EXPM2, 1 - channel._EXPM2, 1e-300]])
    mine = np.array([channel.ndtri_cephes(float(x)) for x in u])
    assert np.array_equal(mine, ndtri(u))


def test_toy_block_golden():
    g = golden("block_toy.npz")
    lay = qc.qc_layout(qc.array_code_shifts(2, 4, 8), 8)
    sigma = float(g["sigma"])
    mu = bp.channel_llrs(g["y"], sigma)
    buf = bp.init_buffer(lay, np.ascontiguousarray(mu.T))
    bp.check_update(buf, lay)
    assert np.array_equal(buf[:-1], g["cnu1"])
    post = bp.var_update(buf, np.ascontiguousarray(mu.T), lay)
    assert np.array_equal(buf[:-1], g["vnu1"]) and np.array_equal(post, g["post1"])
    bits, post, ok, its = bp.decode_llr(lay, mu, 30)
    assert np.array_equal(bits, g["bits30"]) and np.array_equal(post, g["post30"])
    assert np.array_equal(ok, g["ok30"])
    bits, post, ok, its = bp.decode_llr(lay, mu, 30, early_stop=True)
    assert np.array_equal(post, g["post_es"]) and np.array_equal(its, g["iters_es"])
    assert np.array_equal(ok, g["ok_es"]) and np.array_equal(bits, g["bits_es"])


def test_code_a_block_golden(codes_npz):
    g = golden("block_code_a.npz")
    lay = qc.qc_layout(codes_npz["code_a_shifts"], int(codes_npz["code_a_p"]))
    sigma = float(g["sigma"])
    y = channel.received(0, sigma, 0, 32, lay.n_vars)
    bits, post, ok, _ = bp.decode_llr(lay, bp.channel_llrs(y, sigma), 30)
    assert np.array_equal(np.packbits(bits, axis=1), g["bits"])
    assert np.array_equal(ok, g["ok"])
    assert np.array_equal(post[:8].astype(np.float32), g["post8"])


def test_stream_small_golden():
    g = golden("stream_small.npz")
    U = qc.unwrap(qc.array_code_shifts(4, 24, 8), 8)
    assert U.lut_c.tolist() == LUT_C_LAM4 and U.lut_v.tolist() == LUT_V_LAM4
    for I in (2, 3):
        dec = stream.StreamOracle(U, I, 3)
        sig = float(g[f"I{I}_sigma"])
        out = [f for f in (dec.push(y, sig) for y in g[f"I{I}_ys"]) if f is not None]
        out += dec.flush()
        assert [f.frame_index for f in out] == g[f"I{I}_index"].tolist()
        assert [f.tail for f in out] == g[f"I{I}_tail"].tolist()
        assert np.array_equal(np.stack([f.hard_bits for f in out]), g[f"I{I}_bits"])
        assert np.array_equal(np.stack([f.posteriors for f in out]), g[f"I{I}_post"])


def test_unwrapped_code_a_constants(codes_npz):
    U = qc.unwrap(codes_npz["code_a_shifts"], int(codes_npz["code_a_p"]))
    assert (U.lam, U.ms, U.c, U.cb, U.edge_count) == (4, 3, 2532, 422, 40512)


def test_toy_campaign_counts():
    camp = json.load(open(os.path.join(GOLDEN, "campaigns.json")))
    lay = qc.qc_layout(qc.array_code_shifts(2, 4, 8), 8)
    for pi, db in enumerate([2.0, 3.0]):
        fr, be, fe = campaign.block_point(lay, db, pi, iters=8, gamma=8, seed=5, stop=15,
                                          max_frames=2000)
        row = camp["toy_block"][pi]
        assert (fr, be, fe) == (row[5], row[6], row[7])
    U = qc.unwrap(qc.array_code_shifts(2, 4, 8), 8)
    fr, be, fe = campaign.stream_point(U, 2.0, 0, processors=2, gamma=8, seed=5, stop=10,
                                       max_frames=500, segment_frames=6)
    row = camp["toy_stream"][0]
    assert (fr, be, fe) == (row[5], row[6], row[7])


def test_campaign_worker_invariance():
    lay = qc.qc_layout(qc.array_code_shifts(2, 4, 8), 8)
    a = campaign.block_point(lay, 2.0, 0, iters=8, gamma=8, seed=5, stop=15, max_frames=2000)
    b = campaign.block_point(lay, 2.0, 0, iters=8, gamma=8, seed=5, stop=15, max_frames=2000,
                             workers=2)
    assert a == b


def test_reference_oracles_restatement_matches_reference():
    """oracle/reference.py (exact_posterior_llr, reference_window_decoder) equals the
    reference's own qcldpc.reference (reference.py:25-182) bit for bit."""
    import pytest
    from oracle import build_ref
    if not build_ref.available():
        pytest.skip("oracle/_ref not built")
    import importlib
    import sys
    sys.path.insert(0, build_ref.site_dir())
    try:
        ref = importlib.import_module("qcldpc.reference")
        qcl = importlib.import_module("qcldpc")
    finally:
        sys.path.remove(build_ref.site_dir())
    from oracle import reference as ours
    rng = np.random.default_rng(3)
    h = qcl.SparseParityCheck(8, [[0, 1, 2], [2, 3, 4], [4, 5, 6, 7], [0, 7], [1, 5]])
    for _ in range(4):
        mu = rng.normal(0, 1.5, 8)
        np.testing.assert_allclose(ours.exact_posterior_llr(h, mu), ref.exact_posterior_llr(h, mu),
                                   rtol=0, atol=1e-12)
    code = qcl.unwrap_qc(qcl.multiplicative_shifts(4, 24, 8))
    llrs = [qcl.channel_llrs(rng.normal(1, 0.8, (1, code.c)), 0.8)[0] for _ in range(14)]
    b0, p0 = ref.reference_window_decoder(code, 2, llrs)
    b1, p1 = ours.reference_window_decoder(code, 2, llrs)
    assert all(np.array_equal(x, y) for x, y in zip(b0, b1))
    assert all(np.array_equal(x, y) for x, y in zip(p0, p1))
