"""GPU parity: block decoder kernels vs the oracle / reference goldens.

Tolerance (north star): single message updates |delta| <= 1e-4 * max(|ref|, 1)
against the float64 reference; decisions, syndromes and error counts bit-exact.
"""
import numpy as np
import pytest
from conftest import golden

from oracle import bp as obp
from oracle import channel as och
from oracle import qc as oqc

pytestmark = pytest.mark.gpu
TOL = 1e-4


def close(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
    assert err.max() <= TOL, f"max scaled error {err.max():.3e}"


def toy(q):
    return q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))


def test_kat_check_update(gpu):
    q = gpu
    lay = q.build_edge_layout(q.SparseParityCheck(3, [[0, 1, 2]]))
    b = q.MessageBatch(lay, np.array([[2.0], [-1.0], [0.5]]))
    q.check_node_update(b, lay)
    close(b.packages[:, 0], [-0.22733629380264572863, 0.37747645630979721384, -0.73532566405551922471])
    lay1 = q.build_edge_layout(q.SparseParityCheck(1, [[0]]))
    b1 = q.MessageBatch(lay1, np.array([[3.0]]))
    q.check_node_update(b1, lay1)
    close(b1.packages[0, 0], 28.324190418452803892)
    lay2 = q.build_edge_layout(q.SparseParityCheck(2, [[0, 1]]))
    b2 = q.MessageBatch(lay2, np.array([[1.25], [-0.75]]))
    q.check_node_update(b2, lay2)
    close(b2.packages[:, 0], [-0.75, 1.25])


def test_single_step_random_degrees(gpu):
    """One CNU + VNU on identical inputs, degrees 1..32, beta spread up to +-50."""
    q = gpu
    rng = np.random.default_rng(1)
    for d in (1, 2, 3, 4, 5, 6, 7, 8, 11, 12, 16, 20, 24, 31, 32):
        n = d + 3
        rows = [sorted(rng.choice(n, size=d, replace=False)) for _ in range(4)]
        lay = q.build_edge_layout(q.SparseParityCheck(n, rows))
        olay = oqc.layout_from_rows(n, rows)
        mu = rng.normal(0, 1, size=(n, 64)) * rng.choice([0.1, 1, 5, 20, 60], size=(n, 1))
        mu = np.clip(mu, -50, 50).astype(np.float32).astype(np.float64)
        mu[0, :3] = 0.0
        b = q.MessageBatch(lay, mu)
        q.check_node_update(b, lay)
        ob = obp.init_buffer(olay, mu)
        obp.check_update(ob, olay)
        close(b.packages, ob[:-1])
        # feed identical alphas into the VNU
        a32 = b.packages.astype(np.float32).astype(np.float64)
        ob[:-1] = a32
        post = q.variable_node_update(b, lay)
        opost = obp.var_update(ob, mu, olay)
        close(post, opost)
        close(b.packages, ob[:-1])


def test_toy_golden(gpu):
    q = gpu
    g = golden("block_toy.npz")
    lay = toy(q)
    mu = q.channel_llrs(g["y"], float(g["sigma"]))
    b = q.MessageBatch(lay, np.ascontiguousarray(mu.T))
    q.check_node_update(b, lay)
    close(b.packages, g["cnu1"])
    r = q.decode_batch(lay, g["y"], float(g["sigma"]), 30)
    assert np.array_equal(r.hard_bits, g["bits30"])
    assert np.array_equal(r.syndrome_ok, g["ok30"])
    close(r.posteriors, g["post30"])
    r = q.decode_batch(lay, g["y"], float(g["sigma"]), 30, early_stop=True)
    assert np.array_equal(r.iterations_run, g["iters_es"])
    assert np.array_equal(r.syndrome_ok, g["ok_es"])
    assert np.array_equal(r.hard_bits, g["bits_es"])
    close(r.posteriors, g["post_es"])


@pytest.mark.parametrize("name", ["code_a", "n18360"])
def test_large_code_golden(gpu, codes_npz, name):
    """Gamma=32 lanes at the operating point: bits, syndromes, bit errors bit-exact."""
    q = gpu
    g = golden(f"block_{name}.npz")
    exp = q.ExponentMatrix(codes_npz[f"{name}_shifts"], int(codes_npz[f"{name}_p"]))
    lay = q.build_edge_layout(q.expand_qc(exp))
    sigma = float(g["sigma"])
    rate = 1.0 - lay.n_checks / lay.n_vars
    db = 3.2 if name == "code_a" else 3.0
    cfg = q.ChannelConfig(db, rate, seed=0, gamma=32)
    assert cfg.sigma == sigma
    y = q.simulate_block(cfg, lay.n_vars)               # on-device channel
    yo = och.received(0, sigma, 0, 32, lay.n_vars)      # oracle channel
    assert np.abs(y - yo).max() < 1e-12
    y = yo
    # single step (lanes 0..3, first edges)
    mu = q.channel_llrs(y, sigma)
    b = q.MessageBatch(lay, np.ascontiguousarray(mu.T))
    q.check_node_update(b, lay)
    close(b.packages[: g["cnu1_lanes0_3"].shape[0], :4], g["cnu1_lanes0_3"])
    r = q.decode_batch(lay, y, sigma, 30)
    assert np.array_equal(np.packbits(r.hard_bits, axis=1), g["bits"])
    assert np.array_equal(r.syndrome_ok, g["ok"])
    assert np.array_equal(r.hard_bits.sum(axis=1), g["bit_errors"])
    conv = g["ok"][:8]
    close(r.posteriors[:8][conv], g["post8"][conv])


def test_wide_batch_matches_single_lane(gpu):
    q = gpu
    lay = toy(q)
    rng = np.random.default_rng(300)
    for _ in range(20):
        y = rng.normal(1.0, 1.0, size=(1, lay.n_vars))
        one = q.decode_batch(lay, y, 1.0, 6)
        wide = q.decode_batch(lay, np.repeat(y, 32, axis=0), 1.0, 6)
        assert np.array_equal(np.repeat(one.posteriors, 32, axis=0), wide.posteriors)
        assert np.array_equal(np.repeat(one.hard_bits, 32, axis=0), wide.hard_bits)
    # also across kernel variants (gamma 32 / 64 / 128 use VEC 1 / 2 / 4)
    y = rng.normal(1.0, 1.0, size=(1, lay.n_vars))
    ref = q.decode_batch(lay, y, 1.0, 9).posteriors
    for G in (64, 128, 256):
        w = q.decode_batch(lay, np.repeat(y, G, axis=0), 1.0, 9).posteriors
        assert np.array_equal(w, np.repeat(ref, G, axis=0))


def test_lane_permutation(gpu):
    q = gpu
    lay = toy(q)
    rng = np.random.default_rng(5)
    y = rng.normal(1.0, 0.9, size=(6, lay.n_vars))
    perm = rng.permutation(6)
    r1 = q.decode_batch(lay, y, 0.9, 8)
    r2 = q.decode_batch(lay, y[perm], 0.9, 8)
    assert np.array_equal(r1.posteriors[perm], r2.posteriors)


def test_irregular_code_against_oracle(gpu):
    q = gpu
    rows = [[0, 1, 2, 3, 5, 7, 9], [0, 2, 3, 6, 7, 8, 9], [1, 3, 7], [0, 4, 6, 7, 8, 9], [2, 3, 4, 6, 8]]
    lay = q.build_edge_layout(q.SparseParityCheck(10, rows))
    olay = oqc.layout_from_rows(10, rows)
    rng = np.random.default_rng(8)
    y = rng.normal(1.0, 0.8, size=(40, 10))
    r = q.decode_batch(lay, y, 0.8, 10)
    bits, post, ok, _ = obp.decode_llr(olay, obp.channel_llrs(y, 0.8), 10)
    assert np.array_equal(r.hard_bits, bits) and np.array_equal(r.syndrome_ok, ok)
    close(r.posteriors, post)
    y1 = np.ones((2, 10)); y1[1, 3] = -0.2
    r = q.decode_batch(lay, y1, 0.6, 10)
    assert not r.hard_bits.any() and r.syndrome_ok.all()


@pytest.mark.parametrize("J,L,p,G", [(3, 6, 31, 128), (3, 12, 29, 96), (2, 8, 37, 64), (4, 16, 23, 256)])
def test_compact_schedule_shapes_against_oracle(gpu, J, L, p, G):
    """Every (d_v, d_c) instantiation of the compact schedule (d_v 2-4, d_c 6-16,
    float / float2 / float4 lanes) decodes a regular QC code like the float64
    oracle: decisions, syndromes and iteration counts bit-exact after 15
    iterations, posteriors within 1e-4 after 3.  (Posterior deviations grow
    with iterations on the (3, 6) array code -- 2.7e-4 after 15, for either phi
    grade -- its short cycles amplify fp32 rounding; the decisions still agree,
    tools/posterior_error_diag.py.)"""
    q = gpu
    exp = q.multiplicative_shifts(J, L, p)
    lay = q.build_edge_layout(q.expand_qc(exp))
    olay = oqc.qc_layout(exp.shifts, p)
    rng = np.random.default_rng(J * 100 + L)
    y = rng.normal(1.0, 0.75, size=(G, lay.n_vars))
    r = q.decode_batch(lay, y, 0.75, 15)
    bits, post, ok, its = obp.decode_llr(olay, obp.channel_llrs(y, 0.75), 15)
    assert np.array_equal(r.hard_bits, bits) and np.array_equal(r.syndrome_ok, ok)
    assert np.array_equal(r.iterations_run, its)
    r3 = q.decode_batch(lay, y, 0.75, 3)
    close(r3.posteriors, obp.decode_llr(olay, obp.channel_llrs(y, 0.75), 3)[1])


def test_early_stop_semantics(gpu):
    q = gpu
    lay = toy(q)
    rng = np.random.default_rng(13)
    y = np.ones((8, lay.n_vars))
    y[4:] = rng.normal(1.0, 1.5, size=(4, lay.n_vars))
    res = q.decode_batch(lay, y, 0.7, 20, early_stop=True)
    assert np.all(res.iterations_run[:4] == 1) and res.syndrome_ok[:4].all()
    r1 = q.decode_batch(lay, y[:4], 0.7, 1)
    assert np.array_equal(res.posteriors[:4], r1.posteriors)
    y = rng.normal(1.0, 2.0, size=(6, lay.n_vars))
    rf = q.decode_batch(lay, y, 2.0, 12)
    rs = q.decode_batch(lay, y, 2.0, 12, early_stop=True)
    hard = ~rs.syndrome_ok
    assert np.all(rs.iterations_run[hard] == 12)
    assert np.array_equal(rs.posteriors[hard], rf.posteriors[hard])
    olay = oqc.qc_layout(oqc.array_code_shifts(2, 4, 8), 8)
    bits, post, ok, its = obp.decode_llr(olay, obp.channel_llrs(y, 2.0), 12, early_stop=True)
    assert np.array_equal(rs.iterations_run, its) and np.array_equal(rs.syndrome_ok, ok)
    assert np.array_equal(rs.hard_bits, bits)


def test_hard_decision_and_syndrome(gpu):
    q = gpu
    lay = q.build_edge_layout(q.SparseParityCheck(3, [[0, 1], [1, 2]]))
    post = np.array([[1.0, 1.0, 1.0], [-1.0, -1.0, 1.0]]).T
    bits, ok = q.hard_decision_and_syndrome(lay, post)
    assert bits[:, 0].tolist() == [0, 0, 0] and ok[0]
    assert bits[:, 1].tolist() == [1, 1, 0] and not ok[1]


def test_decode_errors(gpu):
    q = gpu
    lay = toy(q)
    with pytest.raises(ValueError):
        q.decode_batch(lay, np.ones((2, lay.n_vars + 1)), 0.8, 5)
    with pytest.raises(ValueError):
        q.decode_llr_batch(lay, np.ones((2, lay.n_vars)), 0)
    r1 = q.decode_batch(lay, np.random.default_rng(2).normal(1, .8, (3, lay.n_vars)), 0.8, 6)
    r2 = q.decode_llr_batch(lay, q.channel_llrs(np.random.default_rng(2).normal(1, .8, (3, lay.n_vars)), 0.8), 6)
    assert np.array_equal(r1.posteriors, r2.posteriors)


def test_pipelined_host_api_matches_single_chunk(gpu, monkeypatch):
    """decode_batch above HOST_CHUNK lanes runs chunked over HOST_SLOTS streams
    (ragged last chunk); pinned and pageable host arrays give identical results."""
    q = gpu
    from paper_1204_0334_b200 import bp as qbp
    monkeypatch.setattr(qbp, "HOST_CHUNK", 64)
    lay = toy(q)
    rng = np.random.default_rng(77)
    y = rng.normal(1.0, 1.0, size=(300, lay.n_vars))
    r = q.decode_batch(lay, y, 1.0, 12)
    olay = oqc.qc_layout(oqc.array_code_shifts(2, 4, 8), 8)
    bits, post, ok, its = obp.decode_llr(olay, obp.channel_llrs(y, 1.0), 12)
    assert np.array_equal(r.hard_bits, bits) and np.array_equal(r.syndrome_ok, ok)
    assert np.array_equal(r.iterations_run, its)
    close(r.posteriors, post)
    r2 = q.decode_batch(lay, y[:64], 1.0, 12)
    assert np.array_equal(r2.posteriors, r.posteriors[:64])
    monkeypatch.setattr(qbp, "PINNED_MIN_BYTES", 0)      # page-locked in and out: DMA in place
    r3 = q.decode_batch(lay, q.host_array(y), 1.0, 12)
    for f in ("hard_bits", "posteriors", "syndrome_ok", "iterations_run"):
        assert np.array_equal(getattr(r3, f), getattr(r, f)), f
    r4 = q.decode_batch(lay, y, 1.0, 12, early_stop=True)
    bits, post, ok, its = obp.decode_llr(olay, obp.channel_llrs(y, 1.0), 12, early_stop=True)
    assert np.array_equal(r4.hard_bits, bits) and np.array_equal(r4.iterations_run, its)


def test_pageable_llr_staging_matches_pinned(gpu, monkeypatch):
    """Pageable inputs are converted to fp32 LLRs by the host staging threads,
    page-locked ones by the device kernel: both must give the same bits,
    including clip boundaries, huge values, +-0 and the unscaled
    decode_llr_batch path."""
    q = gpu
    from paper_1204_0334_b200 import bp as qbp
    monkeypatch.setattr(qbp, "HOST_CHUNK", 64)
    monkeypatch.setattr(qbp, "STAGE_PAGEABLE_MAX_BYTES", 0)   # keep the native pageable staging in play
    lay = toy(q)
    rng = np.random.default_rng(9)
    sigma = 0.7
    y = rng.normal(1.0, 1.5, size=(200, lay.n_vars))
    edge = np.array([0.0, -0.0, 1e300, -1e300, 25 * sigma * sigma, -25 * sigma * sigma,
                     np.nextafter(25 * sigma * sigma, 0), 5e-324, -5e-324, 1e-30])
    y[0, :edge.size] = edge
    y[1, :edge.size] = edge[::-1]
    for fn, arg in ((q.decode_batch, sigma), (q.decode_llr_batch, None)):
        args = (arg,) if arg is not None else ()
        monkeypatch.setattr(qbp, "PINNED_MIN_BYTES", 1 << 60)
        r_page = fn(lay, y, *args, 8)
        monkeypatch.setattr(qbp, "PINNED_MIN_BYTES", 0)
        r_pin = fn(lay, q.host_array(y), *args, 8)
        for f in ("hard_bits", "posteriors", "syndrome_ok", "iterations_run"):
            assert np.array_equal(getattr(r_page, f), getattr(r_pin, f)), (fn.__name__, f)


def test_host_pipeline_production_size_matches_device_decoder(gpu):
    """n18360 at 1500 lanes through decode_batch (default chunk 512: ramp 128,
    256, full chunks, remainder, 256, 128 over 4 streams, pageable and
    page-locked input) equals one device BlockDecoder run over all lanes."""
    q = gpu
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    N, M = lay.n_vars, lay.n_checks
    sigma = q.ebn0_to_sigma(2.9, 1 - M / N)          # waterfall: many failing lanes
    y = 1.0 + sigma * np.random.default_rng(11).standard_normal((1500, N))
    dec = q.BlockDecoder(lay, 1500, 30, graph=False, count_bits=False)
    dec.load_lane_major(y, sigma)
    dec.run()
    ref = dec.result(1500)
    assert 0 < int(ref.syndrome_ok.sum()) < 1500
    for x in (y, q.host_array(y)):
        r = q.decode_batch(lay, x, sigma, 30)
        for f in ("hard_bits", "posteriors", "syndrome_ok", "iterations_run"):
            assert np.array_equal(getattr(r, f), getattr(ref, f)), f


_ES_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1204_0334_b200 as q
h, exp = q.load_code(q.codes.bundled_code_path('n18360'))
lay = q.build_edge_layout(h)
G, it = int(sys.argv[3]), int(sys.argv[4])
y = q.simulate_block(q.ChannelConfig(float(sys.argv[2]), 5 / 6, seed=6, gamma=G), lay.n_vars)
r = q.decode_batch(lay, y, q.ebn0_to_sigma(float(sys.argv[2]), 5 / 6), it, early_stop=True)
np.savez(sys.argv[1], post=r.posteriors, bits=r.hard_bits, ok=r.syndrome_ok, its=r.iterations_run)
"""


def test_compact_early_stop_is_bit_identical(gpu, tmp_path):
    """Early-stop decode on the compact schedule (default for regular (4, 24)
    grids at gamma % 256 == 0: syndrome and freeze folded into the fused
    launches) equals the two-pass early-stop decode (QCB_AGG=0) bit for bit:
    posteriors captured at the freeze iteration, hard bits, syndrome flags,
    iteration counts -- where lanes freeze at many different iterations, where
    half the frames fail, and for the 1- and 2-iteration edge cases of the
    launch sequence."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for db, G, it in (("3.2", 512, 30), ("2.9", 512, 30), ("3.6", 256, 1), ("3.6", 256, 2), ("3.4", 768, 7)):
        outs = []
        for env in ({"QCB_AGG": "0"}, {}):
            f = tmp_path / f"es{db}_{G}_{it}_{len(outs)}.npz"
            subprocess.run([sys.executable, "-c", _ES_SNIPPET, str(f), db, str(G), str(it)], cwd=repo,
                           check=True, env={**os.environ, **env})
            outs.append(np.load(f))
        its = outs[0]["its"]
        if it == 30:
            assert its.min() < its.max()                       # lanes froze at different iterations
        for k in ("post", "bits", "ok", "its"):
            assert np.array_equal(outs[0][k], outs[1][k]), (db, G, it, k)


def test_graded_chunk_plans_agree(gpu, monkeypatch):
    """The host pipeline's chunk plans (C/4, C/2, C.., remainder, C/2, C/4 from
    2.5 C lanes up; C/4, C/2, C.., remainder, C/4 below) and its
    per-size graphs give the same DecodeResult for every batch size around the
    plan's break points as one single-chunk decode."""
    q = gpu
    from paper_1204_0334_b200 import bp as qbp
    lay = toy(q)
    rng = np.random.default_rng(5)
    y = rng.normal(1.0, 0.9, size=(700, lay.n_vars))
    monkeypatch.setattr(qbp, "HOST_CHUNK", 1024)
    ref = q.decode_batch(lay, y, 0.9, 9)                  # one chunk
    monkeypatch.setattr(qbp, "HOST_CHUNK", 128)
    for G in (129, 160, 161, 224, 300, 319, 320, 321, 383, 384, 385, 417, 448, 700):
        r = q.decode_batch(lay, y[:G], 0.9, 9)
        for f in ("hard_bits", "posteriors", "syndrome_ok", "iterations_run"):
            assert np.array_equal(getattr(r, f), getattr(ref, f)[:G]), (G, f)


def test_host_pipeline_abi(gpu):
    """qc_host_* through ctypes: argument errors map to ValueError, dims round-trip."""
    import ctypes
    q = gpu
    from paper_1204_0334_b200 import _lib
    lay = toy(q)
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):
        _lib.call("qc_host_create", lay.plan().handle, 48, 2, 5, 0, ctypes.byref(h))
    with pytest.raises(ValueError):
        _lib.call("qc_host_create", lay.plan().handle, 64, 0, 5, 0, ctypes.byref(h))
    dec = q.HostDecoder(lay, 64, 2, 5, True)
    dims = np.zeros(5, dtype=np.int64)
    _lib.call("qc_host_dims", dec.handle, dims.ctypes.data)
    assert list(dims[:4]) == [64, 2, 5, 1]
    r = dec.decode(np.zeros((0, lay.n_vars)), 1.0)
    assert r.hard_bits.shape == (0, lay.n_vars)


def test_compact_schedule_passes_are_bit_identical(gpu):
    """qc_agg_check + qc_agg_var (compact check records) == qc_cnu_ex(phi) +
    qc_vnu_ex(phi) on the same phi-form packages, bit for bit; also the fused
    first iteration (records from mu) and the last (posteriors + hard bits)."""
    import torch
    q = gpu
    from paper_1204_0334_b200 import _lib
    for name, G in (("n18360", 256), ("code_c_like", 96), ("code_b_like", 64)):   # float4 / float / float2 lanes
        h, exp = q.load_code(q.codes.bundled_code_path(name))
        lay = q.build_edge_layout(h)
        N, M, E = lay.n_vars, lay.n_checks, lay.edge_count
        p, st = lay.plan().handle, _lib.stream_handle()
        sigma = q.ebn0_to_sigma(2.6, 5 / 6)
        mu = torch.empty((N, G), dtype=torch.float32, device="cuda")
        _lib.call("qc_channel", 3, 0, 0, 0, N, G, sigma, mu.data_ptr(), None, None, st)
        a = torch.zeros((E, G), dtype=torch.float32, device="cuda")
        # iteration 1 (fused init) on both schedules
        _lib.call("qc_cnu_ex", p, G, 1, a.data_ptr(), mu.data_ptr(), None, st)
        _lib.call("qc_vnu_ex", p, G, 1, a.data_ptr(), mu.data_ptr(), None, None, None, st)
        b = torch.zeros((E, G), dtype=torch.float32, device="cuda")
        agg = torch.zeros((M, 3, G), dtype=torch.float32, device="cuda")
        _lib.call("qc_agg_check", p, G, 1, b.data_ptr(), mu.data_ptr(), agg.data_ptr(), st)
        _lib.call("qc_agg_var", p, G, 1, b.data_ptr(), mu.data_ptr(), agg.data_ptr(), None, None, st)
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), name
        for _ in range(3):       # middle iterations
            _lib.call("qc_cnu_ex", p, G, 2, a.data_ptr(), mu.data_ptr(), None, st)
            _lib.call("qc_vnu_ex", p, G, 1, a.data_ptr(), mu.data_ptr(), None, None, None, st)
            _lib.call("qc_agg_check", p, G, 0, b.data_ptr(), mu.data_ptr(), agg.data_ptr(), st)
            _lib.call("qc_agg_var", p, G, 0, b.data_ptr(), mu.data_ptr(), agg.data_ptr(), None, None, st)
            assert torch.equal(a.view(torch.int32), b.view(torch.int32)), name
        pa = torch.zeros((N, G), dtype=torch.float32, device="cuda")
        pb = torch.zeros_like(pa)
        ha = torch.zeros((N, G // 32), dtype=torch.int32, device="cuda")
        hb = torch.zeros_like(ha)
        _lib.call("qc_cnu_ex", p, G, 2, a.data_ptr(), mu.data_ptr(), None, st)
        _lib.call("qc_vnu_ex", p, G, 2, a.data_ptr(), mu.data_ptr(), pa.data_ptr(), ha.data_ptr(), None, st)
        _lib.call("qc_agg_check", p, G, 0, b.data_ptr(), mu.data_ptr(), agg.data_ptr(), st)
        _lib.call("qc_agg_var", p, G, 2, b.data_ptr(), mu.data_ptr(), agg.data_ptr(), pb.data_ptr(),
                  hb.data_ptr(), st)
        assert torch.equal(pa.view(torch.int32), pb.view(torch.int32)) and torch.equal(ha, hb), name


_AGG_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1204_0334_b200 as q
h, exp = q.load_code(q.codes.bundled_code_path('n18360'))
lay = q.build_edge_layout(h)
y = q.simulate_block(q.ChannelConfig(2.9, 5 / 6, seed=5, gamma=int(sys.argv[2])), lay.n_vars)
r = q.decode_batch(lay, y, q.ebn0_to_sigma(2.9, 5 / 6), 30)
np.save(sys.argv[1], r.posteriors)
"""


def test_compact_schedule_decode_is_bit_identical(gpu, tmp_path):
    """QCB_AGG=0 (two-pass reference schedule) and the default compact schedule
    decode the same batch to bit-identical posteriors, with the fused
    half-iteration kernels (gamma 512) and the unfused compact passes (384)."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for gamma in (384, 512):      # 512: fused half-iteration kernels; 384: unfused compact passes
        outs = []
        for env in ({"QCB_AGG": "0"}, {"QCB_AGG": "1"}):
            f = tmp_path / f"post{gamma}_{len(outs)}.npy"
            subprocess.run([sys.executable, "-c", _AGG_SNIPPET, str(f), str(gamma)], cwd=repo, check=True,
                           env={**os.environ, **env})
            outs.append(np.load(f))
        for o in outs[1:]:
            assert np.array_equal(outs[0], o), gamma


_SMALL_SNIPPET = r"""
import sys, numpy as np
import paper_1204_0334_b200 as q
out = {}
for name in ("toy", "n18360"):
    if name == "toy":
        lay = q.build_edge_layout(q.expand_qc(q.multiplicative_shifts(2, 4, 8)))
    else:
        lay = q.build_edge_layout(q.load_code(q.codes.bundled_code_path("n18360"))[0])
    for gamma in (32, 64, 96):
        y = np.random.default_rng(gamma).normal(1.0, 0.8, size=(gamma, lay.n_vars))
        dec = q.BlockDecoder(lay, gamma, 12, early_stop=False, graph=False)
        dec.load_lane_major(y, 0.8)
        dec.run()
        r = dec.result(gamma)
        out[f"{name}{gamma}p"] = r.posteriors
        out[f"{name}{gamma}b"] = r.hard_bits
np.savez(sys.argv[1], **out)
"""


def test_small_batch_passes_are_bit_identical(gpu, tmp_path):
    """Batches below 128 lanes run the compact passes with several lanes per
    thread from 8 lane vectors per row (agg.cu pick_vec_small: gamma 32 -> 4
    rows per warp); decisions and posteriors equal the two-pass reference
    schedule (QCB_AGG=0) bit for bit, including gamma 96 (3 lane groups)."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({"QCB_AGG": "0"}, {"QCB_AGG": "1"}):
        f = tmp_path / f"small_{len(outs)}.npz"
        subprocess.run([sys.executable, "-c", _SMALL_SNIPPET, str(f)], cwd=repo, check=True, env={**os.environ, **env})
        outs.append(dict(np.load(f)))
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k


def rel_err(got, ref, atol=1e-12):
    """|delta| / (|ref| + atol): the north star's relative measure (atol only
    guards exact zeros of the reference; fp32 cannot represent below ~1e-38)."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return np.abs(got - ref) / (np.abs(ref) + atol)


def test_single_step_relative_tolerance(gpu):
    """One public check + variable update on identical fp32-representable inputs
    against the float64 reference (bp.py:134-188), in RELATIVE terms:
    * check update: |d alpha| <= 1e-4 |alpha| (atol 1e-12 only guards exact zeros);
    * variable update and posterior: |d| <= 1e-4 |ref| + 2^-20 (|mu| + sum |alpha|)
      -- the second term is a few ulp of fp32 rounding of the running total
      itself (bp.py:179-182: total - alpha and the total cancel when the terms
      have mixed signs), which no fp32 implementation can avoid."""
    q = gpu
    rng = np.random.default_rng(5)
    w_c = w_v = w_p = 0.0
    for d in (2, 3, 4, 6, 8, 16, 24, 32):
        n = d + 5
        rows = [sorted(rng.choice(n, size=d, replace=False)) for _ in range(6)]
        lay = q.build_edge_layout(q.SparseParityCheck(n, rows))
        olay = oqc.layout_from_rows(n, rows)
        mu = rng.normal(0, 1, size=(n, 64)) * rng.choice([0.01, 0.1, 1, 5, 20, 60], size=(n, 1))
        mu = np.clip(mu, -50, 50).astype(np.float32).astype(np.float64)
        b = q.MessageBatch(lay, mu)
        q.check_node_update(b, lay)
        ob = obp.init_buffer(olay, mu)
        obp.check_update(ob, olay)
        w_c = max(w_c, rel_err(b.packages, ob[:-1]).max())
        ob[:-1] = b.packages.astype(np.float32).astype(np.float64)
        mag = np.abs(mu) + np.abs(ob[olay.var_pad]).sum(axis=1)          # |mu| + sum |alpha| per (n, lane)
        post = q.variable_node_update(b, lay)
        opost = obp.var_update(ob, mu, olay)
        w_p = max(w_p, (np.abs(post - opost) / (TOL * np.abs(opost) + 2.0 ** -20 * mag)).max())
        scale = np.zeros_like(ob[:-1])
        for k in range(olay.var_pad.shape[1]):
            e = olay.var_pad[:, k]
            ok = e < olay.edge_count
            scale[e[ok]] = mag[ok]
        w_v = max(w_v, (np.abs(b.packages - ob[:-1]) / (TOL * np.abs(ob[:-1]) + 2.0 ** -20 * scale)).max())
    print(f"check: max relative error {w_c:.3e} (<= 1e-4); variable / posterior: max of "
          f"|d| / (1e-4 |ref| + 2^-20 magnitude) = {w_v:.3f} / {w_p:.3f} (<= 1)")
    assert w_c <= TOL and w_p <= 1.0 and w_v <= 1.0


@pytest.mark.parametrize("shape", ["irregular", "qc"])
def test_masked_single_steps(gpu, shape):
    """check_node_update / variable_node_update with an `active` lane mask
    (bp.py:154-157, 183-187): frozen lanes keep their packages bit for bit,
    active lanes update, and the posteriors of EVERY lane -- frozen ones
    included -- are clip(mu + sum alpha)."""
    q = gpu
    rng = np.random.default_rng(11)
    if shape == "qc":
        exp = q.multiplicative_shifts(3, 6, 11)
        lay = q.build_edge_layout(q.expand_qc(exp))
        olay = oqc.qc_layout(exp.shifts, exp.p)
        n = lay.n_vars
    else:
        n = 40
        rows = [sorted(rng.choice(n, size=int(rng.integers(2, 9)), replace=False)) for _ in range(22)]
        lay = q.build_edge_layout(q.SparseParityCheck(n, rows))
        olay = oqc.layout_from_rows(n, rows)
    G = 96
    mu = np.clip(rng.normal(1.5, 2.5, size=(n, G)), -50, 50).astype(np.float32).astype(np.float64)
    b = q.MessageBatch(lay, mu)
    ob = obp.init_buffer(olay, mu)
    for step in range(3):
        active = rng.random(G) < 0.6
        active[:2] = [True, False]
        before = b.packages.copy()
        q.check_node_update(b, lay, active)
        obp.check_update(ob, olay, active)
        close(b.packages, ob[:-1])
        assert np.array_equal(b.packages[:, ~active], before[:, ~active])
        ob[:-1] = b.packages.astype(np.float32).astype(np.float64)     # identical inputs to the next step
        before = b.packages.copy()
        post = q.variable_node_update(b, lay, active)
        opost = obp.var_update(ob, mu, olay, active)
        close(post, opost)                                         # all lanes, frozen too
        close(b.packages, ob[:-1])
        assert np.array_equal(b.packages[:, ~active], before[:, ~active])
        ob[:-1] = b.packages.astype(np.float32).astype(np.float64)


def test_packages_view_semantics(gpu):
    """MessageBatch.packages behaves like the reference's writable view
    (bp.py:82-84): one host mirror, refreshed in place by updates, caller
    writes honoured by the next update."""
    q = gpu
    lay = toy(q)
    mu = np.random.default_rng(2).normal(2, 2, size=(lay.n_vars, 32)).astype(np.float32).astype(np.float64)
    b = q.MessageBatch(lay, mu)
    pk = b.packages
    assert b.packages is pk                       # O(1) after the first access
    assert np.array_equal(pk, mu[lay.edge_var])
    q.check_node_update(b, lay)
    olay = oqc.qc_layout(q.multiplicative_shifts(2, 4, 8).shifts, 8)
    ob = obp.init_buffer(olay, mu)
    obp.check_update(ob, olay)
    close(pk, ob[:-1])                            # the held array saw the update
    pk[:, 5] = 0.75                               # write through the view
    ob[:-1] = pk
    q.check_node_update(b, lay)
    obp.check_update(ob, olay)
    close(b.packages, ob[:-1])


@pytest.mark.parametrize("db,G,it", [("3.2", 1024, 30), ("3.0", 1024, 30), ("3.6", 1024, 30), ("3.3", 2048, 15),
                                     ("3.2", 1024, 40), ("3.4", 1024, 12), ("3.4", 1024, 11)])
def test_compacted_early_stop_matches_uncompacted(gpu, db, G, it):
    """Early stop with lane compaction (qc_decode_es: continuing lanes packed
    into a second buffer set at checkpoint iterations 11/14/18) equals the
    uncompacted compact-schedule early-stop decode bit for bit -- posteriors at
    each lane's freeze iteration, hard-bit planes, syndrome flags, iteration
    counts, per-lane bit counts -- at waterfall, high-error and high-SNR points,
    for 1-3 checkpoints and for an iteration cap at the first one."""
    import torch
    from paper_1204_0334_b200 import _lib
    q = gpu
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    sigma = q.ebn0_to_sigma(float(db), 1 - lay.n_checks / lay.n_vars)
    outs = []
    small = q.BlockDecoder(lay, 512, it, early_stop=True, graph=False)
    assert small.es_scratch is None                           # below 1024 lanes: the plain early-stop decode
    del small
    for compact in (False, True):
        dec = q.BlockDecoder(lay, G, it, early_stop=True, graph=False, compact=compact)
        assert (dec.es_scratch is not None) == compact
        _lib.call("qc_channel", 9, 1, 77 * G, 0, lay.n_vars, G, sigma, dec.mu.data_ptr(), None, None, 0)
        dec.run()
        dec.run()                                   # repeat: scratch state from a previous decode is harmless
        torch.cuda.synchronize()
        outs.append([x.cpu().numpy() for x in (dec.post, dec.hb, dec.ok, dec.iters, dec.lane_bits)])
    for k, (a, b) in enumerate(zip(*outs)):
        assert np.array_equal(a, b), ("post", "hb", "ok", "iters", "lane_bits")[k]
    its = outs[0][3]
    if it == 30 and db == "3.2":
        assert its.min() < 11 and its.max() > 18               # lanes finish in every segment


def test_compacted_early_stop_against_oracle(gpu):
    """decode through the compacted early-stop engine vs the float64 oracle's
    early-stop decode on the same fixed-seed LLRs (bits, ok, iterations exact;
    posteriors of converged lanes within the north-star tolerance)."""
    import torch
    from oracle import bp as obp
    from oracle import qc as oqc
    q = gpu
    h, exp = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    G = 1024
    sigma = q.ebn0_to_sigma(3.2, 1 - lay.n_checks / lay.n_vars)
    y = q.simulate_block(q.ChannelConfig(3.2, 1 - lay.n_checks / lay.n_vars, seed=4, gamma=G), lay.n_vars)
    dec = q.BlockDecoder(lay, G, 30, early_stop=True, graph=False)
    assert dec.es_scratch is not None
    dec.load_lane_major(y, sigma)
    dec.run()
    r = dec.result(G)
    sel = np.arange(0, G, 64)                              # 16 lanes through the float64 oracle
    olay = oqc.qc_layout(exp.shifts, exp.p)
    bits, post, ok, its = obp.decode_llr(olay, obp.channel_llrs(y[sel], sigma), 30, early_stop=True)
    assert np.array_equal(r.hard_bits[sel], bits)
    assert np.array_equal(r.syndrome_ok[sel], ok)
    assert np.array_equal(r.iterations_run[sel], its)
    # posteriors after 8-20 fp32 iterations: the decisions are exact; values
    # drift like any multi-iteration fp32 decode (DESIGN.md section 3,
    # "Tolerance"): 99.99% within the single-update bound, all within 1e-3
    err = (np.abs(r.posteriors[sel] - post) / np.maximum(np.abs(post), 1.0))[ok]
    assert np.quantile(err, 0.9999) <= 1e-4 and err.max() <= 1e-3, (np.quantile(err, 0.9999), err.max())
    assert len(set(its.tolist())) > 2


def test_host_pipeline_compacted_early_stop_equals_plain(gpu):
    """decode_batch(..., early_stop=True) on 2560 lanes -- 1024-lane chunks
    through the compacted early-stop decode in the host pipeline, smaller
    ramp chunks through the plain one -- equals one uncompacted early-stop
    decode of the whole batch: bits, posteriors, ok, iterations_run."""
    q = gpu
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    G = 2560
    sigma = q.ebn0_to_sigma(3.2, 1 - lay.n_checks / lay.n_vars)
    y = q.simulate_block(q.ChannelConfig(3.2, 1 - lay.n_checks / lay.n_vars, seed=8, gamma=G), lay.n_vars)
    r = q.decode_batch(lay, y, sigma, 30, early_stop=True)
    dec = q.BlockDecoder(lay, G, 30, early_stop=True, graph=False, compact=False)
    dec.load_lane_major(y, sigma)
    dec.run()
    ref = dec.result(G)
    assert np.array_equal(r.iterations_run, ref.iterations_run)
    assert np.array_equal(r.syndrome_ok, ref.syndrome_ok)
    assert np.array_equal(r.hard_bits, ref.hard_bits)
    assert np.array_equal(r.posteriors, ref.posteriors)
    assert r.iterations_run.min() < 12 < r.iterations_run.max()


def test_decode_outputs_pageable_and_page_locked_agree(gpu):
    """decode_batch returns page-locked result arrays by default and ordinary
    ones with set_pinned_outputs(False); small pageable inputs are staged
    page-locked in one copy, large ones go through the pipeline's staging
    threads -- identical results on every path."""
    q = gpu
    from paper_1204_0334_b200 import bp as qbp
    h, _ = q.load_code(q.codes.bundled_code_path("n18360"))
    lay = q.build_edge_layout(h)
    sigma = q.ebn0_to_sigma(3.0, 5 / 6)
    y = 1.0 + sigma * np.random.default_rng(3).standard_normal((96, lay.n_vars))
    ref = q.decode_batch(lay, q.host_array(y), sigma, 20)
    outs = []
    for pinned, stage in ((False, qbp.STAGE_PAGEABLE_MAX_BYTES), (True, 0), (False, 0)):
        q.set_pinned_outputs(pinned)
        old = qbp.STAGE_PAGEABLE_MAX_BYTES
        qbp.STAGE_PAGEABLE_MAX_BYTES = stage
        try:
            outs.append(q.decode_batch(lay, y, sigma, 20))
        finally:
            qbp.STAGE_PAGEABLE_MAX_BYTES = old
            q.set_pinned_outputs(True)
    for r in outs:
        for f in ("hard_bits", "posteriors", "syndrome_ok", "iterations_run"):
            assert np.array_equal(getattr(r, f), getattr(ref, f)), f


def test_small_call_chunking_matches_device_decoder(gpu):
    """decode_batch splits calls from 65 lanes into 64 / 128-lane chunks (bp.py
    _host_decoder); every size around the break points equals one device
    BlockDecoder run over the same lanes (toy code, 9 iterations)."""
    q = gpu
    lay = toy(q)
    y = np.random.default_rng(12).normal(1.0, 0.9, size=(255, lay.n_vars))
    dec = q.BlockDecoder(lay, 256, 9, graph=False, count_bits=False)
    dec.load_lane_major(y, 0.9)
    dec.run()
    ref = dec.result(255)
    for G in (1, 33, 64, 65, 96, 127, 128, 129, 200, 255):
        r = q.decode_batch(lay, y[:G], 0.9, 9)
        for f in ("hard_bits", "posteriors", "syndrome_ok", "iterations_run"):
            assert np.array_equal(getattr(r, f), getattr(ref, f)[:G]), (G, f)
