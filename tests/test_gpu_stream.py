"""GPU parity: pipelined LDPCCC stream decoder vs the reference (goldens) and oracle."""
import numpy as np
import pytest
from conftest import golden

from oracle import qc as oqc
from oracle import stream as ost

pytestmark = pytest.mark.gpu
TOL = 1e-4


def close(got, ref):
    err = np.abs(np.asarray(got) - np.asarray(ref)) / np.maximum(np.abs(ref), 1.0)
    assert err.max() <= TOL, err.max()


def run(q, code, I, G, ys, sigma):
    dec = q.StreamDecoder(code, I, gamma=G)
    out = [f for f in (dec.push_frame(y, sigma) for y in ys) if f is not None]
    return out + dec.flush()


def test_stream_small_golden(gpu):
    q = gpu
    g = golden("stream_small.npz")
    code = q.unwrap_qc(q.multiplicative_shifts(4, 24, 8))
    for I in (2, 3):
        out = run(q, code, I, 3, g[f"I{I}_ys"], float(g[f"I{I}_sigma"]))
        assert [f.frame_index for f in out] == g[f"I{I}_index"].tolist()
        assert [f.tail for f in out] == g[f"I{I}_tail"].tolist()
        assert np.array_equal(np.stack([f.hard_bits for f in out]), g[f"I{I}_bits"])
        close(np.stack([f.posteriors for f in out]), g[f"I{I}_post"])


def test_stream_code_a_golden(gpu, codes_npz):
    q = gpu
    g = golden("stream_code_a.npz")
    code = q.unwrap_qc(q.ExponentMatrix(codes_npz["code_a_shifts"], int(codes_npz["code_a_p"])))
    sigma, I, K = float(g["sigma"]), int(g["I"]), int(g["K"])
    ys = [np.stack([1.0 + sigma * q.lane_normals(0, lane, t * code.c, code.c) for lane in range(2)])
          for t in range(K)]
    out = run(q, code, I, 2, ys, sigma)
    assert [f.frame_index for f in out] == g["index"].tolist()
    assert [f.tail for f in out] == g["tail"].tolist()
    assert np.array_equal(np.stack([np.packbits(f.hard_bits, axis=1) for f in out]), g["bits"])


def test_stream_vs_oracle_with_zero_blocks(gpu):
    """Shift grid with -1 blocks exercises the table path of the LDPCCC kernels."""
    q = gpu
    rng = np.random.default_rng(9)
    sh = rng.integers(0, 11, size=(4, 8))
    sh[0, 1] = sh[2, 5] = sh[3, 3] = -1
    code = q.unwrap_qc(q.ExponentMatrix(sh, 11))
    U = oqc.unwrap(sh, 11)
    sigma, I, G = 0.8, 3, 4
    ys = rng.normal(1.0, sigma, size=(20, G, code.c))
    out = run(q, code, I, G, ys, sigma)
    dec = ost.StreamOracle(U, I, G)
    ref = [f for f in (dec.push(y, sigma) for y in ys) if f is not None] + dec.flush()
    assert [f.frame_index for f in out] == [f.frame_index for f in ref]
    for a, b in zip(out, ref):
        assert np.array_equal(a.hard_bits, b.hard_bits)
        close(a.posteriors, b.posteriors)


def test_stream_lanes_independent_and_gamma_invariant(gpu):
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(4, 24, 8))
    rng = np.random.default_rng(23)
    ys = rng.normal(1.0, 1.0, size=(12, 3, code.c))
    wide = {f.frame_index: f for f in run(q, code, 2, 3, ys, 1.0)}
    for lane in range(3):
        single = {f.frame_index: f for f in run(q, code, 2, 1, ys[:, lane:lane + 1], 1.0)}
        for j in range(12):
            assert np.array_equal(wide[j].posteriors[lane], single[j].posteriors[0])
    # padded widths 64, 96, 160: 4 / 2 lanes per thread with 16, 24, 40 lane
    # vectors per row (stream.cu vec_for) -- same bits as the 32-lane run
    for G in (50, 96, 130):
        big = {f.frame_index: f for f in run(q, code, 2, G, np.repeat(ys[:, :1], G, axis=1), 1.0)}
        for j in range(12):
            assert np.array_equal(big[j].posteriors, np.repeat(wide[j].posteriors[:1], G, axis=0)), G


def test_stream_api_contract(gpu):
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(4, 24, 8))
    dec = q.StreamDecoder(code, processors=3, gamma=5)
    assert dec.window == 12
    assert dec.channel_memory.shape == (12, code.c, 5)
    assert dec.message_memory.shape == (3, code.edge_count, 5)
    dec = q.StreamDecoder(code, processors=2)
    outs = [dec.push_frame(np.ones((1, code.c)), 0.8) for _ in range(8)]
    assert all(o is None for o in outs[:7]) and outs[7].frame_index == 0 and not outs[7].tail
    rest = dec.flush()
    assert [f.frame_index for f in rest] == list(range(1, 8)) and all(f.tail for f in rest)
    assert not any(f.hard_bits.any() for f in rest)
    with pytest.raises(RuntimeError):
        dec.push_frame(np.ones((1, code.c)), 0.8)
    with pytest.raises(RuntimeError):
        dec.flush()
    with pytest.raises(ValueError):
        q.StreamDecoder(code, processors=0)
    with pytest.raises(ValueError):
        q.StreamDecoder(code, 2, gamma=2).push_frame(np.ones((2, code.c + 1)), 0.8)
    with pytest.raises(ValueError):
        q.unwrap_qc(q.multiplicative_shifts(3, 5, 7))


def test_device_slot_counter_matches_host_slots(gpu):
    """cc_slot with a device-resident slot counter (t_dev + cc_advance, the form a
    captured CUDA graph replays) is bit-identical to host-indexed slots."""
    import torch
    from paper_1204_0334_b200 import _lib
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(4, 24, 8))
    plan = code.plan()
    I, G, K = 2, 32, 14
    window = I * (code.ms + 1)
    rng = np.random.default_rng(5)
    frames = torch.from_numpy(rng.normal(2.0, 3.0, size=(K, code.c, G)).astype(np.float32)).cuda()
    outs = []
    for mode in ("host", "device"):
        msg = torch.zeros((I * code.edge_count, G), dtype=torch.float32, device="cuda")
        ring = torch.zeros((window, code.c, G), dtype=torch.float32, device="cuda")
        post = torch.zeros((K, code.c, G), dtype=torch.float32, device="cuda")
        cnt = torch.zeros((3, G), dtype=torch.int32, device="cuda")
        tdev = torch.zeros(1, dtype=torch.int64, device="cuda")
        s = _lib.stream_handle()
        for t in range(K):
            emit = post[t].data_ptr() if t >= window - 1 else None
            if mode == "host":
                _lib.call("cc_slot", plan.handle, I, G, t, None, msg.data_ptr(), ring.data_ptr(),
                          frames[t].data_ptr(), emit, cnt.data_ptr(), s)
            else:
                _lib.call("cc_slot", plan.handle, I, G, 0, tdev.data_ptr(), msg.data_ptr(), ring.data_ptr(),
                          frames[t].data_ptr(), emit, cnt.data_ptr(), s)
                _lib.call("cc_advance", tdev.data_ptr(), 1, s)
        _lib.call("cc_fold", cnt.data_ptr(), G, s)
        torch.cuda.synchronize()
        if mode == "device":
            assert int(tdev.item()) == K
        outs.append((msg.cpu().numpy(), post.cpu().numpy(), cnt.cpu().numpy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    # one emitted frame per slot from window-1 on, counters folded per frame
    assert int(outs[0][2][1].sum()) == int((outs[0][1][window - 1:] < 0).sum())


@pytest.mark.parametrize("shape", ["qc_4x24", "zero_blocks", "n18360_prime"])
def test_lookahead_slots_match_cc_slot(gpu, shape):
    """cc_slot_ahead (check + variable phase, the emitting processor entering
    frame t+1, the check phase folding counters) and cc_channel_frames (K frames
    per launch) -- the StreamCampaign flow -- equal channel + cc_slot per slot
    bit for bit: message store, ring, emitted posteriors, lane counters."""
    import torch
    from paper_1204_0334_b200 import _lib
    q = gpu
    if shape == "qc_4x24":
        code, I, G = q.unwrap_qc(q.multiplicative_shifts(4, 24, 8)), 3, 64
    elif shape == "zero_blocks":
        sh = np.random.default_rng(9).integers(0, 11, size=(4, 8))
        sh[0, 1] = sh[2, 5] = sh[3, 3] = -1
        code, I, G = q.unwrap_qc(q.ExponentMatrix(sh, 11)), 2, 32
    else:
        _, exp = q.load_code(q.codes.bundled_code_path("n18360"))
        code, I, G = q.unwrap_qc(exp), 2, 128
    plan = code.plan()
    window = I * (code.ms + 1)
    P = window + 9                                   # pushes: bootstrap, steady state, emissions
    sigma, k0, k1 = 0.9, 11, 3
    lane0 = torch.tensor([5 * G], dtype=torch.int64, device="cuda")
    outs = []
    for mode in ("slot", "ahead"):
        msg = torch.zeros((I * code.edge_count, G), dtype=torch.float32, device="cuda")
        ring = torch.zeros((window, code.c, G), dtype=torch.float32, device="cuda")
        post = torch.zeros((P, code.c, G), dtype=torch.float32, device="cuda")
        cnt = torch.zeros((3, G), dtype=torch.int32, device="cuda")
        s = _lib.stream_handle()
        if mode == "slot":
            mu = torch.zeros((code.c, G), dtype=torch.float32, device="cuda")
            for t in range(P):
                _lib.call("cc_channel", plan.handle, k0, k1, 0, lane0.data_ptr(), t, None, G, sigma,
                          mu.data_ptr(), s)
                _lib.call("cc_slot", plan.handle, I, G, t, None, msg.data_ptr(), ring.data_ptr(), mu.data_ptr(),
                          post[t].data_ptr(), cnt.data_ptr(), s)
        else:
            K = 4
            mu = torch.zeros((K, code.c, G), dtype=torch.float32, device="cuda")
            frame = lambda t: mu[t % K].data_ptr()
            _lib.call("cc_channel_frames", plan.handle, k0, k1, 0, lane0.data_ptr(), 0, K, G, sigma,
                      mu.data_ptr(), s)
            _lib.call("cc_slot_part", plan.handle, I, G, 0, None, msg.data_ptr(), ring.data_ptr(), frame(0),
                      None, cnt.data_ptr(), 0, 0, 1, s)
            for t in range(P):
                nxt = t + 1 < P
                if nxt and (t + 1) % K == 0:
                    _lib.call("cc_channel_frames", plan.handle, k0, k1, 0, lane0.data_ptr(), t + 1,
                              min(K, P - t - 1), G, sigma, mu.data_ptr(), s)
                _lib.call("cc_slot_ahead", plan.handle, I, G, t, None, msg.data_ptr(), ring.data_ptr(),
                          frame(t + 1) if nxt else None, int(nxt), post[t].data_ptr(), cnt.data_ptr(), s)
        _lib.call("cc_fold", cnt.data_ptr(), G, s)
        torch.cuda.synchronize()
        outs.append((msg.cpu().numpy(), ring.cpu().numpy(), post[window - 1:].cpu().numpy(), cnt.cpu().numpy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    assert int(outs[0][3][1].sum()) > 0 or float(np.abs(outs[0][2]).sum()) > 0


def test_push_frame_outputs_pageable_and_page_locked_agree(gpu):
    """Emitted frames land in page-locked arrays (asynchronous copy-out) by
    default; with set_pinned_outputs(False) they are ordinary numpy arrays and
    each push waits for its copy.  Same frames, same bits either way; also
    through push_llr_device and flush."""
    q = gpu
    import torch
    from paper_1204_0334_b200 import bp as qbp
    code = q.unwrap_qc(q.multiplicative_shifts(4, 24, 11))
    rng = np.random.default_rng(41)
    G = 40
    ys = rng.normal(1.0, 0.8, size=(30, G, code.c))
    runs = []
    for pinned in (True, False):
        q.set_pinned_outputs(pinned)
        try:
            dec = q.StreamDecoder(code, 3, gamma=G)
            out = [f for f in (dec.push_frame(y, 0.8) for y in ys[:20]) if f is not None]
            gp = (G + 31) // 32 * 32
            for y in ys[20:]:
                mu = np.full((code.c, gp), 50.0, dtype=np.float32)
                mu[:, :G] = np.clip(2.0 * y.T / 0.64, -50, 50)
                f = dec.push_llr_device(torch.from_numpy(mu).cuda())
                if f is not None:
                    out.append(f)
            out += dec.flush()
            runs.append(out)
        finally:
            q.set_pinned_outputs(True)
    assert [f.frame_index for f in runs[0]] == [f.frame_index for f in runs[1]]
    for a, b in zip(*runs):
        assert np.array_equal(a.posteriors, b.posteriors) and np.array_equal(a.hard_bits, b.hard_bits)
        assert a.tail == b.tail
    assert qbp._lib.load().qc_host_is_pinned(runs[0][0].posteriors.ctypes.data, runs[0][0].posteriors.nbytes) == 1
    assert qbp._lib.load().qc_host_is_pinned(runs[1][0].posteriors.ctypes.data, runs[1][0].posteriors.nbytes) == 0
