"""GPU parity: on-device Philox4x64-10 + inverse-CDF channel vs reference vectors."""
import json
import os

import numpy as np
import pytest
from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


def ulps(a, b):
    return np.abs(a - b) / np.spacing(np.maximum(np.abs(a), np.abs(b)))


def test_lane_normals_golden(gpu):
    q = gpu
    cases = json.load(open(os.path.join(GOLDEN, "channel_cases.json")))
    g = golden("channel.npz")
    for i, (seed, lane, start, count) in enumerate(cases):
        got = q.lane_normals(seed, lane, start, count)
        assert ulps(got, g[f"normals_{i}"]).max() <= 2


def test_simulate_block_golden(gpu):
    q = gpu
    g = golden("channel.npz")
    cfg = q.ChannelConfig(3.2, 5 / 6, seed=11, gamma=5)
    y = q.simulate_block(cfg, 300, lane_offset=(1 << 32) + 64, start=20)
    assert np.abs(y - g["block_y"]).max() < 1e-13


def test_seekable_and_pure(gpu):
    q = gpu
    full = q.lane_normals(7, 3, 0, 200)
    assert np.array_equal(q.lane_normals(7, 3, 50, 100), full[50:150])
    parts = np.concatenate([q.lane_normals(7, 3, s, 40) for s in range(0, 200, 40)])
    assert np.array_equal(parts, full)
    a = q.simulate_block(q.ChannelConfig(5.0, 0.5, seed=3, gamma=2), 50)
    b = q.simulate_block(q.ChannelConfig(5.0, 0.5, seed=3, gamma=6), 50)
    assert np.array_equal(a, b[:2])
    with pytest.raises(ValueError):
        q.lane_normals(1, -1, 0, 4)


def test_llrs_match_oracle_fp32(gpu):
    """Device mu (fp32) equals the float64 reference LLR rounded once to fp32."""
    import torch
    from oracle import channel as och
    from paper_1204_0334_b200 import _lib
    sigma = och.ebn0_to_sigma(3.2, 5 / 6)
    n, G = 4096, 64
    mu = torch.empty((n, G), dtype=torch.float32, device="cuda")
    _lib.call("qc_channel", 0, 0, 1 << 32, 0, n, G, sigma, mu.data_ptr(), None, None, 0)
    got = mu.cpu().numpy().T
    y = och.received(0, sigma, 1 << 32, G, n)
    ref = np.clip(2.0 * y / (sigma * sigma), -50, 50).astype(np.float32)
    assert (got != ref).sum() <= 2


def test_normal_statistics(gpu):
    q = gpu
    d = np.concatenate([q.lane_normals(123, g, 0, 250_000) for g in range(4)])
    assert abs(d.mean()) < 0.004 and abs(d.var() - 1.0) < 0.006
    assert abs((d > 0).mean() - 0.5) < 0.002
