"""AWGN/BPSK channel with a counter-based, seekable RNG -- generated on the GPU.

Drop-in for /root/reference/pkg/src/qcldpc/channel.py: the same contract
(sample (lane, position) is a pure function of (seed, lane, position); word q
of lane l is Philox4x64-10 keyed by seed at counter (l << 64) + q//4 + 1,
mapped through the inverse normal CDF), evaluated by the `qc_channel` kernel
(csrc/channel.cu, csrc/philox.cuh) in fp64.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import _lib
from .plan import require_cuda

__all__ = ["ChannelConfig", "ebn0_to_sigma", "simulate_block", "lane_normals", "seed_words"]

_M64 = (1 << 64) - 1


@dataclasses.dataclass(frozen=True)
class ChannelConfig:
    """AWGN operating point: Eb/N0 in dB, code rate, seed, lanes per block."""

    ebn0_db: float
    rate: float
    seed: int
    gamma: int = 32

    def __post_init__(self):
        if not 0.0 < self.rate <= 1.0:
            raise ValueError(f"rate must be in (0, 1], got {self.rate}")
        if self.gamma < 1:
            raise ValueError("gamma must be positive")

    @property
    def sigma(self) -> float:
        return ebn0_to_sigma(self.ebn0_db, self.rate)


def ebn0_to_sigma(ebn0_db: float, rate: float) -> float:
    """sigma^2 = 1 / (2 R 10^(dB/10)) for unit-energy BPSK."""
    return math.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0)))


def seed_words(seed: int):
    """128-bit Philox key of an integer seed (numpy's Philox(key=seed))."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("seed must be non-negative")
    return seed & _M64, (seed >> 64) & _M64


def _draw(seed, lane0, start, n, gamma, sigma, want):
    torch = require_cuda()
    k0, k1 = seed_words(seed)
    out = torch.empty((gamma, n), dtype=torch.float64, device="cuda")
    args = [None, None, None]
    args[1 if want == "y" else 2] = out.data_ptr()
    _lib.call("qc_channel", k0, k1, int(lane0), int(start), int(n), int(gamma), float(sigma),
              None, args[1], args[2], _lib.stream_handle())
    return out.cpu().numpy()


def lane_normals(seed: int, lane: int, start: int, count: int) -> np.ndarray:
    """Standard normals at positions start..start+count-1 of one lane."""
    if lane < 0 or start < 0:
        raise ValueError("lane and start must be non-negative")
    if count <= 0:
        return np.zeros(0)
    return _draw(seed, lane, start, count, 1, 1.0, "g")[0]


def simulate_block(cfg: ChannelConfig, n: int, *, lane_offset: int = 0, start: int = 0) -> np.ndarray:
    """Received values y = 1 + sigma g, shape (gamma, n), lanes lane_offset.."""
    if lane_offset < 0 or start < 0:
        raise ValueError("lane and start must be non-negative")
    if n <= 0:
        return np.zeros((cfg.gamma, 0))
    return _draw(cfg.seed, lane_offset, start, n, cfg.gamma, cfg.sigma, "y")
