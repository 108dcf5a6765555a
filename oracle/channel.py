"""AWGN/BPSK channel restatement (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/qcldpc/channel.py:
* sigma = sqrt(1 / (2 R 10^(dB/10))), channel.py:53-58;
* lane_normals, channel.py:61-77: position q of lane l is 64-bit word q mod 4
  of Philox4x64-10(key = [seed_lo, seed_hi], counter = [q//4 + 1, l, 0, 0])
  -- numpy's Philox pre-increments its 256-bit counter before each block --
  mapped to u = ((w >> 11) + 0.5) 2^-53 and g = ndtri(u);
* y = 1 + sigma g, channel.py:80-105.

Third-party arithmetic the reference relies on (not vendored, version floors
numpy>=1.24 / scipy>=1.10, pyproject.toml:10-13): numpy's Philox bit
generator (Random123 Philox4x64-10) and scipy.special.ndtri (Cephes ndtri).
Both are restated below in pure Python (`philox4x64_10`, `ndtri_cephes`) and
pinned bit-for-bit against numpy/scipy by tests/test_oracle.py; the fast
helpers call numpy/scipy directly.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import ndtri

MASK64 = (1 << 64) - 1
PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)


def ebn0_to_sigma(ebn0_db: float, rate: float) -> float:
    return math.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0)))


def philox4x64_10(ctr, key):
    """Random123 Philox4x64 with 10 rounds on python ints."""
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = PHILOX_M[0] * c0
        p1 = PHILOX_M[1] * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0, p1 & MASK64,
                          (p0 >> 64) ^ c3 ^ k1, p0 & MASK64)
        k0 = (k0 + PHILOX_W[0]) & MASK64
        k1 = (k1 + PHILOX_W[1]) & MASK64
    return c0, c1, c2, c3


def lane_words_slow(seed: int, lane: int, start: int, count: int):
    """Raw 64-bit words at positions start.. of a lane (pure Python restatement)."""
    out = []
    key = (seed & MASK64, (seed >> 64) & MASK64)
    for q in range(start, start + count):
        ctr = q // 4 + 1 + (lane << 64)
        words = philox4x64_10(((ctr) & MASK64, (ctr >> 64) & MASK64,
                               (ctr >> 128) & MASK64, (ctr >> 192) & MASK64), key)
        out.append(words[q % 4])
    return out


def lane_words(seed: int, lane: int, start: int, count: int) -> np.ndarray:
    first, off = divmod(start, 4)
    bg = np.random.Philox(key=seed, counter=(lane << 64) + first)
    return np.random.Generator(bg).integers(0, 2**64, dtype=np.uint64,
                                            size=off + count, endpoint=False)[off:]


def words_to_uniform(w: np.ndarray) -> np.ndarray:
    return ((w >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53


def lane_normals(seed: int, lane: int, start: int, count: int) -> np.ndarray:
    if lane < 0 or start < 0:
        raise ValueError("lane and start must be non-negative")
    return ndtri(words_to_uniform(lane_words(seed, lane, start, count)))


def received(seed, sigma, lane0, gamma, n, start=0) -> np.ndarray:
    """(gamma, n) received block for lanes lane0.. (channel.py:80-105)."""
    out = np.empty((gamma, n))
    for g in range(gamma):
        out[g] = 1.0 + sigma * lane_normals(seed, lane0 + g, start, n)
    return out


# Cephes ndtri (scipy.special.ndtri) -------------------------------------------
_P0 = (-5.99633501014107895267E1, 9.80010754185999661536E1, -5.66762857469070293439E1,
       1.39312609387279679503E1, -1.23916583867381258016E0)
_Q0 = (1.95448858338141759834E0, 4.67627912898881538453E0, 8.63602421390890590575E1,
       -2.25462687854119370527E2, 2.00260212380060660359E2, -8.20372256168333339912E1,
       1.59056225126211695515E1, -1.18331621121330003142E0)
_P1 = (4.05544892305962419923E0, 3.15251094599893866154E1, 5.71628192246421288162E1,
       4.40805073893200834700E1, 1.46849561928858024014E1, 2.18663306850790267539E0,
       -1.40256079171354495875E-1, -3.50424626827848203418E-2, -8.57456785154685413611E-4)
_Q1 = (1.57799883256466749731E1, 4.53907635128879210584E1, 4.13172038254672030440E1,
       1.50425385692907503408E1, 2.50464946208309415979E0, -1.42182922854787788574E-1,
       -3.80806407691578277194E-2, -9.33259480895457427372E-4)
_P2 = (3.23774891776946035970E0, 6.91522889068984211695E0, 3.93881025292474443415E0,
       1.33303460815807542389E0, 2.01485389549179081538E-1, 1.23716634817820021358E-2,
       3.01581553508235416007E-4, 2.65806974686737550832E-6, 6.23974539184983293730E-9)
_Q2 = (6.02427039364742014255E0, 3.67983563856160859403E0, 1.37702099489081330271E0,
       2.16236993594496635890E-1, 1.34204006088543189037E-2, 3.28014464682127739104E-4,
       2.89247864745380683936E-6, 6.79019408009981274425E-9)
_EXPM2 = 0.13533528323661269189
_S2PI = 2.50662827463100050242E0


def _horner(x, c, monic=False):
    a = x + c[0] if monic else c[0]
    for v in c[1:]:
        a = a * x + v
    return a


def ndtri_cephes(y0: float) -> float:
    """Inverse standard-normal CDF, Cephes algorithm, for 0 < y0 < 1."""
    neg = True
    y = y0
    if y > 1.0 - _EXPM2:
        y = 1.0 - y
        neg = False
    if y > _EXPM2:
        y -= 0.5
        y2 = y * y
        return (y + y * (y2 * _horner(y2, _P0) / _horner(y2, _Q0, True))) * _S2PI
    x = math.sqrt(-2.0 * math.log(y))
    x0 = x - math.log(x) / x
    z = 1.0 / x
    if x < 8.0:
        x1 = z * _horner(z, _P1) / _horner(z, _Q1, True)
    else:
        x1 = z * _horner(z, _P2) / _horner(z, _Q2, True)
    x = x0 - x1
    return -x if neg else x
