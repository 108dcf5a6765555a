"""Flooding sum-product restatement, float64 (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/qcldpc/bp.py:
* constants L_MAX / TANH_CLAMP, bp.py:48-51;
* channel LLR 2y/sigma^2 clipped, bp.py:54-56;
* beta^0 = mu[edge_var] with a neutral scratch row at index E, bp.py:74-84;
* tanh-rule check update with sequential forward/backward exclusive
  products, clamp, 2*atanh, clip, optional lane mask, bp.py:120-162;
* variable update: running total in increasing edge order, beta = clip(total
  - alpha), posterior = clip(total), bp.py:165-188;
* hard decision (bit 1 iff LLR < 0) + per-lane parity, bp.py:191-210;
* decode loop with the early-stop freeze semantics, bp.py:213-265.

Messages are edge-major (E+1, gamma); inputs/outputs lane-major (gamma, N).
"""

from __future__ import annotations

import numpy as np

L_MAX = 50.0
TANH_CLAMP = 1e-12


def channel_llrs(y, sigma):
    return np.clip(2.0 * np.asarray(y, dtype=np.float64) / (sigma * sigma), -L_MAX, L_MAX)


def init_buffer(lay, mu_vg):
    """mu_vg: (N, gamma) -> message buffer (E+1, gamma), scratch row zero."""
    buf = np.zeros((lay.edge_count + 1, mu_vg.shape[1]))
    buf[: lay.edge_count] = mu_vg[lay.edge_var]
    return buf


def _excl_prod(t):
    """Exclusive products along axis 1, fixed sequential order (bp.py:120-131)."""
    d = t.shape[1]
    f = np.ones_like(t)
    b = np.ones_like(t)
    for k in range(1, d):
        f[:, k] = f[:, k - 1] * t[:, k - 1]
    for k in range(d - 2, -1, -1):
        b[:, k] = b[:, k + 1] * t[:, k + 1]
    return f * b


def check_update(buf, lay, active=None):
    if lay.edge_count == 0:
        return
    t = np.tanh(0.5 * buf)
    t[-1] = 1.0
    g = t[lay.check_pad]                              # (M, dc, gamma)
    pr = np.clip(_excl_prod(g), -1.0 + TANH_CLAMP, 1.0 - TANH_CLAMP)
    a = np.clip(2.0 * np.arctanh(pr), -L_MAX, L_MAX)
    if active is not None:
        a = np.where(active, a, buf[lay.check_pad])
    buf[lay.check_pad] = a
    buf[-1] = 0.0


def var_update(buf, mu_vg, lay, active=None):
    a = buf[lay.var_pad]                              # (N, dv, gamma), pads read 0
    tot = mu_vg.copy()
    for k in range(a.shape[1]):
        tot = tot + a[:, k]
    beta = np.clip(tot[:, None, :] - a, -L_MAX, L_MAX)
    if active is not None:
        beta = np.where(active, beta, a)
    buf[lay.var_pad] = beta
    buf[-1] = 0.0
    return np.clip(tot, -L_MAX, L_MAX)


def hd_syndrome(lay, post_vg):
    bits = (post_vg < 0).astype(np.uint8)
    if lay.edge_count == 0:
        return bits, np.ones(post_vg.shape[1], bool)
    eb = np.concatenate([bits[lay.edge_var], np.zeros((1, bits.shape[1]), np.uint8)])
    par = eb[lay.check_pad].sum(axis=1) & 1
    return bits, ~par.any(axis=0)


def decode_llr(lay, mu, iterations, early_stop=False):
    """mu (gamma, N) -> (bits (gamma,N) u8, post (gamma,N), ok (gamma,), iters (gamma,))."""
    if iterations < 1:
        raise ValueError("need at least one iteration")
    mu = np.clip(np.atleast_2d(np.asarray(mu, np.float64)), -L_MAX, L_MAX)
    G = mu.shape[0]
    mv = np.ascontiguousarray(mu.T)
    buf = init_buffer(lay, mv)
    bits = np.zeros((lay.n_vars, G), np.uint8)
    post = np.zeros((lay.n_vars, G))
    ok = np.zeros(G, bool)
    its = np.full(G, iterations, np.int64)
    act = np.ones(G, bool)
    for it in range(1, iterations + 1):
        m = act if early_stop else None
        check_update(buf, lay, m)
        npost = var_update(buf, mv, lay, m)
        if early_stop:
            nb, nok = hd_syndrome(lay, npost)
            post[:, act] = npost[:, act]
            bits[:, act] = nb[:, act]
            ok[act] = nok[act]
            its[act & nok] = it
            act = act & ~nok
            if not act.any():
                break
        else:
            post = npost
    if not early_stop:
        bits, ok = hd_syndrome(lay, post)
    return bits.T.copy(), post.T.copy(), ok, its
