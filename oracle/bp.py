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
    """Exclusive products along axis 1, fixed sequential order, written in
    place with np.multiply(out=) exactly as bp.py:120-131 does (same floats,
    same memory traffic as the reference)."""
    d = t.shape[1]
    f = np.empty_like(t)
    b = np.empty_like(t)
    f[:, 0] = 1.0
    for k in range(1, d):
        np.multiply(f[:, k - 1], t[:, k - 1], out=f[:, k])
    b[:, d - 1] = 1.0
    for k in range(d - 2, -1, -1):
        np.multiply(b[:, k + 1], t[:, k + 1], out=b[:, k])
    return f * b


def _regular_degree(lay):
    """d when every check has degree d (row-major edge ids: check m owns edges
    m*d .. m*d+d-1, so the (E, gamma) buffer reshapes to (M, d, gamma) without
    a gather -- the reference's check_regular path, codes.py:239-247)."""
    d = lay.check_pad.shape[1] if lay.check_pad.ndim == 2 else 0
    return d if d and lay.n_checks * d == lay.edge_count else None


def check_update(buf, lay, active=None):
    """bp.py:134-162 (regular codes reshape, irregular ones gather check_pad)."""
    if lay.edge_count == 0:
        return
    t = np.tanh(0.5 * buf)
    t[-1] = 1.0
    d = _regular_degree(lay)
    g = t[:-1].reshape(lay.n_checks, d, buf.shape[1]) if d else t[lay.check_pad]
    pr = _excl_prod(g)
    np.clip(pr, -1.0 + TANH_CLAMP, 1.0 - TANH_CLAMP, out=pr)
    a = 2.0 * np.arctanh(pr)
    np.clip(a, -L_MAX, L_MAX, out=a)
    if active is not None:
        old = buf[:-1].reshape(a.shape) if d else buf[lay.check_pad]
        a = np.where(active, a, old)
    if d:
        buf[:-1] = a.reshape(lay.edge_count, buf.shape[1])
    else:
        buf[lay.check_pad] = a
        buf[-1] = 0.0


def var_update(buf, mu_vg, lay, active=None):
    """bp.py:165-188: running total in increasing edge order, in place."""
    a = buf[lay.var_pad]                              # (N, dv, gamma), pads read 0
    tot = mu_vg.copy()
    for k in range(a.shape[1]):
        tot += a[:, k]
    beta = np.clip(tot[:, None, :] - a, -L_MAX, L_MAX)
    post = np.clip(tot, -L_MAX, L_MAX)
    if active is not None:
        beta = np.where(active, beta, a)
    buf[lay.var_pad] = beta
    buf[-1] = 0.0
    return post


def hd_syndrome(lay, post_vg):
    """bp.py:191-210."""
    bits = (post_vg < 0).astype(np.uint8)
    if lay.edge_count == 0:
        return bits, np.ones(post_vg.shape[1], bool)
    eb = bits[lay.edge_var]
    d = _regular_degree(lay)
    if d:
        par = eb.reshape(lay.n_checks, d, -1).sum(axis=1)
    else:
        eb = np.concatenate([eb, np.zeros((1, bits.shape[1]), np.uint8)])
        par = eb[lay.check_pad].sum(axis=1)
    return bits, ~np.any(par & 1, axis=0)


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
