"""Pipelined LDPCCC window decoder restatement, float64 (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/qcldpc/convolutional.py:180-357
(StreamDecoder): I processor groups each holding one copy of the base edge
space ordered by sub-block label (convolutional.py:200-218), a ring of
I*(ms+1) channel frames, and per slot t:
* entry: mu_t into ring slot t mod window and into the LUT_v[t mod T]
  sub-blocks of group (t // T) mod I (convolutional.py:256-267);
* check phase: processors i=1..I refresh layer s=t-(i-1)T over frames
  s-ms..s, absent (negative) frames skipped (convolutional.py:269-298);
* variable phase: processors i=1..I refresh frame j=t-iT+1; processor I
  emits posterior/bits (convolutional.py:300-334).
The emission-time zero clear (convolutional.py:328-330) is reproduced.
"""

from __future__ import annotations

import numpy as np

from .bp import L_MAX, TANH_CLAMP, _excl_prod, channel_llrs


class Frame:
    def __init__(self, index, bits, post, tail):
        self.frame_index, self.hard_bits, self.posteriors, self.tail = index, bits, post, tail


class StreamOracle:
    def __init__(self, code, processors: int, gamma: int = 1):
        if processors < 1 or gamma < 1:
            raise ValueError("processors and gamma must be positive")
        self.code, self.I, self.gamma = code, processors, gamma
        self.T = code.ms + 1
        self.window = processors * self.T
        self.t = 0
        self.flushed = False
        E = code.edge_count
        self.scratch = processors * E
        self.msg = np.zeros((processors * E + 1, gamma))
        self.mu = np.zeros((self.window, code.c, gamma))

    def _idx(self, base, tab):
        return np.where(tab < 0, self.scratch, base + tab)

    def push(self, y_frame, sigma):
        if self.flushed:
            raise RuntimeError("decoder already flushed")
        y = np.atleast_2d(np.asarray(y_frame, np.float64))
        if y.shape != (self.gamma, self.code.c):
            raise ValueError("bad frame shape")
        return self._slot(np.ascontiguousarray(channel_llrs(y, sigma).T), False)

    def push_llr(self, mu_cg, tail=False):
        return self._slot(mu_cg, tail)

    def flush(self):
        if self.flushed:
            raise RuntimeError("decoder already flushed")
        out = [f for f in (self._slot(None, True) for _ in range(self.window - 1)) if f]
        self.flushed = True
        return out

    def _slot(self, mu, tail):
        cd, t, T, I = self.code, self.t, self.T, self.I
        E, msg = cd.edge_count, self.msg
        ph = t % T
        grp = ((t // T) % I) * E
        self.mu[t % self.window] = 0.0 if mu is None else mu
        mt = self.mu[t % self.window]
        for d in range(T):
            lb = cd.lut_v[ph, d]
            msg[self._idx(grp + cd.sub_offset[lb], cd.var_tab[lb])] = mt[:, None, :]
        msg[self.scratch] = 0.0
        for i in range(1, I + 1):
            s = t - (i - 1) * T
            if s < 0:
                break
            cols = []
            for d in range(T):
                f = s - cd.ms + d
                if f < 0:
                    continue
                lb = cd.lut_c[ph, d]
                cols.append(self._idx(((f // T) % I) * E + cd.sub_offset[lb], cd.check_tab[lb]))
            idx = np.concatenate(cols, axis=1)
            tv = np.tanh(0.5 * msg[idx])
            tv[idx == self.scratch] = 1.0
            pr = np.clip(_excl_prod(tv), -1.0 + TANH_CLAMP, 1.0 - TANH_CLAMP)
            msg[idx] = np.clip(2.0 * np.arctanh(pr), -L_MAX, L_MAX)
            msg[self.scratch] = 0.0
        out = None
        for i in range(1, I + 1):
            j = t - i * T + 1
            if j < 0:
                break
            pj = j % T
            gb = ((j // T) % I) * E
            idx = np.concatenate([self._idx(gb + cd.sub_offset[cd.lut_v[pj, d]],
                                            cd.var_tab[cd.lut_v[pj, d]]) for d in range(T)],
                                 axis=1)
            a = msg[idx]
            tot = self.mu[j % self.window].copy()
            for k in range(a.shape[1]):
                tot = tot + a[:, k]
            if i == I:
                post = np.clip(tot, -L_MAX, L_MAX)
                out = Frame(j, (post < 0).astype(np.uint8).T.copy(), post.T.copy(), tail)
                msg[idx] = 0.0
                self.mu[j % self.window] = 0.0
            else:
                msg[idx] = np.clip(tot[:, None, :] - a, -L_MAX, L_MAX)
            msg[self.scratch] = 0.0
        self.t = t + 1
        return out
