"""Code model restatement (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Follows /root/reference/pkg/src/qcldpc/codes.py:
* shift-grid expansion, codes.py:159-178 (block (j,l), shift s: ones at
  row j*p+r, column l*p+(r+s) mod p; columns sorted per check);
* row-major edge numbering and padded gather tables, codes.py:224-257;
* the array-code construction, codes.py:78-86;
* the qc-exponent text format, codes.py:494-517.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def array_code_shifts(J: int, L: int, p: int) -> np.ndarray:
    """(j*l) mod p grid -- codes.py:78-86."""
    return (np.arange(J)[:, None] * np.arange(L)[None, :]) % p


def parse_qc_text(text: str):
    """'J L p' header then J rows of shifts, '#' comments -- codes.py:494-517."""
    body = [ln.split("#", 1)[0].split() for ln in text.splitlines()]
    body = [b for b in body if b]
    J, L, p = (int(v) for v in body[0])
    shifts = np.array([[int(v) for v in row] for row in body[1:]], dtype=np.int64)
    assert shifts.shape == (J, L)
    return shifts, p


def expand(shifts: np.ndarray, p: int):
    """Per-check sorted column lists of the expanded H -- codes.py:159-178."""
    shifts = np.asarray(shifts, dtype=np.int64)
    rows = []
    r = np.arange(p)
    for j in range(shifts.shape[0]):
        live = np.flatnonzero(shifts[j] >= 0)
        cols = live[None, :] * p + (r[:, None] + shifts[j, live][None, :]) % p
        cols.sort(axis=1)
        rows.extend(list(cols))
    return shifts.shape[1] * p, rows


@dataclass
class Layout:
    """Row-major edge numbering -- codes.py:181-257."""

    n_vars: int
    n_checks: int
    edge_count: int
    check_ptr: np.ndarray      # (M+1,)
    edge_var: np.ndarray       # (E,)
    check_pad: np.ndarray      # (M, dc_max), pad = E
    var_pad: np.ndarray        # (N, dv_max), pad = E, edge ids ascending


def layout_from_rows(n_vars: int, rows) -> Layout:
    deg = np.array([len(r) for r in rows], dtype=np.int64)
    ptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    E = int(ptr[-1])
    ev = np.concatenate([np.asarray(r, dtype=np.int64) for r in rows]) if E else \
        np.zeros(0, np.int64)
    M = len(rows)
    dcm = int(deg.max()) if M else 0
    cpad = np.full((M, dcm), E, dtype=np.int64)
    for m in range(M):
        cpad[m, : deg[m]] = np.arange(ptr[m], ptr[m + 1])
    # variable edge lists in increasing edge id (stable sort, codes.py:232-235)
    order = np.argsort(ev, kind="stable")
    vdeg = np.bincount(ev, minlength=n_vars)
    dvm = int(vdeg.max()) if n_vars else 0
    vpad = np.full((n_vars, dvm), E, dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(vdeg)])
    for n in range(n_vars):
        ids = order[starts[n]:starts[n + 1]]
        vpad[n, : ids.size] = ids
    return Layout(n_vars, M, E, ptr, ev, cpad, vpad)


def qc_layout(shifts, p) -> Layout:
    n, rows = expand(shifts, p)
    return layout_from_rows(n, rows)


# ---------------------------------------------------------------------------
# unwrapped (LDPCCC) tables -- convolutional.py:67-151
# ---------------------------------------------------------------------------

@dataclass
class Unwrapped:
    shifts: np.ndarray
    p: int
    lam: int
    ms: int
    sub_j: int
    sub_l: int
    c: int
    cb: int
    lut_c: np.ndarray          # (lam, lam)
    lut_v: np.ndarray          # (lam, lam)
    sub_offset: np.ndarray     # (lam*lam,)
    edge_count: int
    check_tab: list            # per label: (cb, wmax) local ids, -1 pad
    var_tab: list              # per label: (c, sub_j) local ids, -1 pad


def unwrap(shifts, p) -> Unwrapped:
    """Diagonal-cut unwrapping of a QC grid -- convolutional.py:67-151."""
    shifts = np.asarray(shifts, dtype=np.int64)
    J, L = shifts.shape
    lam = math.gcd(J, L)
    if lam < 2:
        raise ValueError("gcd(J, L) < 2: nothing to unwrap")
    sj, sl = J // lam, L // lam
    grid = np.arange(lam * lam).reshape(lam, lam)
    k = np.arange(lam)
    # layer phase kappa couples frames kappa-ms..kappa (convolutional.py:90-93)
    lut_c = np.array([[grid[kap, (kap + 1 + d) % lam] for d in k] for kap in k])
    # frame phase phi couples layers phi..phi+ms (convolutional.py:94-96)
    lut_v = np.array([[grid[(ph + d) % lam, ph] for d in k] for ph in k])
    subs = [shifts[(b // lam) * sj:(b // lam + 1) * sj, (b % lam) * sl:(b % lam + 1) * sl]
            for b in range(lam * lam)]
    counts = np.array([int((g >= 0).sum()) * p for g in subs])
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]])
    cb, c = sj * p, sl * p
    check_tab, var_tab = [], []
    for g in subs:
        w = (g >= 0).sum(axis=1)
        per_row = np.repeat(w, p)
        ptr = np.concatenate([[0], np.cumsum(per_row)])
        wmax = int(per_row.max())
        ct = ptr[:-1, None] + np.arange(wmax)[None, :]
        ct[np.arange(wmax)[None, :] >= per_row[:, None]] = -1
        check_tab.append(ct)
        vt = np.full((c, sj), -1, dtype=np.int64)
        for br in range(sj):
            live = np.flatnonzero(g[br] >= 0)
            rank = np.full(sl, -1)
            rank[live] = np.arange(live.size)
            for v in range(c):
                bc, cc = divmod(v, p)
                s = g[br, bc]
                if s >= 0:
                    vt[v, br] = ptr[br * p + (cc - s) % p] + rank[bc]
        var_tab.append(vt)
    return Unwrapped(shifts, p, lam, lam - 1, sj, sl, c, cb, lut_c, lut_v, offs,
                     int(counts.sum()), check_tab, var_tab)
