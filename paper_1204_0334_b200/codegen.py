"""Seeded girth->=8 QC-LDPC shift-grid search (host tool, not on the hot path).

The reference ships exactly one code (`pkg/src/qcldpc/data/code_a.qc:1-3`,
"(4,24)-regular, p=422, girth >= 8, shift grid found by randomized search")
and no search tool.  The metric's n=18360 code (J=4, L=24, p=765) is produced
here by the same kind of randomized column-by-column search, seeded so the
committed `data/n18360.qc` is reproducible:

* 4-cycle free  <=>  for every row pair (j1,j2) the column differences
  D[j1,j2,l] = s[j1,l] - s[j2,l] (mod p) are pairwise distinct;
* 6-cycle free  <=>  D[j1,j2,l1] + D[j2,j3,l2] + D[j3,j1,l3] != 0 (mod p) for
  distinct rows and distinct columns.

Columns are added one at a time; a candidate column is accepted when it
creates no 4- or 6-cycle with the columns already placed.
"""

from __future__ import annotations

import itertools

import numpy as np


def _col_ok_mask(cands, placed, p):
    """Vectorised acceptance test of candidate columns (K, J) against placed (n, J)."""
    K, J = cands.shape
    ok = np.ones(K, dtype=bool)
    if placed.shape[0] == 0:
        return ok
    for j1, j2 in itertools.combinations(range(J), 2):
        dn = (cands[:, j1] - cands[:, j2]) % p
        forb = np.zeros(p, bool)
        forb[(placed[:, j1] - placed[:, j2]) % p] = True
        ok &= ~forb[dn]
    n = placed.shape[0]
    if n >= 2:
        a, b = np.where(~np.eye(n, dtype=bool))
        for j1, j2, j3 in itertools.permutations(range(J), 3):
            forb = np.zeros(p, bool)
            s = ((placed[a, j2] - placed[a, j3]) + (placed[b, j3] - placed[b, j1])) % p
            forb[s] = True
            need = (-(cands[:, j1] - cands[:, j2])) % p
            ok &= ~forb[need]
    return ok


def girth8_shifts(J: int, L: int, p: int, seed: int = 0, max_tries: int = 2000) -> np.ndarray:
    """Random (J, L) shift grid over Z_p whose Tanner graph has girth >= 8."""
    rng = np.random.default_rng(seed)
    placed = np.zeros((0, J), dtype=np.int64)
    batch = 4096
    for col in range(L):
        for _ in range(max_tries):
            cands = rng.integers(0, p, size=(batch, J))
            ok = _col_ok_mask(cands, placed, p)
            if ok.any():
                placed = np.vstack([placed, cands[np.argmax(ok)][None, :]])
                break
        else:
            raise RuntimeError(f"no girth-8 column found for column {col} (p={p} too small?)")
    return placed.T.copy()


def has_short_cycles(shifts: np.ndarray, p: int) -> bool:
    """True when the expanded graph has a 4- or 6-cycle (full recheck)."""
    s = np.asarray(shifts, dtype=np.int64)
    placed = np.zeros((0, s.shape[0]), dtype=np.int64)
    for col in s.T:
        if not _col_ok_mask(col[None, :], placed, p)[0]:
            return True
        placed = np.vstack([placed, col[None, :]])
    return False


def render_qc(shifts: np.ndarray, p: int, comment: str = "") -> str:
    J, L = shifts.shape
    out = [f"# {comment}"] if comment else []
    out.append(f"{J} {L} {p}")
    out += [" ".join(str(int(v)) for v in row) for row in shifts]
    return "\n".join(out) + "\n"
