"""Code model: QC shift grids, sparse parity-check matrices, edge layouts.

Host-side plan input (built once per code, never on the hot path).  Mirrors
the names and semantics of /root/reference/pkg/src/qcldpc/codes.py so code
written against the reference keeps working:

* `ExponentMatrix` / `multiplicative_shifts` / `expand_qc`  (codes.py:39-178)
* `SparseParityCheck`                                      (codes.py:89-156)
* `EdgeLayout` / `build_edge_layout`: row-major edge ids, per-variable edge
  lists in increasing id order, padded tables with pad index E (codes.py:181-257)
* `code_stats`, `infer_qc_structure`, `load_code`, `save_code` (codes.py:260-523)

The B200 addition is `EdgeLayout.plan()`: the immutable device plan of the
C ABI (`qc_plan_create_qc` for all-live QC grids -- the kernels then address
edges by shift arithmetic -- else `qc_plan_create_csr`).
"""

from __future__ import annotations

import dataclasses
import math
import os

import numpy as np

__all__ = [
    "CodeFormatError", "ExponentMatrix", "SparseParityCheck", "EdgeLayout", "CodeStats",
    "multiplicative_shifts", "expand_qc", "build_edge_layout", "code_stats",
    "infer_qc_structure", "load_code", "save_code",
]


class CodeFormatError(ValueError):
    """Malformed code file; the message names the offending line."""


@dataclasses.dataclass(frozen=True, eq=False)
class ExponentMatrix:
    """J x L circulant-shift grid; -1 marks an all-zero p x p block."""

    shifts: np.ndarray
    p: int

    def __post_init__(self):
        s = np.asarray(self.shifts, dtype=np.int64)
        if s.ndim != 2 or s.size == 0:
            raise ValueError("shifts must be a non-empty 2-D array")
        if self.p < 1:
            raise ValueError(f"circulant size must be positive, got {self.p}")
        if s.min() < -1 or s.max() >= self.p:
            raise ValueError(f"shifts must lie in [-1, {self.p - 1}]")
        object.__setattr__(self, "shifts", s)

    @property
    def block_rows(self) -> int:
        return self.shifts.shape[0]

    @property
    def block_cols(self) -> int:
        return self.shifts.shape[1]

    @property
    def edge_count(self) -> int:
        return int((self.shifts >= 0).sum()) * self.p


def multiplicative_shifts(block_rows: int, block_cols: int, p: int) -> ExponentMatrix:
    """Array-code grid s[j, l] = j*l mod p."""
    return ExponentMatrix(np.outer(np.arange(block_rows), np.arange(block_cols)) % p, p)


class SparseParityCheck:
    """Binary H stored as strictly increasing per-check column lists."""

    def __init__(self, n_vars: int, check_cols):
        if n_vars < 1:
            raise ValueError("need at least one variable node")
        rows = []
        for m, cols in enumerate(check_cols):
            c = np.asarray(cols, dtype=np.int64)
            if c.ndim != 1:
                raise ValueError(f"check {m}: column list must be 1-D")
            if c.size:
                if c.min() < 0 or c.max() >= n_vars:
                    raise ValueError(f"check {m}: column index out of range")
                if np.unique(c).size != c.size:
                    raise ValueError(f"check {m}: duplicate column")
                c = np.sort(c)
            rows.append(c)
        self.n = int(n_vars)
        self.rows = rows
        self.qc = None          # ExponentMatrix when produced by expand_qc

    @property
    def m(self) -> int:
        return len(self.rows)

    @property
    def edge_count(self) -> int:
        return int(sum(r.size for r in self.rows))

    def row_weights(self) -> np.ndarray:
        return np.array([r.size for r in self.rows], dtype=np.int64)

    def col_weights(self) -> np.ndarray:
        if not self.rows:
            return np.zeros(self.n, np.int64)
        return np.bincount(np.concatenate(self.rows), minlength=self.n).astype(np.int64)

    def to_dense(self) -> np.ndarray:
        h = np.zeros((self.m, self.n), dtype=np.uint8)
        for i, r in enumerate(self.rows):
            h[i, r] = 1
        return h

    @classmethod
    def from_dense(cls, h) -> "SparseParityCheck":
        h = np.asarray(h)
        return cls(h.shape[1], [np.flatnonzero(row) for row in h])

    def __eq__(self, other):
        if not isinstance(other, SparseParityCheck):
            return NotImplemented
        return (self.n == other.n and self.m == other.m
                and all(np.array_equal(a, b) for a, b in zip(self.rows, other.rows)))


def expand_qc(exp: ExponentMatrix) -> SparseParityCheck:
    """Block (j,l) with shift s: ones at (j*p + r, l*p + (r+s) mod p)."""
    p = exp.p
    r = np.arange(p, dtype=np.int64)
    rows = []
    for j in range(exp.block_rows):
        live = np.flatnonzero(exp.shifts[j] >= 0)
        cols = np.sort(live[None, :] * p + (r[:, None] + exp.shifts[j, live][None, :]) % p, axis=1)
        rows.extend(cols)
    h = SparseParityCheck(exp.block_cols * p, rows)
    h.qc = exp
    return h


class EdgeLayout:
    """Row-major edge numbering of H plus padded gather tables (pad = E)."""

    def __init__(self, edge_count, check_ptr, edge_var, var_edges, check_regular,
                 check_pad=None, var_pad=None, qc=None):
        self.edge_count = int(edge_count)
        self.check_ptr = check_ptr
        self.edge_var = edge_var
        self.var_edges = var_edges
        self.check_regular = check_regular
        self.check_pad = check_pad
        self.var_pad = var_pad
        self.qc = qc
        self._plans = {}

    @property
    def n_checks(self) -> int:
        return self.check_ptr.size - 1

    @property
    def n_vars(self) -> int:
        return len(self.var_edges)

    def check_edges(self, m: int) -> np.ndarray:
        return np.arange(self.check_ptr[m], self.check_ptr[m + 1], dtype=np.int64)

    def plan(self):
        """Device plan of the current CUDA device (created on first use, immutable)."""
        import torch
        from .plan import BlockPlan
        dev = torch.cuda.current_device()
        if dev not in self._plans:
            self._plans[dev] = BlockPlan(self)
        return self._plans[dev]

    def __repr__(self):
        return (f"EdgeLayout(N={self.n_vars}, M={self.n_checks}, E={self.edge_count}, "
                f"check_regular={self.check_regular})")


def build_edge_layout(h: SparseParityCheck) -> EdgeLayout:
    w = h.row_weights()
    ptr = np.concatenate([[0], np.cumsum(w)]).astype(np.int64)
    E = int(ptr[-1])
    ev = np.concatenate(h.rows).astype(np.int64) if E else np.zeros(0, np.int64)
    order = np.argsort(ev, kind="stable")           # increasing edge ids per variable
    cw = h.col_weights()
    var_edges = list(np.split(order, np.cumsum(cw)[:-1]))
    regular = int(w[0]) if h.m and np.all(w == w[0]) else None
    dcm = int(w.max()) if h.m else 0
    cpad = np.full((h.m, dcm), E, dtype=np.int64)
    k = np.arange(dcm)
    mask = k[None, :] < w[:, None]
    cpad[mask] = np.arange(E)
    dvm = int(cw.max()) if cw.size else 0
    vpad = np.full((h.n, dvm), E, dtype=np.int64)
    vmask = np.arange(dvm)[None, :] < cw[:, None]
    vpad[vmask] = order
    return EdgeLayout(E, ptr, ev, var_edges, regular, cpad, vpad, qc=getattr(h, "qc", None))


@dataclasses.dataclass(frozen=True)
class CodeStats:
    n: int
    m: int
    edge_count: int
    row_weight_min: int
    row_weight_max: int
    col_weight_min: int
    col_weight_max: int
    regular: bool
    rate_bound: float
    degenerate: bool


def code_stats(h: SparseParityCheck) -> CodeStats:
    rw, cw = h.row_weights(), h.col_weights()
    return CodeStats(
        n=h.n, m=h.m, edge_count=h.edge_count,
        row_weight_min=int(rw.min()) if rw.size else 0,
        row_weight_max=int(rw.max()) if rw.size else 0,
        col_weight_min=int(cw.min()) if cw.size else 0,
        col_weight_max=int(cw.max()) if cw.size else 0,
        regular=bool(rw.size and cw.size and np.all(rw == rw[0]) and np.all(cw == cw[0])),
        rate_bound=1.0 - h.m / h.n,
        degenerate=bool((rw.size and rw.min() == 0) or (cw.size and cw.min() == 0)),
    )


def infer_qc_structure(h: SparseParityCheck) -> ExponentMatrix | None:
    """Coarsest circulant structure (largest p > 1 dividing gcd(M, N)), else None."""
    g = math.gcd(h.m, h.n)
    dense = h.to_dense()
    r = np.arange
    for p in sorted((d for d in range(2, g + 1) if g % d == 0), reverse=True):
        J, L = h.m // p, h.n // p
        blocks = dense.reshape(J, p, L, p).transpose(0, 2, 1, 3)
        shifts = np.full((J, L), -1, dtype=np.int64)
        ok = True
        for j in range(J):
            for l in range(L):
                b = blocks[j, l]
                if not b.any():
                    continue
                s = np.flatnonzero(b[0])
                if s.size != 1:
                    ok = False
                    break
                want = np.zeros((p, p), np.uint8)
                want[r(p), (r(p) + s[0]) % p] = 1
                if not np.array_equal(b, want):
                    ok = False
                    break
                shifts[j, l] = s[0]
            if not ok:
                break
        if ok:
            return ExponentMatrix(shifts, p)
    return None


# ---------------------------------------------------------------------------
# file formats: alist and qc-exponent ("J L p" header, J rows, '#' comments)
# ---------------------------------------------------------------------------
_FORMATS = ("alist", "qc-exponent")


def _fmt(path, format):
    if format:
        if format not in _FORMATS:
            raise CodeFormatError(f"unknown format {format!r}; expected one of {_FORMATS}")
        return format
    ext = os.path.splitext(path)[1].lower()
    if ext == ".alist":
        return "alist"
    if ext == ".qc":
        return "qc-exponent"
    raise CodeFormatError(f"{path}: cannot infer format from extension {ext!r}; pass format=")


def _ints(path, lineno, text, expect=None):
    try:
        vals = [int(t) for t in text.split()]
    except ValueError:
        raise CodeFormatError(f"{path}:{lineno}: non-integer token in {text!r}") from None
    if expect is not None and len(vals) != expect:
        raise CodeFormatError(f"{path}:{lineno}: expected {expect} integers, got {len(vals)}")
    return vals


def _parse_qc(path, lines) -> ExponentMatrix:
    body = [(i + 1, ln.split("#", 1)[0].strip()) for i, ln in enumerate(lines)]
    body = [(i, b) for i, b in body if b]
    if not body:
        raise CodeFormatError(f"{path}:1: empty file")
    lineno, head = body[0]
    J, L, p = _ints(path, lineno, head, 3)
    if min(J, L, p) < 1:
        raise CodeFormatError(f"{path}:{lineno}: J, L, p must be positive")
    if len(body) - 1 != J:
        raise CodeFormatError(f"{path}:{lineno}: header declares {J} shift rows, file has {len(body) - 1}")
    rows = []
    for ln, b in body[1:]:
        v = _ints(path, ln, b, L)
        if min(v) < -1 or max(v) >= p:
            raise CodeFormatError(f"{path}:{ln}: shift outside [-1, {p - 1}]")
        rows.append(v)
    return ExponentMatrix(np.array(rows, dtype=np.int64), p)


def _parse_alist(path, lines) -> SparseParityCheck:
    def line(i):
        if i >= len(lines):
            raise CodeFormatError(f"{path}:{i + 1}: unexpected end of file")
        return lines[i]

    n, m = _ints(path, 1, line(0), 2)
    if n < 1 or m < 1:
        raise CodeFormatError(f"{path}:1: matrix dimensions must be positive")
    mcw, mrw = _ints(path, 2, line(1), 2)
    cw = _ints(path, 3, line(2), n)
    rw = _ints(path, 4, line(3), m)
    if sum(cw) != sum(rw):
        raise CodeFormatError(f"{path}:4: column weights sum to {sum(cw)} but row weights to {sum(rw)}")
    if max(cw, default=0) > mcw or max(rw, default=0) > mrw:
        raise CodeFormatError(f"{path}:2: declared maximum weight exceeded")

    def adj(first, count, weights, limit, kind):
        out = []
        for k in range(count):
            ln = first + k + 1
            vals = _ints(path, ln, line(first + k))
            live = [v for v in vals if v != 0]
            if any(v == 0 for v in vals[:len(live)]):
                raise CodeFormatError(f"{path}:{ln}: zero padding before last entry")
            if len(live) != weights[k]:
                raise CodeFormatError(f"{path}:{ln}: {kind} {k} lists {len(live)} neighbors, "
                                      f"declared weight is {weights[k]}")
            idx = np.array(live, dtype=np.int64) - 1
            if idx.size and (idx.min() < 0 or idx.max() >= limit):
                raise CodeFormatError(f"{path}:{ln}: neighbor index out of range")
            if np.unique(idx).size != idx.size:
                raise CodeFormatError(f"{path}:{ln}: duplicate neighbor")
            out.append(np.sort(idx))
        return out

    vadj = adj(4, n, cw, m, "variable")
    cadj = adj(4 + n, m, rw, n, "check")
    h = SparseParityCheck(n, cadj)
    back = [[] for _ in range(n)]
    for mm, rr in enumerate(h.rows):
        for v in rr:
            back[v].append(mm)
    for v in range(n):
        if not np.array_equal(np.array(back[v], dtype=np.int64), vadj[v]):
            raise CodeFormatError(f"{path}:{5 + v}: variable {v} adjacency disagrees with check lists")
    return h


def load_code(path: str, format: str | None = None):
    """(SparseParityCheck, ExponentMatrix or None) from an alist / .qc file."""
    fmt = _fmt(path, format)
    with open(path) as fh:
        lines = fh.readlines()
    if fmt == "alist":
        return _parse_alist(path, lines), None
    exp = _parse_qc(path, lines)
    return expand_qc(exp), exp


def save_code(path: str, h: SparseParityCheck, exp: ExponentMatrix | None = None,
              format: str | None = None) -> None:
    fmt = _fmt(path, format)
    if fmt == "qc-exponent":
        if exp is None:
            raise ValueError("qc-exponent format needs an ExponentMatrix")
        text = "\n".join([f"{exp.block_rows} {exp.block_cols} {exp.p}"] +
                         [" ".join(str(int(s)) for s in row) for row in exp.shifts]) + "\n"
    else:
        cw, rw = h.col_weights(), h.row_weights()
        vadj = [[] for _ in range(h.n)]
        for mm, r in enumerate(h.rows):
            for v in r:
                vadj[v].append(mm)
        mcw = int(cw.max()) if h.n else 0
        mrw = int(rw.max()) if h.m else 0

        def pad(ids, width):
            return " ".join(str(i + 1) for i in ids) + "".join(" 0" for _ in range(width - len(ids)))

        out = [f"{h.n} {h.m}", f"{mcw} {mrw}", " ".join(map(str, cw)), " ".join(map(str, rw))]
        out += [pad(vadj[v], mcw).strip() for v in range(h.n)]
        out += [pad(list(h.rows[mm]), mrw).strip() for mm in range(h.m)]
        text = "\n".join(out) + "\n"
    with open(path, "w") as fh:
        fh.write(text)


def bundled_code_path(name: str) -> str:
    """Path of a code shipped with this package (data/<name>.qc)."""
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", f"{name}.qc")
