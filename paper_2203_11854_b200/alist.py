"""ParityCheckMatrix (alist.py:25-84): the Tanner-graph type bp_decode takes,
and the alist text format it is read from (alist.py:86-179, SURVEY.md 8f
item 3: the generic-graph path).

Host-side data structure with the reference's consistency checks; the
device CSR handle for the GPU decoder is built lazily and cached on the
instance, the way the reference caches its _EdgeGraph (ldpc.py:57-62).
parse_alist / to_alist are host text I/O with the reference's format,
padding rule, validation order and AlistParseError line numbers.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass
class ParityCheckMatrix:
    n: int
    m: int
    col_adj: list  # per-variable sorted check indices
    row_adj: list  # per-check sorted variable indices

    def __post_init__(self):
        self.col_adj = [np.asarray(a, dtype=np.int64) for a in self.col_adj]
        self.row_adj = [np.asarray(a, dtype=np.int64) for a in self.row_adj]
        if len(self.col_adj) != self.n or len(self.row_adj) != self.m:
            raise ValueError("adjacency list lengths do not match n, m")
        col_pairs = set()
        for v, checks in enumerate(self.col_adj):
            if len(np.unique(checks)) != len(checks):
                raise ValueError(f"duplicate edges at variable {v}")
            for c in checks.tolist():
                if not 0 <= c < self.m:
                    raise ValueError(f"check index {c} out of range")
                col_pairs.add((v, c))
        seen = 0
        for c, variables in enumerate(self.row_adj):
            if len(np.unique(variables)) != len(variables):
                raise ValueError(f"duplicate edges at check {c}")
            for v in variables.tolist():
                if not 0 <= v < self.n:
                    raise ValueError(f"variable index {v} out of range")
                if (v, c) not in col_pairs:
                    raise ValueError(f"edge ({v},{c}) missing from column lists")
                seen += 1
        if seen != len(col_pairs):
            raise ValueError("row and column adjacency are inconsistent")
        self._graph = None

    @classmethod
    def _trusted(cls, n, m, row_ptr, row_var):
        """Build from a validated CSR without the O(E) Python checks (lifted codes)."""
        obj = cls.__new__(cls)
        obj.n, obj.m = int(n), int(m)
        obj.row_adj = np.split(np.asarray(row_var, np.int64), np.asarray(row_ptr[1:-1]))
        order = np.argsort(row_var, kind="stable")
        chk = np.repeat(np.arange(m), np.diff(row_ptr))[order]
        counts = np.bincount(np.asarray(row_var), minlength=n)
        obj.col_adj = np.split(chk, np.cumsum(counts)[:-1])
        obj._graph = None
        obj._csr = (np.asarray(row_ptr, np.int64), np.asarray(row_var, np.int64))
        return obj

    @property
    def num_edges(self) -> int:
        return int(sum(len(a) for a in self.col_adj))

    @classmethod
    def from_dense(cls, h) -> "ParityCheckMatrix":
        h = np.asarray(h)
        m, n = h.shape
        return cls(n=n, m=m, col_adj=[np.flatnonzero(h[:, v]) for v in range(n)],
                   row_adj=[np.flatnonzero(h[c, :]) for c in range(m)])

    def to_dense(self) -> np.ndarray:
        h = np.zeros((self.m, self.n), dtype=np.uint8)
        for c, variables in enumerate(self.row_adj):
            h[c, variables] = 1
        return h

    def csr(self):
        """Check-major CSR (cptr[m+1], cvar[E]) with ascending variables."""
        if getattr(self, "_csr", None) is None:
            ptr = np.zeros(self.m + 1, np.int64)
            ptr[1:] = np.cumsum([len(a) for a in self.row_adj])
            var = np.concatenate([np.sort(a) for a in self.row_adj]) if self.m else np.zeros(0, np.int64)
            self._csr = (ptr, var.astype(np.int64))
        return self._csr

    def syndrome(self, bits) -> np.ndarray:
        """H @ bits.T over GF(2) for [batch, n] bits (host helper, alist.py:78-84)."""
        bits = np.atleast_2d(np.asarray(bits))
        syn = np.empty((bits.shape[0], self.m), dtype=np.uint8)
        for c, variables in enumerate(self.row_adj):
            syn[:, c] = np.bitwise_xor.reduce(bits[:, variables], axis=1)
        return syn

    def device_graph(self):
        """ls_graph* handle of this matrix (cached)."""
        if self._graph is None:
            ptr, var = self.csr()
            h = ctypes.c_void_p()
            L.call("ls_graph_create", self.n, self.m, ptr.ctypes.data, var.ctypes.data, ctypes.byref(h))
            self._graph = _GraphHandle(h)
        return self._graph.value

    def __getstate__(self):
        d = dict(self.__dict__)
        d["_graph"] = None
        return d


class _GraphHandle:
    def __init__(self, h: ctypes.c_void_p):
        self.h = h

    @property
    def value(self):
        return self.h

    def __del__(self):
        try:
            if self.h and L._lib is not None:
                L._lib.ls_graph_destroy(self.h)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class AlistParseError(ValueError):
    """Malformed alist text; `line` is the 1-based line the problem is on
    (alist.py:18-23)."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


def _int_tokens(tokens, line):
    out = []
    for t in tokens:
        try:
            out.append(int(t))
        except ValueError as exc:
            raise AlistParseError(line, f"non-integer token: {exc}") from None
    return out


def _neighbours(line, tokens, expected, limit, who, idx, what):
    """One adjacency line: non-zero 1-based entries (zeros are padding),
    their count equal to the header degree, each in 1..limit; 0-based and
    sorted on return."""
    nz = [x for x in _int_tokens(tokens, line) if x != 0]
    if len(nz) != expected:
        raise AlistParseError(line, f"{who} {idx}: header says degree {expected}, found {len(nz)}")
    if any(x < 1 or x > limit for x in nz):
        raise AlistParseError(line, f"{what} index out of range 1..{limit}")
    return np.asarray(sorted(x - 1 for x in nz), dtype=np.int64)


def parse_alist(text: str) -> ParityCheckMatrix:
    """alist text -> ParityCheckMatrix (alist.py:93-161).  Blank lines are
    skipped; header degrees are checked against the neighbour lists, and
    every problem raises AlistParseError with its line number."""
    all_lines = text.splitlines()
    rows = [(no, ln.split()) for no, ln in enumerate(all_lines, start=1) if ln.strip()]
    if len(rows) < 4:
        raise AlistParseError(len(all_lines), "truncated file: missing header")
    (l1, t1), (l2, t2), (l3, t3), (l4, t4) = rows[:4]
    if len(t1) != 2:
        raise AlistParseError(l1, "expected 'n m'")
    n, m = _int_tokens(t1, l1)
    if n < 1 or m < 1:
        raise AlistParseError(l1, f"invalid dimensions n={n} m={m}")
    if len(t2) != 2:
        raise AlistParseError(l2, "expected 'max_col_degree max_row_degree'")
    max_col, max_row = _int_tokens(t2, l2)
    col_deg = _int_tokens(t3, l3)
    if len(col_deg) != n:
        raise AlistParseError(l3, f"expected {n} column degrees, got {len(col_deg)}")
    row_deg = _int_tokens(t4, l4)
    if len(row_deg) != m:
        raise AlistParseError(l4, f"expected {m} row degrees, got {len(row_deg)}")
    if max(col_deg) > max_col or max(row_deg) > max_row:
        raise AlistParseError(l4, "degree exceeds declared maximum")
    if len(rows) < 4 + n + m:
        raise AlistParseError(len(all_lines), f"truncated file: expected {4 + n + m} lines")
    body = rows[4:]
    col_adj = [_neighbours(body[v][0], body[v][1], col_deg[v], m, "variable", v, "check") for v in range(n)]
    row_adj = [_neighbours(body[n + c][0], body[n + c][1], row_deg[c], n, "check", c, "variable")
               for c in range(m)]
    try:
        return ParityCheckMatrix(n=n, m=m, col_adj=col_adj, row_adj=row_adj)
    except ValueError as exc:
        raise AlistParseError(4 + n + m, str(exc)) from None


def to_alist(pcm: ParityCheckMatrix) -> str:
    """ParityCheckMatrix -> alist text (alist.py:164-179): 1-based
    neighbours, each line zero-padded to the maximum degree, trailing
    newline."""
    cols = [np.asarray(a) for a in pcm.col_adj]
    rows = [np.asarray(a) for a in pcm.row_adj]
    wc = max((len(a) for a in cols), default=0)
    wr = max((len(a) for a in rows), default=0)

    def line(vals):
        return " ".join(str(int(x)) for x in vals)

    text = [f"{pcm.n} {pcm.m}", f"{wc} {wr}", line(len(a) for a in cols), line(len(a) for a in rows)]
    text += [line([int(x) + 1 for x in a] + [0] * (wc - len(a))) for a in cols]
    text += [line([int(x) + 1 for x in a] + [0] * (wr - len(a))) for a in rows]
    return "\n".join(text) + "\n"
