"""ParityCheckMatrix (alist.py:25-84): the Tanner-graph type bp_decode takes.

Host-side data structure with the reference's consistency checks; the
device CSR handle for the GPU decoder is built lazily and cached on the
instance, the way the reference caches its _EdgeGraph (ldpc.py:57-62).
alist text parsing is outside the hot path.
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
