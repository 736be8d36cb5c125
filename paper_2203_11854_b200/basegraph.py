"""Synthetic quasi-cyclic base graphs BG1 (46x68, k_b=22) and BG2 (42x52, k_b=10).

The reference does not use the TS 38.212 tables: it ships graphs drawn from a
fixed seed by its asset tool (/root/reference/pkg/tools/generate_assets.py:
54-116, seeds 20240817 / 20240818 at :134-140) and loads them from
data/ldpc_bg{1,2}.txt (ldpc.py:191-211).  Parity needs the identical graphs,
so this module re-derives them with the same published construction and the
same numpy PCG64 draw sequence instead of shipping the reference's files.
tests/test_host.py (test_base_graph_restatement_matches_reference_tables) checks the
result against the golden copy of the reference tables entry by entry.

Construction (per graph):
  1. accumulate core on parity columns k_b..k_b+3 -- the sum of the four core
     rows leaves one shift-1 circulant on column k_b (what makes the
     encoder's structured solve valid);
  2. one identity block per extension row r >= 4 at column k_b + r;
  3. core rows connect to columns 0, 1 and a random subset of 2..k_b-1;
  4. extension rows draw a few columns from the systematic + core parity
     columns, weighting the punctured columns 0/1 three times;
  5. every systematic column is topped up to degree >= 3;
  each new block gets the first random shift in [0, 384) that does not close
  a length-4 cycle for any of the lifting sizes in CYCLE_MODULI.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

MAX_SHIFT = 384
CYCLE_MODULI = (384, 192, 96, 48, 24, 16, 10, 20, 40)

# (seed, m_b, n_b, k_b, core row degree, extension degree profile)
_SPECS = {
    1: (20240817, 46, 68, 22, 16, (8, 6, 5, 4, 3)),
    2: (20240818, 42, 52, 10, 8, (6, 5, 4, 3, 3)),
}


def _closes_4cycle(blocks: dict, r: int, c: int, s: int) -> bool:
    """True if block (r, c) with shift s would form a 4-cycle r-c-r2-c2 with
    existing blocks, for any modulus in CYCLE_MODULI."""
    same_col = [(rr, ss) for (rr, cc), ss in blocks.items() if cc == c and rr != r]
    same_row = [(cc, ss) for (rr, cc), ss in blocks.items() if rr == r and cc != c]
    for r2, s_r2_c in same_col:
        for c2, s_r_c2 in same_row:
            s_r2_c2 = blocks.get((r2, c2))
            if s_r2_c2 is None:
                continue
            walk = s - s_r_c2 + s_r2_c2 - s_r2_c
            for z in CYCLE_MODULI:
                if walk % z == 0:
                    return True
    return False


def _place(blocks: dict, gen: np.random.Generator, r: int, c: int) -> None:
    if (r, c) in blocks:
        return
    for _attempt in range(400):
        s = int(gen.integers(0, MAX_SHIFT))
        if not _closes_4cycle(blocks, r, c, s):
            blocks[(r, c)] = s
            return
    blocks[(r, c)] = int(gen.integers(0, MAX_SHIFT))


def _derive(seed: int, mb: int, nb: int, kb: int, core_deg: int, ext_profile) -> dict:
    gen = np.random.default_rng(seed)
    blocks = {(0, kb): 1, (1, kb): 0, (3, kb): 0, (0, kb + 1): 0, (1, kb + 1): 0,
              (1, kb + 2): 0, (2, kb + 2): 0, (2, kb + 3): 0, (3, kb + 3): 0}
    for r in range(4, mb):
        blocks[(r, kb + r)] = 0
    for r in range(4):
        want = core_deg if r < 2 else core_deg - 2
        extra = gen.choice(np.arange(2, kb), size=want - 2, replace=False)
        for c in (0, 1, *extra.tolist()):
            _place(blocks, gen, r, int(c))
    n_ext = mb - 4
    prob = np.ones(kb + 4)
    prob[:2] = 3.0
    prob = prob / prob.sum()
    for j in range(n_ext):
        deg = ext_profile[min(j * len(ext_profile) // n_ext, len(ext_profile) - 1)]
        cols = gen.choice(np.arange(kb + 4), size=deg, replace=False, p=prob)
        for c in cols:
            _place(blocks, gen, 4 + j, int(c))
    for c in range(kb):
        deg = sum(1 for (_, cc) in blocks if cc == c)
        while deg < 3:
            r = int(gen.integers(4, mb))
            if (r, c) not in blocks:
                _place(blocks, gen, r, c)
                deg += 1
    return blocks


@lru_cache(maxsize=None)
def base_graph(bg: int):
    """Return (entries, m_b, n_b, k_b); entries is an int64 [nnz, 3] array of
    (row, col, shift) sorted by (row, col), the order of ldpc_bg*.txt."""
    if bg not in _SPECS:
        raise ValueError(f"unknown base graph {bg}")
    seed, mb, nb, kb, core_deg, prof = _SPECS[bg]
    blocks = _derive(seed, mb, nb, kb, core_deg, prof)
    ent = np.array([(r, c, blocks[(r, c)]) for (r, c) in sorted(blocks)], dtype=np.int64)
    ent.setflags(write=False)
    return ent, mb, nb, kb
