"""alist text format (paper_2203_11854_b200/alist.py; reference alist.py:86-179).

CPU: parsing and serialising against hand-built matrices, the validation
errors with their line numbers, random round trips, and -- where the
reference is importable (this build container) -- identical results and
identical AlistParseError messages to the reference's parse_alist/to_alist
on valid and malformed inputs.  GPU: a parsed graph decodes exactly like
the same graph built from its dense matrix.
"""
import os
import sys

import numpy as np
import pytest

import paper_2203_11854_b200 as lb
from paper_2203_11854_b200.alist import AlistParseError, ParityCheckMatrix, parse_alist, to_alist

H74 = np.array([[1, 1, 0, 1, 1, 0, 0],
                [1, 0, 1, 1, 0, 1, 0],
                [0, 1, 1, 1, 0, 0, 1]], dtype=np.uint8)
# Hamming (7,4), neighbour lines zero-padded to the maximum degree
H74_ALIST = """7 3
3 4
2 2 2 3 1 1 1
4 4 4
1 2 0
1 3 0
2 3 0
1 2 3
1 0 0
2 0 0
3 0 0
1 2 4 5
1 3 4 6
2 3 4 7
"""


def _random_pcm(rng, n, m, p):
    h = (rng.random((m, n)) < p).astype(np.uint8)
    h[rng.integers(0, m, n), np.arange(n)] = 1  # no empty column
    h[np.arange(m), rng.integers(0, n, m)] = 1  # no empty row
    return ParityCheckMatrix.from_dense(h)


def test_parse_hamming_and_serialise_canonically():
    pcm = parse_alist(H74_ALIST)
    assert (pcm.n, pcm.m) == (7, 3)
    assert np.array_equal(pcm.to_dense(), H74)
    assert to_alist(pcm) == H74_ALIST
    # padding is optional, blank lines are skipped
    loose = "\n".join(ln.replace(" 0", "") for ln in H74_ALIST.splitlines())
    assert np.array_equal(parse_alist("\n" + loose.replace("4 4 4", "4 4 4\n")).to_dense(), H74)
    assert isinstance(lb.parse_alist(H74_ALIST), ParityCheckMatrix)


def test_random_round_trips():
    rng = np.random.default_rng(5)
    for _ in range(20):
        pcm = _random_pcm(rng, int(rng.integers(4, 60)), int(rng.integers(2, 30)), 0.15)
        again = parse_alist(to_alist(pcm))
        assert np.array_equal(again.to_dense(), pcm.to_dense())
        assert to_alist(again) == to_alist(pcm)


MALFORMED = [
    ("7 3\n3 4\n", 2),                                   # truncated header
    ("7 3 1\n3 4\n1\n1\n", 1),                           # 'n m' expected
    ("0 3\n3 4\n1\n1 1 1\n", 1),                         # invalid dimensions
    ("7 3\n3\n1\n1\n", 2),                               # 'max_col max_row' expected
    ("7 3\n3 4\n2 2 2 3 1 1\n4 4 4\n", 3),               # 6 column degrees for n = 7
    ("7 3\n3 4\n2 2 2 3 1 1 1\n4 4\n", 4),               # 2 row degrees for m = 3
    ("7 3\n3 3\n2 2 2 3 1 1 1\n4 4 4\n", 4),             # degree above the declared maximum
    ("7 3\n3 4\n2 2 2 3 1 1 x\n4 4 4\n", 3),             # non-integer token
]


def _variants():
    lines = H74_ALIST.splitlines()
    out = list(MALFORMED)
    out.append(("\n".join(lines[:10]) + "\n", 10))                     # body truncated
    bad = list(lines)
    bad[4] = "1 0 0"                                                   # variable 0: degree 1 vs 2
    out.append(("\n".join(bad) + "\n", 5))
    bad = list(lines)
    bad[5] = "1 4 0"                                                   # check index 4 > m
    out.append(("\n".join(bad) + "\n", 6))
    bad = list(lines)
    bad[11] = "1 2 4 6"                                                # rows disagree with columns
    out.append(("\n".join(bad) + "\n", 14))
    return out


@pytest.mark.parametrize("text,line", _variants())
def test_malformed_inputs_raise_with_line_numbers(text, line):
    with pytest.raises(AlistParseError) as ei:
        parse_alist(text)
    assert ei.value.line == line
    assert str(ei.value).startswith(f"line {line}: ")
    assert isinstance(ei.value, ValueError)


REF_SRC = "/root/reference/pkg/src"


def _reference_alist():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not importable here (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from linksim import alist
    return alist


def test_same_results_and_errors_as_the_reference():
    ref = _reference_alist()
    texts = [H74_ALIST] + [t for t, _ in _variants()]
    rng = np.random.default_rng(9)
    for _ in range(10):
        texts.append(to_alist(_random_pcm(rng, int(rng.integers(4, 40)), int(rng.integers(2, 20)), 0.2)))
    for text in texts:
        try:
            want = ref.parse_alist(text)
        except ref.AlistParseError as exc:
            with pytest.raises(AlistParseError) as ei:
                parse_alist(text)
            assert (ei.value.line, str(ei.value)) == (exc.line, str(exc))
            continue
        got = parse_alist(text)
        assert (got.n, got.m) == (want.n, want.m)
        assert all(np.array_equal(a, b) for a, b in zip(got.col_adj, want.col_adj))
        assert all(np.array_equal(a, b) for a, b in zip(got.row_adj, want.row_adj))
        assert to_alist(got) == ref.to_alist(want)


@pytest.mark.gpu
def test_parsed_graph_decodes_like_its_dense_matrix():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(3)
    a = parse_alist(H74_ALIST)
    b = ParityCheckMatrix.from_dense(H74)
    llr = rng.normal(0.0, 2.0, size=(257, 7)).astype(np.float32)
    for variant in ("min-sum", "scaled-min-sum", "sum-product"):
        x = lb.bp_decode(llr, a, 20, variant, 0.75, True, return_iters=True)
        y = lb.bp_decode(llr, b, 20, variant, 0.75, True, return_iters=True)
        for u, v in zip(x, y):
            assert np.array_equal(np.asarray(u), np.asarray(v))
