"""Statistical parity of the FAST decoders with real power (SURVEY.md 8c
tier 3: BER/BLER within the reference's Monte-Carlo confidence).

The reference side of every comparison is the EXACT decoder on the same
LLRs: it is bit-identical to the reference's bp_decode (min-sum and
scaled-min-sum: tests/test_gpu_qc_exact.py, against the oracle that is pinned
to reference-minted goldens; sum-product: the CSR exact engine, identical
hard decisions), so its block-error indicator per codeword IS the
reference's.  That lets every test use >= 8,192 codewords at waterfall
points (a pure-Python reference run of that size takes hours).  Two tests
per point: the two-proportion z statistic of the BLERs, |z| < 3 (the
north_star bar: BLER inside the reference's Monte-Carlo interval), and
McNemar's paired statistic on the discordant blocks, one-sided: the fast
decoder is not significantly WORSE (z < 3).  The paired test is far more
sensitive than the bar and does detect one difference in the other
direction: fp16x2 scaled-min-sum at 2.25 dB (config 3) decodes more blocks
than the f64 reference (26 vs 56 discordant, z = -3.3).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402


def _chain_llrs(k, n, m, ebno, B, seed):
    """The reference chain's own f32 LLRs (numpy-exact payload and noise,
    f64 demapper cast to f32: Pipeline exact mode, sweep.py:347-363)."""
    cfg = lb.SimConfig.from_dict({"code": {"family": "ldpc5g", "k": k, "n": n, "decoder": {"mode": "exact"}},
                                  "modulation": {"kind": "qam", "bits_per_symbol": m},
                                  "sweep": {"ebno_db": [ebno], "batch_size": B}, "seed": seed})
    pipe = lb.Pipeline(cfg)
    payload, llr = pipe._llr(ebno, B, lb.RngStream(seed, 1))
    return pipe.ldpc, payload, llr


def _block_ok(code, llr, payload, variant, precision, **kw):
    if precision == "csr-exact":
        mother = code.derate_match(llr, device=True)
        _, h = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, True, engine="csr", device=True)
        hard = h[:, : code.k]
    else:
        hard = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision=precision, **kw)["hard"]
    return (hard == payload).all(dim=1).cpu().numpy()


def _z_tests(ok_ref, ok_fast):
    n = len(ok_ref)
    e1, e2 = int((~ok_ref).sum()), int((~ok_fast).sum())
    p = (e1 + e2) / (2 * n)
    z2 = 0.0 if p in (0.0, 1.0) else (e2 - e1) / n / math.sqrt(2 * p * (1 - p) / n)
    b = int((ok_ref & ~ok_fast).sum())  # reference decodes, fast fails
    c = int((~ok_ref & ok_fast).sum())
    zm = 0.0 if b + c == 0 else (b - c) / math.sqrt(b + c)
    return e1, e2, z2, zm, b, c


# (k, n, m, Eb/N0) in the waterfall of each variant on the synthetic graphs
POINTS = {
    "min-sum": [(4096, 8192, 2, 2.75), (4096, 8192, 2, 3.0), (8448, 16896, 4, 5.6)],
    "scaled-min-sum": [(4096, 8192, 2, 2.0), (4096, 8192, 2, 2.25), (8448, 16896, 4, 4.9)],
}
CASES = [(v, *pt) for v, pts in POINTS.items() for pt in pts]


@pytest.mark.parametrize("variant,k,n,m,ebno", CASES)
@pytest.mark.parametrize("precision", ["fp16x2", "fp32-full"])
def test_fast_min_sum_bler_matches_reference(variant, k, n, m, ebno, precision):
    B = 16384 if k < 8000 else 8192
    code, payload, llr = _chain_llrs(k, n, m, ebno, B, 1000 + int(10 * ebno))
    ok_ref = _block_ok(code, llr, payload, variant, "exact")
    ok_fast = _block_ok(code, llr, payload, variant, precision)
    e1, e2, z2, zm, b, c = _z_tests(ok_ref, ok_fast)
    print(f"{k},{n} {ebno} dB {variant} {precision}: ref {e1}/{B} fast {e2}/{B} z={z2:.2f} mcnemar={zm:.2f} ({b},{c})")
    assert e1 >= 20, "point outside the waterfall"
    assert abs(z2) < 3 and zm < 3


@pytest.mark.parametrize("k,n,m,ebno", [(4096, 8192, 2, 1.75), (4096, 8192, 2, 1.5), (8448, 16896, 4, 4.4)])
def test_fast_sum_product_bler_matches_reference(k, n, m, ebno):
    B = 8192 if k < 8000 else 4096
    code, payload, llr = _chain_llrs(k, n, m, ebno, B, 2000 + int(10 * ebno))
    ok_ref = _block_ok(code, llr, payload, "sum-product", "csr-exact")
    ok_fast = _block_ok(code, llr, payload, "sum-product", "fp32")
    e1, e2, z2, zm, b, c = _z_tests(ok_ref, ok_fast)
    print(f"{k},{n} {ebno} dB sum-product: ref {e1}/{B} fast {e2}/{B} z={z2:.2f} mcnemar={zm:.2f} ({b},{c})")
    assert e1 >= 20, "point outside the waterfall"
    assert abs(z2) < 3 and zm < 3


def test_exact_decoder_blocks_equal_oracle_on_4096_codewords():
    """The proxy itself, on the oracle: 4,096 config-3 codewords at 3.0 dB,
    min-sum, block-error indicators (and every hard decision) identical."""
    from oracle import linksim_oracle as O

    k, n = 4096, 8192
    code, payload, llr = _chain_llrs(k, n, 2, 3.0, 4096, 77)
    hard = LD.qc_decode(llr, code, 20, "min-sum", early_stop=True, precision="exact")["hard"].cpu().numpy()
    dec_o, _, _ = O.decode(llr.cpu().numpy(), O.code(k, n), 20, "min-sum", 0.75, True)
    assert np.array_equal(hard, dec_o)
