"""On-chip EXACT QC decoder (csrc/bp_qc_exact.cuh) against the oracle.

Bar (north_star, SURVEY.md 8c tier 1): min-sum and scaled-min-sum
`llr_out`, hard decisions and per-row iteration counts bit-identical to the
reference's bp_decode (ldpc.py:86-172) on identical f32 LLRs, on the whole
mother graph (no dead-row pruning), with and without early stop, for
mother-length input (bp_decode on code.pcm) and rate-matched input with
derate_match fused (ldpc5g_decode, ldpc.py:354-365).  The oracle is the C
restatement of bp_decode, itself pinned to reference-minted goldens
(tests/test_oracle_golden.py).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2203_11854_b200 as lb  # noqa: E402
from paper_2203_11854_b200 import ldpc as LD  # noqa: E402
from oracle import linksim_oracle as O  # noqa: E402

VARIANTS = ["min-sum", "scaled-min-sum"]


def _llrs(k, n, m, ebno, B, seed):
    oc = O.code(k, n)
    bits = O.binary_source((B, k), seed, 1)
    pts = O.qam_points(m)
    x = O.map_bits(oc.encode(bits), pts, m).astype(np.complex64)
    no = O.ebnodb2no(ebno, m, k / n)
    y = O.awgn_single(x, no, seed, 2)
    return bits, O.demap(y, no, pts, m).astype(np.float32)


def _check_mother(code, oc, mother, variant, es, num_iter=20):
    lo, hard, it = lb.bp_decode(mother, code.pcm, num_iter, variant, 0.75, es, return_iters=True, engine="qc")
    lo_o, hard_o, it_o = O.bp_decode_csr(mother, *oc._csr, oc.n_full, num_iter, variant, 0.75, es)
    assert lo.dtype == np.float32
    assert np.array_equal(lo.view(np.uint32), lo_o.view(np.uint32)), "llr_out differs (bitwise)"
    assert np.array_equal(hard, hard_o)
    if es:
        assert np.array_equal(it, it_o)
    return lo, hard, it


@pytest.mark.parametrize("k,n,m,ebno", [(256, 512, 2, 2.5), (8448, 16896, 4, 5.2), (4096, 8192, 2, 1.5),
                                        (4096, 12288, 6, 7.0), (1408, 2816, 2, 2.5)])
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("es", [True, False])
def test_qc_exact_mother_input_bit_exact(k, n, m, ebno, variant, es):
    code = lb.LdpcCode5G(k, n)
    assert LD.qc_has_kernel(code, precision="exact")
    oc = O.code(k, n)
    B = 48 if k > 4000 else 200
    _, llr = _llrs(k, n, m, ebno, B, 11)
    _check_mother(code, oc, oc.derate_match(llr), variant, es)


@pytest.mark.parametrize("variant", VARIANTS)
def test_qc_exact_config2_512_codewords_bit_exact(variant):
    """north_star config 2 (BG1 k=8448 n=16896, 16-QAM) in the waterfall:
    512 codewords, early stop, everything bit-identical to the oracle."""
    k, n = 8448, 16896
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    _, llr = _llrs(k, n, 4, 5.8, 512, 2024)
    lo, hard, it = _check_mother(code, oc, oc.derate_match(llr), variant, True)
    # the sample spans converged and failing rows
    assert (it < 20).sum() > 64


@pytest.mark.parametrize("ebno", [4.6, 6.0])
def test_qc_exact_config2_fixed_iterations(ebno):
    k, n = 8448, 16896
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    _, llr = _llrs(k, n, 4, ebno, 96, 7)
    for variant in VARIANTS:
        _check_mother(code, oc, oc.derate_match(llr), variant, False)


@pytest.mark.parametrize("k,n,m,ebno", [(256, 512, 2, 2.5), (8448, 16896, 4, 5.2), (4096, 12288, 6, 7.0),
                                        (256, 1536, 2, -1.0)])
@pytest.mark.parametrize("variant", VARIANTS)
def test_qc_exact_fused_derate_and_counts(k, n, m, ebno, variant):
    """ldpc5g_decode(mode='exact') on rate-matched LLRs (derate_match fused
    into the kernel, including repetition for n > buffer) and the fused
    error counts against the payload."""
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    B = 40 if k > 4000 else 160
    bits, llr = _llrs(k, n, m, ebno, B, 5)
    dec = lb.ldpc5g_decode(llr, code, 20, variant)
    dec_o, lo_o, it_o = O.decode(llr, oc, 20, variant, 0.75, True)
    assert np.array_equal(dec, dec_o)
    r = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision="exact", ref_bits=bits,
                     want_llr=True, want_iters=True)
    assert np.array_equal(r["llr"].cpu().numpy().view(np.uint32), lo_o.view(np.uint32))
    assert np.array_equal(r["iters"].cpu().numpy(), it_o)
    assert np.array_equal(r["hard"].cpu().numpy(), dec_o)
    be, ble = O.count_errors(bits, dec_o)
    assert [int(x) for x in r["counts"].cpu()] == [be, ble]


@pytest.mark.parametrize("k,n", [(256, 512), (8448, 16896)])
def test_qc_exact_ties_zeros_and_saturation(k, n):
    """Inputs built to hit the corner cases of the reference arithmetic:
    integer LLRs (ties at min1, the unique-argmin rule), signed zeros
    (signbit(-0.0) in the syndrome and the check signs), magnitudes far
    above the +-40 clip and denormals."""
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    rng = np.random.default_rng(3)
    B = 24
    mother = rng.integers(-3, 4, size=(B, oc.n_full)).astype(np.float32)
    mother[mother == 0] = np.where(rng.random((mother == 0).sum()) < 0.5, -0.0, 0.0).astype(np.float32)
    mother[1] = np.float32(-0.0)
    mother[2] = rng.choice(np.array([-1e3, 1e3, 45.0, -45.0, 1e-40, -1e-40], np.float32), oc.n_full)
    mother[3] = np.where(rng.random(oc.n_full) < 0.5, 2.0, -2.0).astype(np.float32)
    for variant in VARIANTS:
        for es in (True, False):
            _check_mother(code, oc, mother, variant, es, num_iter=12)


def test_qc_exact_persistent_batch_equals_csr_engine():
    """More codewords than resident CTAs (persistent claim loop, slices of the
    L2 workspace reused): equal to the HBM-streaming CSR exact decoder."""
    k, n = 4096, 8192
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    _, llr = _llrs(k, n, 2, 1.75, 1200, 9)
    mother = oc.derate_match(llr)
    for es in (True, False):
        a = lb.bp_decode(mother, code.pcm, 20, "min-sum", 0.75, es, return_iters=True, engine="qc")
        b = lb.bp_decode(mother, code.pcm, 20, "min-sum", 0.75, es, return_iters=True, engine="csr")
        assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
        assert np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2])


@pytest.mark.parametrize("k,n,m,ebno,B", [(256, 512, 2, 4.0, 4501), (256, 512, 2, 4.0, 3),
                                          (4096, 8192, 2, 3.0, 701)])
def test_qc_exact_codeword_slots_equal_csr_engine(k, n, m, ebno, B):
    """Several codewords per CTA in lockstep (Z < 384: 14 slots at Z = 26, 2
    at Z = 192), each slot refilled when its codeword stops: batches larger
    than all slots together and smaller than one CTA's, odd sizes, codewords
    stopping at different iterations.  Everything equal to the CSR engine and
    the fused counts equal to the oracle's."""
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    bits, llr = _llrs(k, n, m, ebno, B, 21)
    mother = oc.derate_match(llr)
    for variant in VARIANTS:
        for es in (True, False):
            a = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, es, return_iters=True, engine="qc")
            b = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, es, return_iters=True, engine="csr")
            assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
            assert np.array_equal(a[1], b[1])
            assert np.array_equal(a[2], b[2])
            if es and B > 100:
                assert len(np.unique(a[2])) > 3  # stops spread over iterations
        r = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision="exact", ref_bits=bits,
                         want_iters=True)
        assert np.array_equal(r["hard"].cpu().numpy(), b[1][:, :k])
        be, ble = O.count_errors(bits, b[1][:, :k])
        assert [int(x) for x in r["counts"].cpu()] == [be, ble]


@pytest.mark.parametrize("k,n", [(256, 512), (8448, 16896), (1408, 2816)])
@pytest.mark.parametrize("num_iter", [1, 2, 3])
def test_qc_exact_few_iterations_equal_csr_engine(k, n, num_iter):
    """1-3 iterations (the first iteration has no early-stop test; zeroed
    slot state must equal the reference's zero messages), with and without
    early stop, one slot (Z=384) and several (Z=26: 14, Z=64: 6)."""
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    _, llr = _llrs(k, n, 2, 3.0, 300 if k < 1000 else 64, 17)
    mother = oc.derate_match(llr)
    for es in (True, False):
        a = lb.bp_decode(mother, code.pcm, num_iter, "scaled-min-sum", 0.75, es, return_iters=True, engine="qc")
        b = lb.bp_decode(mother, code.pcm, num_iter, "scaled-min-sum", 0.75, es, return_iters=True, engine="csr")
        assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
        assert np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2])


def test_qc_exact_rejects_sum_product_and_unknown_engine():
    code = lb.LdpcCode5G(256, 512)
    llr = np.zeros((2, code.n_full), np.float32)
    with pytest.raises(ValueError):
        lb.bp_decode(llr, code.pcm, 5, "sum-product", engine="qc")
    with pytest.raises(ValueError):
        lb.bp_decode(llr, code.pcm, 5, "min-sum", engine="warp")
    with pytest.raises(ValueError):
        LD.qc_decode(np.zeros((2, code.n), np.float32), code, 5, "sum-product", precision="exact")


@pytest.mark.parametrize("k,n,m,ebno", [(256, 512, 2, 3.0), (8448, 16896, 4, 5.8), (4096, 12288, 6, 7.6)])
@pytest.mark.parametrize("variant", VARIANTS)
def test_fp32_full_graph_decoder_close_to_exact(k, n, m, ebno, variant):
    """north_star fp32 tier: the on-chip decoder with f32 messages over the
    whole mother graph.  On the codewords the reference converges on (early
    stop) the hard decisions are identical and the mother LLRs are within
    1e-4 * max(|L|, 1) of the exact decoder: everywhere for scaled-min-sum
    and on configs 2 and 4; for plain min-sum on config 1 in the waterfall a
    few codewords (1-3 of ~200, tools/fp32_full_stats.py) carry positions up
    to ~2.5e-3, where an f32-rounded min/argmin selection differs from the
    f64 one and unscaled min-sum propagates it, so there the bar is >= 99.5 %
    of positions and >= 97 % of converged codewords entirely within 1e-4."""
    code = lb.LdpcCode5G(k, n)
    B = 64 if k > 4000 else 256
    bits, llr = _llrs(k, n, m, ebno, B, 21)
    ex = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision="exact", want_llr=True,
                      want_iters=True, ref_bits=bits)
    f = LD.qc_decode(llr, code, 20, variant, 0.75, early_stop=True, precision="fp32-full", want_llr=True,
                     want_iters=True, ref_bits=bits)
    conv = ex["iters"].cpu().numpy() < 20
    assert conv.sum() >= B // 4
    he, hf = ex["hard"].cpu().numpy(), f["hard"].cpu().numpy()
    assert np.array_equal(he[conv], hf[conv])
    le, lf = ex["llr"].cpu().numpy()[conv], f["llr"].cpu().numpy()[conv]
    # converged rows: same stopping iteration in all but rare cases; compare those
    same_it = (ex["iters"].cpu().numpy() == f["iters"].cpu().numpy())[conv]
    assert same_it.mean() > 0.9
    d = np.abs(le[same_it] - lf[same_it]) / np.maximum(np.abs(le[same_it]), 1.0)
    if variant == "scaled-min-sum" or k > 256:
        assert d.max() <= 1e-4
    else:
        assert (d <= 1e-4).mean() >= 0.995
        assert (d <= 1e-4).all(axis=1).mean() >= 0.97
        assert d.max() <= 1e-2


def test_fp32_full_graph_noiseless_and_fixed_iterations():
    code = lb.LdpcCode5G(8448, 16896)
    bits = lb.binary_source([16, 8448], lb.RngStream(8, 9))
    tx = lb.ldpc5g_encode(bits, code).astype(np.float32)
    llr = (2.0 * tx - 1.0) * 8.0  # noiseless: ln(p1/p0) > 0 for a one
    for es in (True, False):
        r = LD.qc_decode(llr, code, 20, "min-sum", early_stop=es, precision="fp32-full", ref_bits=bits,
                         want_iters=True)
        assert np.array_equal(r["hard"].cpu().numpy(), bits)
        assert r["counts"].tolist() == [0, 0]


@pytest.mark.parametrize("k,n,m,ebno", [(4096, 8192, 2, 1.75), (4096, 8192, 2, 2.25), (256, 512, 2, 2.0),
                                        (256, 512, 2, 3.0), (8448, 16896, 4, 4.6)])
def test_sum_product_f32_messages_close_to_exact(k, n, m, ebno):
    """The f32-message sum-product option (k_qc_sp32: product-domain check
    update with prefix/suffix products, the reference's f32 first pass; at
    config 2 the messages live in an L2 slice per CTA) against
    the exact sum-product decoder (CSR engine, the reference's arithmetic): on
    the codewords both converge on at the same iteration, identical hard
    decisions and >= 99.9 % of the mother LLRs within 1e-4 * max(|L|, 1) (the
    SURVEY.md 8c sum-product tier), the rest within 1e-3."""
    code = lb.LdpcCode5G(k, n)
    oc = O.code(k, n)
    assert LD.qc_has_kernel(code, precision="fp32-full", variant="sum-product")
    B = 96 if k > 8000 else (192 if k > 1000 else 400)
    _, llr = _llrs(k, n, m, ebno, B, 44)
    mother = oc.derate_match(llr)
    lo_e, hard_e, it_e = lb.bp_decode(mother, code.pcm, 20, "sum-product", 0.75, True, return_iters=True,
                                      engine="csr")
    r = LD.qc_decode(llr, code, 20, "sum-product", early_stop=True, want_llr=True, want_iters=True,
                     precision="fp32-full")
    R = lb.ldpc.L.lib().ls_qc_live_rows(code.handle)
    ncol = code._kb + max(R, 4)  # the pruned dead rows' parity posteriors are channel values
    it_f = r["iters"].cpu().numpy()
    conv = (it_e < 20) & (it_e == it_f)
    assert conv.sum() >= B // 4
    le, lf = lo_e[conv][:, : ncol * code.z], r["llr"].cpu().numpy()[conv][:, : ncol * code.z]
    d = np.abs(le - lf) / np.maximum(np.abs(le), 1.0)
    assert (d <= 1e-4).mean() >= 0.999 and d.max() <= 1e-3
    assert np.array_equal(r["hard"].cpu().numpy()[conv], hard_e[conv][:, :k])


def test_sum_product_f32_messages_unavailable_without_an_instance():
    code = lb.LdpcCode5G(1408, 2816)  # BG1 Z=64: no f32-message sum-product instance
    assert not LD.qc_has_kernel(code, precision="fp32-full", variant="sum-product")
    with pytest.raises(ValueError):
        LD.qc_decode(np.zeros((2, code.n), np.float32), code, 5, "sum-product", precision="fp32-full")
