"""BG2 lifted at Z in {32, 64, 128, 256, 384}: the config-5 decoder-only
sweep's harness-lifted graphs (the reference only reaches
BG2 at k <= 292, ldpc.py:232-238, so LdpcCode5G(k, n, base_graph=2, z=Z)
lifts the same base graph at any Z with the reference's rule, ldpc.py:282-295).

Each is pinned against the oracle restatement O.Code(k, n, bg=2, z=Z):
encoder codewords bit-exact and H.c = 0; exact-mode BP (min-sum,
scaled-min-sum) llr_out / hard / iteration counts bit-exact; the fast fp16x2
decoder identical on every block the reference converges on.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2203_11854_b200 as lb  # noqa: E402
from oracle import linksim_oracle as O  # noqa: E402

ZS = [32, 64, 128, 256, 384]


def _codes(z, rate3=True):
    k = 10 * z
    n = 3 * k if rate3 else 2 * k
    return lb.LdpcCode5G(k, n, base_graph=2, z=z), O.Code(k, n, bg=2, z=z), k, n


def _llrs(oc, k, n, ebno, B, seed):
    bits = O.binary_source((B, k), seed, 1)
    pts = O.qam_points(2)
    x = O.map_bits(oc.encode(bits), pts, 2).astype(np.complex64)
    no = O.ebnodb2no(ebno, 2, k / n)
    y = O.awgn_single(x, no, seed, 2)
    return bits, O.demap(y, no, pts, 2).astype(np.float32)


@pytest.mark.parametrize("z", ZS)
def test_bg2_lifted_encoder_bit_exact(z):
    code, oc, k, n = _codes(z)
    assert (code.base_graph, code.z, code.n_full) == (2, z, 52 * z)
    bits = lb.binary_source([24, k], lb.RngStream(z, 5))
    full = code.encode_full(bits)
    assert np.array_equal(full, oc.encode_full(bits))
    assert np.array_equal(lb.ldpc5g_encode(bits, code), oc.encode(bits))
    assert np.array_equal(code.transmit_idx, oc.transmit_idx)
    assert not code.pcm.syndrome(full).any()  # H c = 0 (ldpc.py:278-296)
    ptr, var = oc.csr
    assert np.array_equal(code.pcm.csr()[0], ptr) and np.array_equal(code.pcm.csr()[1], var)


@pytest.mark.parametrize("z", ZS)
@pytest.mark.parametrize("variant", ["min-sum", "scaled-min-sum"])
def test_bg2_lifted_exact_bp_bit_exact(z, variant):
    code, oc, k, n = _codes(z)
    B = 12 if z >= 256 else 24
    _, llr = _llrs(oc, k, n, 1.2, B, 31 + z)
    mother = oc.derate_match(llr)
    ptr, var = oc.csr
    lo, hard, it = lb.bp_decode(mother, code.pcm, 20, variant, 0.75, True, return_iters=True)
    lo_o, hard_o, it_o = O.bp_decode_csr(mother, ptr, var, oc.n_full, 20, variant, 0.75, True)
    assert np.array_equal(lo.view(np.uint32), lo_o.view(np.uint32))
    assert np.array_equal(hard, hard_o)
    assert np.array_equal(it, it_o)
    dec = lb.ldpc5g_decode(llr, code, 20, variant)
    assert np.array_equal(dec, hard_o[:, :k])


@pytest.mark.parametrize("z", ZS)
def test_bg2_lifted_fast_decoder_converged_blocks(z):
    code, oc, k, n = _codes(z)
    B = 24 if z >= 256 else 48
    bits, llr = _llrs(oc, k, n, 3.6, B, 7 + z)
    res = lb.qc_decode(llr, code, 20, "min-sum", early_stop=True, ref_bits=bits, precision="fp16x2")
    hard = res["hard"].cpu().numpy()
    mother = oc.derate_match(llr)
    ptr, var = oc.csr
    _, hard_o, it_o = O.bp_decode_csr(mother, ptr, var, oc.n_full, 20, "min-sum", 0.75, True)
    ref_hard = hard_o[:, :k]
    ok_ref = (ref_hard == bits).all(axis=1)
    conv = (it_o <= 16) & ok_ref
    assert conv.sum() >= B // 4
    assert np.array_equal(hard[conv], ref_hard[conv])
    ok_fast = (hard == bits).all(axis=1)
    assert (ok_ref != ok_fast).sum() <= max(1, B // 12)
