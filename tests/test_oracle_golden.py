"""Pin the CPU oracle (oracle/) to the golden vectors minted from the reference.

These run on CPU only.  The oracle is the checker for every GPU parity test,
so it must itself reproduce the reference (tests/golden/make_goldens.py):
bit-exact for RNG words, payload bits, codewords, rate-matching maps and the
min-sum BP variants; sum-product within the north-star 1e-4 relative
tolerance with identical hard decisions.
"""
import numpy as np
import pytest

from oracle import linksim_oracle as O


def unpack(a, count):
    return np.unpackbits(a, axis=-1, count=count)


def test_philox_words_bits_and_children(golden):
    z = golden("rng")
    for i in range(3):
        seed, sid = (int(x) for x in z[f"key{i}"])
        assert np.array_equal(O.philox_raw(seed, sid, 64), z[f"raw{i}"])
        assert np.array_equal(O.binary_source((3, 100), seed, sid), z[f"bits{i}"])
        assert [O.child_stream(sid, j) for j in range(4)] == [int(x) for x in z[f"child{i}"]]


def test_complex_gaussian_composition(golden):
    z = golden("rng")
    for i in range(3):
        seed, sid = (int(x) for x in z[f"key{i}"])
        re, im = O.standard_normal_pair((4, 500), seed, O.child_stream(sid, 2))
        got = (np.sqrt(0.3 / 2.0) * (re + 1j * im)).astype(np.complex64)
        assert np.array_equal(got, z[f"cn{i}"])


def test_ebnodb2no_known_values(golden):
    z = golden("rng")
    got = [O.ebnodb2no(10.0, 4, 0.5), O.ebnodb2no(2.5, 2, 0.5), O.ebnodb2no(6.0, 4, 0.5),
           O.ebnodb2no(-1.0, 6, 1.0 / 3)]
    assert np.array_equal(np.array(got), z["ebnodb2no"])
    assert O.ebnodb2no(10.0, 4, 0.5) == pytest.approx(0.05)  # test_core.py:65-67


@pytest.mark.parametrize("i", range(9))
def test_encoder_codes_and_rate_matching(golden, i):
    e = golden("encoder")
    k, n, bg, z = (int(x) for x in e[f"k{i}"])
    c = O.Code(k, n)
    assert (c.bg, c.z) == (bg, z)
    bits = unpack(e[f"bits{i}"], k)
    full = c.encode_full(bits)
    assert np.array_equal(np.packbits(full, axis=-1), e[f"full{i}"])
    assert np.array_equal(np.packbits(c.encode(bits), axis=-1), e[f"tx{i}"])
    assert np.array_equal(c.transmit_idx, e[f"tidx{i}"])
    assert np.array_equal(c.derate_match(e[f"derate_in{i}"]), e[f"derate_out{i}"])


@pytest.mark.parametrize("m", [2, 4, 6])
def test_mapping_and_demapping(golden, m):
    d = golden("demap")
    pts = O.qam_points(m)
    assert np.array_equal(pts, d[f"points{m}"])
    assert np.array_equal(O.map_bits(d[f"mbits{m}"], pts, m), d[f"mapped{m}"])
    for no in (0.05, 0.5):
        app = O.demap(d[f"y{m}"], no, pts, m, "app")
        ref = d[f"app{m}_{no}"]
        assert np.allclose(app, ref, rtol=1e-12, atol=1e-12)
        ml = O.demap(d[f"y{m}"], no, pts, m, "maxlog")
        assert np.allclose(ml, d[f"maxlog{m}_{no}"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("m", [2, 4, 6])
def test_demapping_with_priors_and_psk(golden, m):
    d = golden("demap")
    pts = O.qam_points(m)
    tol = dict(rtol=1e-12, atol=1e-12)
    assert np.allclose(O.demap(d[f"y{m}"], 0.5, pts, m, "app", d[f"prior_flat{m}"]), d[f"app_pf{m}"], **tol)
    assert np.allclose(O.demap(d[f"y{m}"], 0.5, pts, m, "app", d[f"prior_full{m}"]), d[f"app_pp{m}"], **tol)
    assert np.allclose(O.demap(d[f"y{m}"], 0.5, pts, m, "maxlog", d[f"prior_full{m}"]), d[f"maxlog_pp{m}"],
                       **tol)
    assert np.allclose(O.demap(d["psk_y"], 0.3, d["psk_points"], 3, "app"), d["psk_app"], **tol)


@pytest.mark.parametrize("variant", ["sum-product", "min-sum", "scaled-min-sum"])
@pytest.mark.parametrize("es", [0, 1])
@pytest.mark.parametrize("dt", ["64", "32"])
def test_bp_hamming(golden, variant, es, dt):
    h = golden("hamming")
    tag = variant.replace("-", "_")
    lo, hard, _ = O.bp_decode_csr(h["llr" + dt], h["cptr"], h["cvar"], 7, 7, variant, 0.75,
                                  bool(es))
    ref = h[f"{tag}_{es}_{dt}_out"]
    assert np.array_equal(hard, h[f"{tag}_{es}_{dt}_hard"])
    if variant == "sum-product":
        assert np.allclose(lo, ref, rtol=1e-4, atol=1e-4)
    else:
        assert np.array_equal(lo, ref)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
def test_chain_stages(golden, cfg):
    d = golden(f"chain_{cfg}")
    k, n, m, B, bg, z = (int(x) for x in d["dims"])
    c = O.code(k, n)
    assert (c.bg, c.z) == (bg, z)
    payload = unpack(d["payload"], k)
    coded = c.encode(payload)
    assert np.array_equal(np.packbits(coded, axis=-1), d["coded"])
    pts = O.qam_points(m)
    x = O.map_bits(coded, pts, m).astype(np.complex64)
    assert np.array_equal(x, d["x"])
    app = O.demap(d["y"], float(d["no"]), pts, m, "app")
    assert np.allclose(app, d["llr_app"], rtol=1e-10, atol=1e-10)
    ml = O.demap(d["y"], float(d["no"]), pts, m, "maxlog")
    assert np.allclose(ml, d["llr_maxlog"], rtol=1e-12, atol=1e-12)
    assert np.array_equal(c.derate_match(d["llr"]), d["mother"])
    cptr, cvar = c._csr
    for variant in ("sum-product", "min-sum", "scaled-min-sum"):
        tag = variant.replace("-", "_")
        if f"{tag}_llr_out" not in d:
            continue
        lo, hard, _ = O.bp_decode_csr(d["mother"], cptr, cvar, c.n_full, 20, variant, 0.75, True)
        ref = d[f"{tag}_llr_out"]
        assert np.array_equal(np.packbits(hard, axis=-1), d[f"{tag}_hard"])
        if variant == "sum-product":
            rel = np.abs(lo - ref) / np.maximum(np.abs(ref), 1.0)
            assert (rel <= 1e-4).mean() >= 0.999
            assert np.array_equal(np.sign(lo), np.sign(ref))
        else:
            assert np.array_equal(lo, ref)
        dec, _, _ = O.decode(d["llr"], c, 20, variant)
        assert np.array_equal(np.packbits(dec, axis=-1), d[f"{tag}_decoded"])
        if f"{tag}_nes_llr_out" in d:
            lo2, hard2, it2 = O.bp_decode_csr(d["mother"], cptr, cvar, c.n_full, 20, variant,
                                              0.75, False)
            assert np.array_equal(np.packbits(hard2, axis=-1), d[f"{tag}_nes_hard"])
            assert (it2 == 20).all()
            if variant != "sum-product":
                assert np.array_equal(lo2, d[f"{tag}_nes_llr_out"])


def test_run_batch_chain_c1(golden):
    """The whole Pipeline.run_batch on the config-1 stream reproduces the
    reference's payload and decoded bits (noise through numpy's ziggurat)."""
    d = golden("chain_c1")
    k, n, m, B, _, _ = (int(x) for x in d["dims"])
    payload, dec = O.run_batch(k, n, m, 2.0, B, 42, (1 << 32) | 1, "sum-product")
    assert np.array_equal(np.packbits(payload, axis=-1), d["payload"])
    assert np.array_equal(np.packbits(dec, axis=-1), d["sum_product_decoded"])


def test_oracle_hard_decide_and_exit_mi(golden):
    d = golden("misc")
    assert np.array_equal(O.hard_decide(d["edge"]), d["edge_hard"])
    assert np.array_equal(O.hard_decide(d["edge"].astype(np.float64)), d["edge64_hard"])
    assert O.exit_mutual_information(d["mi_llr"], d["mi_bits"]) == float(d["mi"])
    assert O.exit_mutual_information(d["mi_llr_sat"], d["mi_bits_sat"]) == float(d["mi_sat"])
