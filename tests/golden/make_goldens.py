"""Mint the golden parity fixtures under tests/golden/ from the reference.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_goldens.py

It imports the unmodified reference in place (PYTHONPATH-style, from
/root/reference/pkg/src) and records its outputs on seeded inputs for every
stage of the hot path (no golden vectors exist in the
reference itself, so they are minted here).  The fixtures are small .npz
files; bits are stored packed.  numpy/scipy versions and the CPU SIMD level
are recorded because numpy's SIMD log/tanh (sum-product) differ by ulps
across hosts.
"""
from __future__ import annotations

import json
import os
import platform
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import linksim  # noqa: F401
    from linksim import channel, core, ldpc, mapping
    from linksim.alist import ParityCheckMatrix
    return core, ldpc, mapping, channel, ParityCheckMatrix


def _meta():
    import scipy
    flags = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = line
                    break
    except OSError:
        pass
    simd = "avx512f" if "avx512f" in flags else ("avx2" if "avx2" in flags else "other")
    return json.dumps({
        "numpy": np.__version__, "scipy": scipy.__version__,
        "python": platform.python_version(), "cpu_simd": simd,
        "reference": "linksim 0.1.0 (/root/reference/pkg)",
    })


def _pcm_csr(pcm):
    ptr = [0]
    var = []
    for row in pcm.row_adj:
        var.extend(int(v) for v in row)
        ptr.append(len(var))
    return np.asarray(ptr, np.int64), np.asarray(var, np.int64)


def base_graphs(ldpc):
    out = {}
    for bg in (1, 2):
        entries, mb, nb, kb = ldpc._base_graph(bg)
        arr = np.array(sorted((r, c, s) for (r, c), s in entries.items()), dtype=np.int16)
        out[f"bg{bg}"] = arr
        out[f"bg{bg}_dims"] = np.array([mb, nb, kb], np.int32)
    return out


def rng_fixture(core, channel):
    out = {}
    keys = [(42, (1 << 32) | 1), (7, 0), (2**63 + 5, 2**64 - 3)]
    for i, (seed, sid) in enumerate(keys):
        s = core.RngStream(seed, sid)
        out[f"raw{i}"] = np.random.Philox(
            key=((seed & (2**64 - 1)) << 64) | (sid & (2**64 - 1))).random_raw(64)
        out[f"bits{i}"] = core.binary_source([3, 100], s)
        out[f"key{i}"] = np.array([seed & (2**64 - 1), sid & (2**64 - 1)], np.uint64)
        out[f"child{i}"] = np.array([s.child(j).stream_id for j in range(4)], np.uint64)
        z = channel.complex_gaussian([4, 500], s.child(2), variance=0.3, dtype=np.complex64)
        out[f"cn{i}"] = z
    out["ebnodb2no"] = np.array([core.ebnodb2no(10.0, 4, 0.5), core.ebnodb2no(2.5, 2, 0.5),
                                 core.ebnodb2no(6.0, 4, 0.5), core.ebnodb2no(-1.0, 6, 1.0 / 3)])
    return out


def chain_fixture(core, ldpc, mapping, channel, k, n, m, ebno_db, batch, seed, sid,
                  variants=("sum-product", "min-sum", "scaled-min-sum"), with_nes=False):
    """One Pipeline.run_batch (sweep.py:347-364, precision 'single') done by hand
    so every intermediate is kept."""
    code = ldpc.LdpcCode5G(k, n)
    const = mapping.Constellation("qam", m)
    rng = core.RngStream(seed, sid)
    no = core.ebnodb2no(ebno_db, m, k / n)
    payload = core.binary_source([batch, k], rng.child(0))
    coded = ldpc.ldpc5g_encode(payload, code)
    x = mapping.map_bits(coded, const).astype(np.complex64)
    y = channel.awgn(x, no, rng.child(2))
    llr_app = mapping.demap_app(y, no, const)
    llr_max = mapping.demap_maxlog(y, no, const)
    llr = np.asarray(llr_app, dtype=np.float32)
    mother = code.derate_match(llr)
    out = dict(payload=np.packbits(payload, axis=-1), coded=np.packbits(coded, axis=-1),
               x=x, y=y, llr_app=llr_app, llr_maxlog=llr_max, llr=llr, mother=mother,
               no=np.float64(no), dims=np.array([k, n, m, batch, code.base_graph, code.z], np.int64),
               transmit_idx=code.transmit_idx.astype(np.int32))
    for var in variants:
        tag = var.replace("-", "_")
        lo, hard = ldpc.bp_decode(mother, code.pcm, num_iter=20, variant=var, scale=0.75)
        out[f"{tag}_llr_out"] = lo
        out[f"{tag}_hard"] = np.packbits(hard, axis=-1)
        dec = ldpc.ldpc5g_decode(llr, code, num_iter=20, variant=var)
        out[f"{tag}_decoded"] = np.packbits(dec, axis=-1)
        if with_nes:
            lo2, hard2 = ldpc.bp_decode(mother, code.pcm, num_iter=20, variant=var,
                                        scale=0.75, early_stop=False)
            out[f"{tag}_nes_llr_out"] = lo2
            out[f"{tag}_nes_hard"] = np.packbits(hard2, axis=-1)
    return out


def chain_double_fixture(core, ldpc, mapping, channel, k, n, m, ebno_db, batch, seed, sid, variants):
    """Pipeline.run_batch with precision 'double' (sweep.py:170, 352, 362):
    complex128 symbols and noise, f64 demapper output decoded as f64.  Done by
    hand to keep the intermediates, then checked against the reference's own
    Pipeline.run_batch."""
    import linksim.sweep as sweep

    code = ldpc.LdpcCode5G(k, n)
    const = mapping.Constellation("qam", m)
    rng = core.RngStream(seed, sid)
    no = core.ebnodb2no(ebno_db, m, k / n)
    payload = core.binary_source([batch, k], rng.child(0))
    coded = ldpc.ldpc5g_encode(payload, code)
    x = mapping.map_bits(coded, const).astype(np.complex128)
    y = channel.awgn(x, no, rng.child(2))
    llr = np.asarray(mapping.demap_app(y, no, const), dtype=np.float64)
    out = dict(payload=np.packbits(payload, axis=-1), y=y, llr=llr, no=np.float64(no),
               dims=np.array([k, n, m, batch, code.base_graph, code.z], np.int64))
    for var in variants:
        tag = var.replace("-", "_")
        dec = ldpc.ldpc5g_decode(llr, code, num_iter=20, variant=var)
        out[f"{tag}_decoded"] = np.packbits(dec, axis=-1)
        cfg = sweep.SimConfig.from_dict({
            "code": {"family": "ldpc5g", "k": k, "n": n, "decoder": {"variant": var, "num_iter": 20}},
            "modulation": {"kind": "qam", "bits_per_symbol": m},
            "sweep": {"ebno_db": [ebno_db], "batch_size": batch}, "seed": seed, "precision": "double"})
        p2, d2 = sweep.Pipeline(cfg).run_batch(ebno_db, batch, core.RngStream(seed, sid))
        assert np.array_equal(p2, payload) and np.array_equal(d2, dec), "by-hand chain != reference Pipeline"
    return out


SWEEP_C1 = {"code": {"family": "ldpc5g", "k": 256, "n": 512,
                     "decoder": {"variant": "min-sum", "num_iter": 20}},
            "modulation": {"kind": "qam", "bits_per_symbol": 2},
            "sweep": {"ebno_db": [1.0, 2.0, 3.0, 4.0, 5.0, 6.0], "batch_size": 64,
                      "target_block_errors": 12, "max_batches_per_point": 5},
            "seed": 11}


def sweep_fixture():
    """The reference's own run_sweep (sweep.py:411-476) on a small config-1
    sweep: per-point counts, batches and stop reasons (deterministic in
    (config, seed) for any worker count), plus its CSV."""
    import linksim.sweep as sweep

    res = sweep.run_sweep(sweep.SimConfig.from_dict(SWEEP_C1), num_workers=4)
    pts = res.points
    csv_text = sweep.format_csv(res)
    return dict(config=json.dumps(SWEEP_C1),
                ebno=np.array([p.ebno_db for p in pts]), bits=np.array([p.bits for p in pts]),
                bit_errors=np.array([p.bit_errors for p in pts]), blocks=np.array([p.blocks for p in pts]),
                block_errors=np.array([p.block_errors for p in pts]),
                batches=np.array([p.batches for p in pts]),
                stop_reason=np.array([p.stop_reason for p in pts]),
                csv_header=csv_text.splitlines()[0])


def misc_fixture(core, ldpc):
    """hard_decide (core.py:102-104) on signed zeros / denormals / ties, and
    exit_mutual_information (ldpc.py:175-188) on seeded LLRs."""
    g = np.random.default_rng(17)
    edge = np.array([0.0, -0.0, 1e-45, -1e-45, 1.0, -1.0, 40.0, -40.0, 1e30, -1e30], np.float32)
    bits = g.integers(0, 2, size=(6, 1000)).astype(np.uint8)
    # consistent Gaussian LLRs L = (2b-1) mu + N(0, 2 mu), mu = 4
    llr = (2.0 * bits - 1.0) * 4.0 + g.normal(size=bits.shape) * np.sqrt(8.0)
    llr_sat = np.concatenate([llr, (2.0 * bits[:1] - 1.0) * 80.0])  # |x| clipped at 40
    llr_sat[-1, :50] *= -1.0
    bits_sat = np.concatenate([bits, bits[:1]])
    return dict(edge=edge, edge_hard=core.hard_decide(edge), edge64_hard=core.hard_decide(edge.astype(np.float64)),
                mi_llr=llr, mi_bits=bits, mi=np.float64(ldpc.exit_mutual_information(llr, bits)),
                mi_llr_sat=llr_sat, mi_bits_sat=bits_sat,
                mi_sat=np.float64(ldpc.exit_mutual_information(llr_sat, bits_sat)),
                mi_perfect=np.float64(ldpc.exit_mutual_information(np.where(bits == 1, 30.0, -30.0), bits)))


def encoder_fixture(core, ldpc):
    out = {}
    for i, (k, n) in enumerate([(256, 512), (8448, 16896), (4096, 8192), (4096, 12288),
                                (500, 1000), (100, 300), (256, 1536), (8448, 25344), (40, 200)]):
        code = ldpc.LdpcCode5G(k, n)
        bits = core.binary_source([4, k], core.RngStream(900 + i, 3))
        out[f"k{i}"] = np.array([k, n, code.base_graph, code.z], np.int64)
        out[f"bits{i}"] = np.packbits(bits, axis=-1)
        out[f"full{i}"] = np.packbits(code.encode_full(bits), axis=-1)
        out[f"tx{i}"] = np.packbits(ldpc.ldpc5g_encode(bits, code), axis=-1)
        out[f"tidx{i}"] = code.transmit_idx.astype(np.int32)
        llr = np.random.default_rng(i).normal(size=(2, n)).astype(np.float32)
        out[f"derate_in{i}"] = llr
        out[f"derate_out{i}"] = code.derate_match(llr)
    return out


def demap_fixture(core, mapping):
    out = {}
    g = np.random.default_rng(1234)
    for m in (2, 4, 6):
        const = mapping.Constellation("qam", m)
        y = (g.normal(size=(3, 64)) + 1j * g.normal(size=(3, 64))).astype(np.complex64) * 0.8
        out[f"points{m}"] = const.points
        out[f"y{m}"] = y
        for no in (0.05, 0.5):
            out[f"app{m}_{no}"] = mapping.demap_app(y, no, const)
            out[f"maxlog{m}_{no}"] = mapping.demap_maxlog(y, no, const)
        bits = g.integers(0, 2, size=(2, 24 * m // 2), dtype=np.uint8)
        out[f"mbits{m}"] = bits
        out[f"mapped{m}"] = mapping.map_bits(bits, const)
        # priors (mapping.py:123-131): flat [m] and per bit [..., S, m]
        flat = g.normal(size=m)
        full = g.normal(size=(3, 64 * m))
        out[f"prior_flat{m}"] = flat
        out[f"prior_full{m}"] = full
        out[f"app_pf{m}"] = mapping.demap_app(y, 0.5, const, prior=flat)
        out[f"app_pp{m}"] = mapping.demap_app(y, 0.5, const, prior=full)
        out[f"maxlog_pp{m}"] = mapping.demap_maxlog(y, 0.5, const, prior=full)
    psk = mapping.Constellation("psk", 3)
    yp = (g.normal(size=(2, 40)) + 1j * g.normal(size=(2, 40))).astype(np.complex64)
    out["psk_points"] = psk.points
    out["psk_y"] = yp
    out["psk_app"] = mapping.demap_app(yp, 0.3, psk)
    return out


def hamming_fixture(core, ldpc, ParityCheckMatrix):
    H = np.array([[1, 1, 0, 1, 1, 0, 0], [1, 0, 1, 1, 0, 1, 0], [0, 1, 1, 1, 0, 0, 1]], np.uint8)
    pcm = ParityCheckMatrix.from_dense(H)
    ptr, var = _pcm_csr(pcm)
    g = np.random.default_rng(99)
    llr64 = g.normal(size=(200, 7)) * 2.0
    llr32 = llr64.astype(np.float32)
    out = dict(H=H, cptr=ptr, cvar=var, llr64=llr64, llr32=llr32)
    for var_ in ("sum-product", "min-sum", "scaled-min-sum"):
        tag = var_.replace("-", "_")
        for es in (True, False):
            for name, llr in (("64", llr64), ("32", llr32)):
                lo, hard = ldpc.bp_decode(llr, pcm, num_iter=7, variant=var_, scale=0.75,
                                          early_stop=es)
                out[f"{tag}_{int(es)}_{name}_out"] = lo
                out[f"{tag}_{int(es)}_{name}_hard"] = hard
    return out


def main():
    core, ldpc, mapping, channel, ParityCheckMatrix = _ref()
    meta = _meta()
    # config 1 in precision 'double' (complex128 / f64 chain)
    np.savez_compressed(os.path.join(OUT, "chain_c1_double.npz"), meta=meta,
                        **chain_double_fixture(core, ldpc, mapping, channel, 256, 512, 2, 2.0, 48, 42,
                                               (1 << 32) | 1, ("min-sum", "scaled-min-sum", "sum-product")))
    np.savez_compressed(os.path.join(OUT, "sweep_c1.npz"), meta=meta, **sweep_fixture())
    np.savez_compressed(os.path.join(OUT, "misc.npz"), meta=meta, **misc_fixture(core, ldpc))
    if "--new-only" in sys.argv:
        return
    np.savez_compressed(os.path.join(OUT, "base_graphs.npz"), meta=meta, **base_graphs(ldpc))
    np.savez_compressed(os.path.join(OUT, "rng.npz"), meta=meta, **rng_fixture(core, channel))
    np.savez_compressed(os.path.join(OUT, "encoder.npz"), meta=meta, **encoder_fixture(core, ldpc))
    np.savez_compressed(os.path.join(OUT, "demap.npz"), meta=meta, **demap_fixture(core, mapping))
    np.savez_compressed(os.path.join(OUT, "hamming.npz"), meta=meta,
                        **hamming_fixture(core, ldpc, ParityCheckMatrix))
    # config 1: BG2 k=256 n=512 QPSK, run_sweep stream of (snr 0, batch 0)
    np.savez_compressed(os.path.join(OUT, "chain_c1.npz"), meta=meta,
                        **chain_fixture(core, ldpc, mapping, channel, 256, 512, 2, 2.0, 48, 42,
                                        (1 << 32) | 1, with_nes=True))
    # config 2: BG1 k=8448 n=16896 (Z=384) 16-QAM; 4 dB sits in the waterfall
    np.savez_compressed(os.path.join(OUT, "chain_c2.npz"), meta=meta,
                        **chain_fixture(core, ldpc, mapping, channel, 8448, 16896, 4, 4.0, 2, 42,
                                        (1 << 32) | 1))
    # config 4: BG1 k=4096 n=12288 64-QAM (r=1/3, fillers, puncturing)
    np.savez_compressed(os.path.join(OUT, "chain_c4.npz"), meta=meta,
                        **chain_fixture(core, ldpc, mapping, channel, 4096, 12288, 6, 0.5, 2, 7,
                                        (3 << 32) | 1, variants=("min-sum",)))
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
