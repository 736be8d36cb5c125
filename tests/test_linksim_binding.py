"""The linksim binding module (paper_2203_11854_b200/linksim_binding.py,
INTEGRATION.md section 2).

CPU part: where the reference is importable (this build container), enable()
patches exactly the names the reference's Pipeline resolves at call time
(sweep / channel / mapping / ldpc / core globals), a Pipeline built after
enable() binds the B200 demapper, the reference objects convert to B200
handles with identical geometry, and restore() puts the originals back.

GPU part (no reference on the GPU box): the wrappers driven the way the
reference's Pipeline.run_batch drives them (sweep.py:347-364), on stand-in
objects with the reference's attribute names, reproduce the reference's
golden run_batch bit for bit.
"""
import os
import sys
import types

import numpy as np
import pytest

from paper_2203_11854_b200 import linksim_binding as LB

REF_SRC = "/root/reference/pkg/src"


def _reference():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not importable here (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import linksim
    import linksim.sweep  # noqa: F401
    return linksim


def test_enable_patches_what_the_pipeline_resolves_and_restores():
    linksim = _reference()
    before = {(m, n): getattr(getattr(linksim, m), n) for m, n in LB.patched_names()}
    restore = LB.enable(linksim)
    try:
        for m, n in LB.patched_names():
            fn = getattr(getattr(linksim, m), n)
            assert fn is not before[(m, n)], (m, n)
            assert fn.__module__.startswith("paper_2203_11854_b200"), (m, n, fn.__module__)
        # the demapper is bound when a Pipeline is constructed (sweep.py:179)
        cfg = linksim.sweep.SimConfig.from_dict({
            "code": {"family": "ldpc5g", "k": 256, "n": 512},
            "modulation": {"kind": "qam", "bits_per_symbol": 4, "demapper": "maxlog"},
            "sweep": {"ebno_db": [2.0]}})
        pipe = linksim.sweep.Pipeline(cfg)
        assert pipe.demap is linksim.sweep.demap_maxlog
        assert pipe.demap.__module__ == "paper_2203_11854_b200.linksim_binding"
        # handle conversion from the reference objects (no GPU needed)
        for k, n in ((256, 512), (8448, 16896), (4096, 12288)):
            ref = linksim.ldpc.LdpcCode5G(k, n)
            g = LB._code(ref)
            assert (g.base_graph, g.z, g.k, g.n) == (ref.base_graph, ref.z, ref.k, ref.n)
            assert np.array_equal(g.transmit_idx, ref.transmit_idx)
            assert LB._code(ref) is g  # cached on the reference object
        for kind, m in (("qam", 2), ("qam", 6), ("psk", 3)):
            c = linksim.mapping.Constellation(kind, m)
            assert np.array_equal(LB._const(c).points, c.points)
        pcm = linksim.ldpc.LdpcCode5G(256, 512).pcm
        gp = LB._pcm(pcm)
        assert (gp.n, gp.m, gp.num_edges) == (pcm.n, pcm.m, sum(len(a) for a in pcm.row_adj))
    finally:
        restore()
    for m, n in LB.patched_names():
        assert getattr(getattr(linksim, m), n) is before[(m, n)]
    with pytest.raises(ValueError):
        LB.enable(linksim, mode="warp")


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["min-sum", "sum-product"])
def test_wrappers_reproduce_reference_run_batch(golden, variant):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2203_11854_b200 as lb

    d = golden("chain_c1")
    k, n, m, B, bg, z = (int(x) for x in d["dims"])
    # stand-ins with the reference's module / attribute names
    fake = types.SimpleNamespace(**{mod: types.SimpleNamespace() for mod in ("sweep", "channel", "mapping",
                                                                              "ldpc", "core")})
    for mod, name in LB.patched_names():
        setattr(getattr(fake, mod), name, None)
    restore = LB.enable(fake)
    code = types.SimpleNamespace(k=k, n=n, base_graph=bg, z=z)
    const = types.SimpleNamespace(kind="qam", num_bits_per_symbol=m, points=lb.Constellation("qam", m).points)

    class Rng:  # RngStream's fields and child rule (core.py:41-44)
        def __init__(self, seed, sid):
            self.seed, self.stream_id = seed, sid

        def child(self, i):
            return Rng(self.seed, (self.stream_id * 0x9E3779B97F4A7C15 + i + 1) & ((1 << 64) - 1))

    rng = Rng(42, (1 << 32) | 1)
    sw, ch = fake.sweep, fake.channel
    no = lb.ebnodb2no(2.0, m, k / n)
    # Pipeline.run_batch (sweep.py:347-364), precision "single"
    payload = sw.binary_source([B, k], rng.child(0))
    x = sw.map_bits(sw.ldpc5g_encode(payload, code), const).astype(np.complex64)
    y = ch.awgn(x, no, rng.child(2))
    llr = sw.demap_app(y, no, const)
    dec = sw.ldpc5g_decode(np.asarray(llr, dtype=np.float32), code, num_iter=20, variant=variant)
    assert np.array_equal(np.packbits(payload, axis=-1), d["payload"])
    assert np.array_equal(y, d["y"])
    assert np.array_equal(np.packbits(dec, axis=-1), d[f"{variant.replace('-', '_')}_decoded"])
    assert sw.count_errors(payload, dec) == lb.count_errors(payload, dec)
    restore()
    assert fake.channel.awgn is None and fake.sweep.map_bits is None
