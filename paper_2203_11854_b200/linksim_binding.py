"""The binding a linksim maintainer would add: route an installed reference
package's hot path through the B200 library.

The reference has no operator registry; its Pipeline resolves the block
functions by name at call time:
  * ldpc5g_encode, ldpc5g_decode, binary_source, map_bits, hard_decide and
    count_errors through `linksim.sweep` globals (sweep.py:24-26, 325-364,
    438-453);
  * awgn through the `linksim.channel` module object (`ch.awgn`, sweep.py:355);
  * the demapper through `sweep.demap_app` / `sweep.demap_maxlog`, bound to
    `self.demap` when a Pipeline is CONSTRUCTED (sweep.py:179), so enable()
    must run before the Pipeline is built;
  * bp_decode / exit_mutual_information through `linksim.ldpc`.

    import linksim
    from paper_2203_11854_b200 import linksim_binding
    restore = linksim_binding.enable(linksim)        # exact mode: bit-identical
    res = linksim.sweep.run_sweep(cfg, num_workers=8)
    restore()

Every wrapper keeps the reference's argument meaning, dtypes (complex64 /
complex128 symbols, f32 / f64 LLRs: precision "double" stays f64) and
ValueErrors; handles (codes, constellations, graphs) are built once per
reference object and cached on it, the way the reference caches
`pcm._edge_graph` (ldpc.py:57-62).
"""
from __future__ import annotations

import numpy as np

from . import channel as _ch
from . import core as _core
from . import ldpc as _ldpc
from . import mapping as _map
from .alist import ParityCheckMatrix as _Pcm

# (module attribute, name) pairs enable() replaces; the same list restores them
_TARGETS = (
    ("sweep", "ldpc5g_encode"), ("sweep", "ldpc5g_decode"), ("sweep", "binary_source"),
    ("sweep", "map_bits"), ("sweep", "demap_app"), ("sweep", "demap_maxlog"),
    ("sweep", "hard_decide"), ("sweep", "count_errors"),
    ("channel", "awgn"),
    ("mapping", "map_bits"), ("mapping", "demap_app"), ("mapping", "demap_maxlog"),
    ("ldpc", "ldpc5g_encode"), ("ldpc", "ldpc5g_decode"), ("ldpc", "bp_decode"),
    ("ldpc", "exit_mutual_information"),
    ("core", "binary_source"), ("core", "hard_decide"), ("core", "count_errors"),
)


def _rng(rng):
    return _core.RngStream(rng.seed, rng.stream_id)


def _code(code):
    """Reference LdpcCode5G -> B200 code (same base graph, Z and rate matching)."""
    g = getattr(code, "_b200_code", None)
    if g is None:
        g = _ldpc.LdpcCode5G(code.k, code.n)
        if (g.base_graph, g.z) != (code.base_graph, code.z):  # pragma: no cover - defensive
            raise ValueError("B200 code selection differs from the reference's")
        code._b200_code = g
    return g


def _const(c):
    g = getattr(c, "_b200_const", None)
    if g is None:
        if c.kind in ("qam", "psk"):
            g = _map.Constellation(c.kind, c.num_bits_per_symbol)
        else:  # custom points: already normalised by the reference object
            g = _map.Constellation("custom", c.num_bits_per_symbol, points=np.asarray(c.points),
                                   normalized=False)
        if not np.array_equal(g.points, np.asarray(c.points)):
            raise ValueError("B200 constellation points differ from the reference's")
        c._b200_const = g
    return g


def _pcm(pcm):
    g = getattr(pcm, "_b200_pcm", None)
    if g is None:
        g = _Pcm(pcm.n, pcm.m, [np.asarray(a) for a in pcm.col_adj], [np.asarray(a) for a in pcm.row_adj])
        pcm._b200_pcm = g
    return g


def _wrappers(mode: str):
    def ldpc5g_encode(bits, code):
        return _ldpc.ldpc5g_encode(bits, _code(code))

    def ldpc5g_decode(llr, code, num_iter=20, variant="sum-product", scale=0.75):
        # f32 or f64 LLRs as given (precision "double" decodes in f64)
        return _ldpc.ldpc5g_decode(llr, _code(code), num_iter, variant, scale, mode=mode)

    def binary_source(shape, rng):
        return _core.binary_source(shape, _rng(rng))

    def map_bits(bits, constellation):
        # the reference returns the f64 points; run_batch casts them (sweep.py:352)
        return _map.map_bits(bits, _const(constellation), dtype="complex128")

    def demap_app(y, no, constellation, prior=None):
        return _map.demap_app(y, no, _const(constellation), prior)

    def demap_maxlog(y, no, constellation, prior=None):
        return _map.demap_maxlog(y, no, _const(constellation), prior)

    def awgn(x, no, rng):
        return _ch.awgn(x, no, _rng(rng))

    def bp_decode(llr, pcm, num_iter=20, variant="sum-product", scale=0.75, early_stop=True):
        return _ldpc.bp_decode(llr, _pcm(pcm), num_iter, variant, scale, early_stop)

    return {
        "ldpc5g_encode": ldpc5g_encode, "ldpc5g_decode": ldpc5g_decode, "binary_source": binary_source,
        "map_bits": map_bits, "demap_app": demap_app, "demap_maxlog": demap_maxlog, "awgn": awgn,
        "bp_decode": bp_decode, "hard_decide": _core.hard_decide, "count_errors": _core.count_errors,
        "exit_mutual_information": _ldpc.exit_mutual_information,
    }


def enable(linksim, mode: str = "exact"):
    """Patch the reference package `linksim` (its sweep, channel, mapping,
    ldpc and core modules) to run on the B200 library; returns a function
    that restores the original functions.  mode "exact" is bit-identical to
    the reference (min-sum variants) / within tolerance (sum-product);
    "fast" uses the on-chip fast decoders (statistically equivalent)."""
    if mode not in ("exact", "fast"):
        raise ValueError(f"unknown mode {mode!r}")
    wrap = _wrappers(mode)
    saved = []
    for modname, name in _TARGETS:
        mod = getattr(linksim, modname)
        if hasattr(mod, name):
            saved.append((mod, name, getattr(mod, name)))
            setattr(mod, name, wrap[name])

    def restore():
        for mod, name, fn in reversed(saved):
            setattr(mod, name, fn)

    return restore


def patched_names():
    """The (module, function) pairs enable() replaces."""
    return list(_TARGETS)
