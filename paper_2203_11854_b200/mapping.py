"""Drop-in mirror of linksim.mapping (mapping.py:1-158) on the B200 path.

`Constellation` is the same host-side table (Gray QAM / PSK, unit energy).
`map_bits` and the demappers run in liblinksim_b200; inputs may be numpy
arrays or CUDA tensors and outputs follow the input kind.  As in the
reference, demapper output is float64 (cast to f32 by the sweep engine).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


def _gray_to_index(g: np.ndarray) -> np.ndarray:
    i = g.copy()
    sh = 1
    while sh < 64:
        i ^= i >> sh
        sh <<= 1
    return i


def _bit_table(m: int) -> np.ndarray:
    """[2^m, m] label bits, MSB first (mapping.py:27-31)."""
    lab = np.arange(1 << m)
    return ((lab[:, None] >> np.arange(m - 1, -1, -1)[None, :]) & 1).astype(np.uint8)


def _qam(m: int) -> np.ndarray:
    # even label bits drive I, odd bits Q, per-axis Gray, label 0 = most
    # positive level (mapping.py:33-48)
    if m % 2:
        raise ValueError("qam requires an even number of bits per symbol")
    half = m // 2
    bits = _bit_table(m).astype(np.int64)
    w = 1 << np.arange(half - 1, -1, -1)
    li = _gray_to_index(bits[:, 0::2] @ w)
    lq = _gray_to_index(bits[:, 1::2] @ w)
    top = (1 << half) - 1
    return (top - 2 * li).astype(np.complex128) + 1j * (top - 2 * lq).astype(np.complex128)


def _psk(m: int) -> np.ndarray:
    order = 1 << m
    idx = _gray_to_index(np.arange(order, dtype=np.int64))
    return np.exp(2j * np.pi * idx / order)


@dataclass
class Constellation:
    """Ordered complex points indexed by bit label (mapping.py:58-93)."""

    kind: str
    num_bits_per_symbol: int
    points: np.ndarray = field(default=None)
    normalized: bool = True

    def __post_init__(self):
        m = self.num_bits_per_symbol
        if m < 1:
            raise ValueError("num_bits_per_symbol must be >= 1")
        if self.points is None:
            if self.kind == "qam":
                self.points = _qam(m)
            elif self.kind == "psk":
                self.points = _psk(m)
            else:
                raise ValueError(f"unknown constellation kind {self.kind!r}")
        else:
            if self.kind not in ("qam", "psk"):
                self.kind = "custom"
            self.points = np.asarray(self.points, dtype=np.complex128)
        if self.points.shape != (1 << m,):
            raise ValueError(f"expected {1 << m} points, got shape {self.points.shape}")
        if self.normalized:
            self.points = self.points / np.sqrt(np.mean(np.abs(self.points) ** 2))
        self._bits = _bit_table(m)
        self._dev = {}

    @property
    def bit_table(self) -> np.ndarray:
        return self._bits

    def qam_axes(self):
        """(amp, lab) per-axis level tables if the points are the library's Gray
        QAM (product of two Gray PAM axes), else None."""
        if getattr(self, "_axes", 0) != 0:
            return self._axes
        self._axes = None
        m = self.num_bits_per_symbol
        if self.kind == "qam" and m % 2 == 0 and m <= 8:
            half = m // 2
            L = 1 << half
            idx = np.arange(L)
            lab = (idx ^ (idx >> 1)).astype(np.int32)       # Gray label of level idx
            w = 1 << np.arange(half - 1, -1, -1)
            bits = self._bits.astype(np.int64)
            lab_i, lab_q = bits[:, 0::2] @ w, bits[:, 1::2] @ w
            amp = np.empty(L)
            ok = True
            for l in range(L):
                pts = self.points[(lab_i == lab[l])]
                amp[l] = pts[0].real
                ok &= np.all(pts.real == amp[l]) and np.all(self.points[lab_q == lab[l]].imag == amp[l])
            if ok:
                self._axes = (np.ascontiguousarray(amp), np.ascontiguousarray(lab))
        return self._axes

    def device_points(self, dtype: str):
        """Points on the GPU as interleaved float32 (complex64-rounded) or float64."""
        if dtype not in self._dev:
            if dtype == "float32":
                host = self.points.astype(np.complex64).view(np.float32)
            else:
                host = self.points.astype(np.complex128).view(np.float64)
            self._dev[dtype] = L.to_device(np.ascontiguousarray(host))
        return self._dev[dtype]


def map_bits(bits, constellation: Constellation, device: bool = False, dtype: str = "complex64"):
    """Big-endian m-bit groups -> points (mapping.py:96-107).

    dtype "complex64" folds in the sweep engine's `astype(complex64)`
    (sweep.py:352, precision "single"); "complex128" keeps the f64 points
    (precision "double").  numpy in -> numpy out unless device=True.
    """
    if dtype not in ("complex64", "complex128"):
        raise ValueError(f"map_bits: unsupported dtype {dtype!r}")
    was_np = not L.is_tensor(bits)
    m = constellation.num_bits_per_symbol
    tb = L.to_device(bits, "uint8")
    if tb.shape[-1] % m != 0:
        raise ValueError(f"bit count {tb.shape[-1]} not divisible by {m} bits/symbol")
    out = L.empty(tuple(tb.shape[:-1]) + (tb.shape[-1] // m,), dtype)
    if dtype == "complex64":
        L.call("ls_map_bits", L.ptr(tb), out.numel(), m, L.ptr(constellation.device_points("float32")),
               L.ptr(out), L.stream_ptr())
    else:
        L.call("ls_map_bits64", L.ptr(tb), out.numel(), m, L.ptr(constellation.device_points("float64")),
               L.ptr(out), L.stream_ptr())
    return L.to_host(out) if (was_np and not device) else out


def _demap(y, no, constellation: Constellation, prior, mode: int, out_dtype: str, device: bool):
    was_np = not L.is_tensor(y)
    c128 = (y.dtype == L.torch().complex128) if L.is_tensor(y) else (np.asarray(y).dtype == np.complex128)
    ty = L.to_device(y, "complex128" if c128 else "complex64")
    m = constellation.num_bits_per_symbol
    tp = None
    if prior is not None:
        # flat prior [m] or one per bit position, broadcastable to [..., S, m]
        # (mapping.py:123-131), laid out per symbol for the kernels
        tp = L.to_device(prior, "float64")
        if tuple(tp.shape) == (m,):
            tp = tp.expand(tuple(ty.shape) + (m,))
        else:
            tp = tp.reshape(tuple(ty.shape) + (m,))
        tp = tp.contiguous()
    no_arr = np.asarray(no, dtype=np.float64) if not L.is_tensor(no) else None
    no_vec = None
    if no_arr is not None and no_arr.ndim == 0:
        if not float(no_arr) > 0:
            raise ValueError("demap: noise variance must be > 0")
        no_s = float(no_arr)
    else:
        tn = L.to_device(no, "float64")
        if bool((tn <= 0).any()):
            raise ValueError("demap: noise variance must be > 0")
        no_vec = tn.expand(ty.shape).contiguous()
        no_s = 1.0
    out = L.empty(tuple(ty.shape[:-1]) + (ty.shape[-1] * m,), out_dtype)
    is64 = out_dtype == "float64"
    axes = constellation.qam_axes()
    if axes is not None:
        amp, lab = axes
        L.call("ls_demap_qam64" if c128 else "ls_demap_qam", L.ptr(ty), ty.numel(), no_s, L.ptr(no_vec),
               L.ptr(tp), amp.ctypes.data,
               lab.ctypes.data, m, mode, None if is64 else L.ptr(out), L.ptr(out) if is64 else None,
               L.stream_ptr())
        return L.to_host(out) if (was_np and not device) else out
    L.call("ls_demap64" if c128 else "ls_demap", L.ptr(ty), ty.numel(), no_s, L.ptr(no_vec), L.ptr(tp),
           L.ptr(constellation.device_points("float64")), m, mode,
           None if is64 else L.ptr(out), L.ptr(out) if is64 else None, L.stream_ptr())
    return L.to_host(out) if (was_np and not device) else out


def modem_qam(coded, constellation: Constellation, no: float, rng, demapper: str = "app", offset: int = 0):
    """Fused map_bits -> awgn -> demap (f32 LLRs, device) for Gray QAM: the
    Pipeline's fast chain (sweep.py:352-356 in one pass).  The noisy symbols
    equal map_bits + awgn with the same stream; the LLRs are computed in f32."""
    axes = constellation.qam_axes()
    if axes is None:
        raise ValueError("modem_qam needs a Gray QAM constellation")
    if demapper not in ("app", "maxlog"):
        raise ValueError(f"unknown demapper {demapper!r}")
    if not no > 0:
        raise ValueError("demap: noise variance must be > 0")
    m = constellation.num_bits_per_symbol
    tb = L.to_device(coded, "uint8")
    if tb.shape[-1] % m != 0:
        raise ValueError(f"bit count {tb.shape[-1]} not divisible by {m} bits/symbol")
    amp, lab = axes
    out = L.empty(tuple(tb.shape), "float32")
    L.call("ls_modem_qam_at", L.ptr(tb), int(offset), tb.numel() // m, m,
           L.ptr(constellation.device_points("float32")),
           amp.ctypes.data, lab.ctypes.data, float(no), rng.seed & ((1 << 64) - 1),
           rng.stream_id & ((1 << 64) - 1), 0 if demapper == "app" else 1, L.ptr(out), L.stream_ptr())
    return out


def demap_app(y, no, constellation: Constellation, prior=None, out_dtype: str = "float64",
              device: bool = False):
    """Exact APP LLRs ln(p1/p0) (mapping.py:146-153), f64 arithmetic on GPU."""
    return _demap(y, no, constellation, prior, 0, out_dtype, device)


def demap_maxlog(y, no, constellation: Constellation, prior=None, out_dtype: str = "float64",
                 device: bool = False):
    """Max-log approximation (mapping.py:156-158)."""
    return _demap(y, no, constellation, prior, 1, out_dtype, device)
