"""Drop-in mirror of the AWGN part of linksim.channel (channel.py:24-40).

Two noise generators, both on the GPU and both keyed by the RngStream:
  * noise="numpy" (default): a bit-exact replica of the reference's draws --
    numpy's Philox4x64-10 stream fed through numpy 2.3.5's 256-level ziggurat
    (SURVEY.md A3/A4), resolved in parallel despite the data-dependent word
    consumption (csrc/rng_normal.cu).  awgn() returns exactly the reference's
    complex64 output.
  * noise="philox": counter-based Philox4x32-10 + Box-Muller, addressable
    per element (chunkable, fusable with the mapper/demapper); statistically
    equivalent.  The sweep engine's fast mode uses it.
Fading/TDL/CIR channels are outside the hot path.
"""
from __future__ import annotations

import numpy as np

from . import _lib as L
from .core import RngStream

_MASK64 = (1 << 64) - 1
NOISE_KINDS = ("numpy", "philox")


def awgn(x, no: float, rng: RngStream, device: bool = False, offset: int = 0, noise: str = "numpy"):
    """x + CN(0, no) per element (channel.py:33-40) in x's precision: the
    noise is cast to x.dtype as the reference does, so complex64 input gets
    complex64 arithmetic and complex128 input (precision "double") f64.
    `offset` (even, philox noise only) = index of x's first element in the
    full stream."""
    if no < 0:
        raise ValueError(f"noise variance must be >= 0, got {no}")
    if noise not in NOISE_KINDS:
        raise ValueError(f"unknown noise generator {noise!r}")
    was_np = not L.is_tensor(x)
    c128 = (x.dtype == L.torch().complex128) if L.is_tensor(x) else (np.asarray(x).dtype == np.complex128)
    if c128:
        if noise != "numpy" or offset:
            raise ValueError("awgn: complex128 input takes the numpy-exact noise of the whole array")
        tx = L.to_device(x, "complex128")
        out = L.empty(tx.shape, "complex128")
        L.call("ls_awgn_numpy64", L.ptr(tx), tx.numel(), float(no), rng.seed & _MASK64, rng.stream_id & _MASK64,
               L.ptr(out), L.stream_ptr())
        return L.to_host(out) if (was_np and not device) else out
    tx = L.to_device(x, "complex64")
    out = L.empty(tx.shape, "complex64")
    if noise == "numpy":
        if offset:
            raise ValueError("awgn: the numpy-exact stream is drawn for the whole array (offset=0)")
        L.call("ls_awgn_numpy", L.ptr(tx), tx.numel(), float(no), rng.seed & _MASK64,
               rng.stream_id & _MASK64, L.ptr(out), L.stream_ptr())
    else:
        L.call("ls_awgn_at", L.ptr(tx), int(offset), tx.numel(), float(no), rng.seed & _MASK64,
               rng.stream_id & _MASK64, L.ptr(out), L.stream_ptr())
    return L.to_host(out) if (was_np and not device) else out


def standard_normal(count: int, rng: RngStream, device: bool = False):
    """`count` draws of rng.generator().standard_normal (f64), bit-exact."""
    out = L.empty((int(count),), "float64")
    L.call("ls_standard_normal", rng.seed & _MASK64, rng.stream_id & _MASK64, int(count), L.ptr(out),
           L.stream_ptr())
    return out if device else L.to_host(out)


def complex_gaussian(shape, rng: RngStream, variance: float = 1.0, dtype=np.complex128,
                     device: bool = False, noise: str = "numpy"):
    """Circularly-symmetric complex Gaussian draws (channel.py:24-30),
    complex128 by default as in the reference, or complex64."""
    dt = np.dtype(dtype)
    if dt not in (np.complex64, np.complex128):
        raise ValueError("complex_gaussian: dtype must be complex64 or complex128")
    zeros = L.zeros(tuple(int(s) for s in np.atleast_1d(shape)), str(dt))
    z = awgn(zeros, variance, rng, device=True, noise=noise)
    return z if device else L.to_host(z)
