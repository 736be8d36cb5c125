"""Drop-in mirror of the AWGN part of linksim.channel (channel.py:24-40).

The noise is drawn on the GPU from a counter-based Philox4x32-10 stream keyed
by the RngStream (seed, stream_id): reproducible for any device count and
statistically equivalent to the reference's numpy ziggurat draws (the
bit-exact ziggurat replica is SURVEY.md 8f item 2).  Fading/TDL/CIR channels
are outside the hot path.
"""
from __future__ import annotations

import numpy as np

from . import _lib as L
from .core import RngStream

_MASK64 = (1 << 64) - 1


def awgn(x, no: float, rng: RngStream, device: bool = False, offset: int = 0):
    """x + CN(0, no) per element (channel.py:33-40); complex64 arithmetic.
    `offset` (even) = index of x's first element in the full stream."""
    if no < 0:
        raise ValueError(f"noise variance must be >= 0, got {no}")
    was_np = not L.is_tensor(x)
    tx = L.to_device(x, "complex64")
    out = L.empty(tx.shape, "complex64")
    L.call("ls_awgn_at", L.ptr(tx), int(offset), tx.numel(), float(no), rng.seed & _MASK64,
           rng.stream_id & _MASK64, L.ptr(out), L.stream_ptr())
    return L.to_host(out) if (was_np and not device) else out


def complex_gaussian(shape, rng: RngStream, variance: float = 1.0, dtype=np.complex64,
                     device: bool = False):
    """Circularly-symmetric complex Gaussian draws (channel.py:24-30)."""
    if np.dtype(dtype) != np.complex64:
        raise ValueError("complex_gaussian: the B200 path produces complex64")
    zeros = L.zeros(tuple(int(s) for s in np.atleast_1d(shape)), "complex64")
    return awgn(zeros, variance, rng, device=True) if device else L.to_host(
        awgn(zeros, variance, rng, device=True))
