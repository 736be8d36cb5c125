"""Drop-in mirror of linksim.core (core.py:1-104) on the B200 path.

Same names, arguments, conventions and errors as the reference.  Array work
(bit generation, error counting, hard decisions) runs in liblinksim_b200;
functions taking arrays accept numpy arrays or CUDA tensors and return the
same kind they were given (numpy in -> numpy out).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L

LLR_MAX = 40.0  # core.py:18, LLR convention ln(p1/p0), ties decide 0

_MASK64 = (1 << 64) - 1
_STREAM_MIX = 0x9E3779B97F4A7C15  # core.py:22


@dataclass(frozen=True)
class RngStream:
    """Counter-based stream (seed, stream_id) (core.py:25-44).

    The GPU kernels key numpy's Philox4x64-10 exactly as the reference does
    (key = [stream_id, seed], counter from 1), so binary_source draws are
    bit-identical to the reference's.
    """

    seed: int
    stream_id: int = 0

    def generator(self) -> np.random.Generator:
        """The reference's host generator for this stream (for host-side draws)."""
        key = ((self.seed & _MASK64) << 64) | (self.stream_id & _MASK64)
        return np.random.Generator(np.random.Philox(key=key))

    def child(self, index: int) -> "RngStream":
        mixed = ((self.stream_id * _STREAM_MIX) + index + 1) & _MASK64
        return RngStream(self.seed, mixed)


def _shape(shape):
    shape = tuple(int(s) for s in np.atleast_1d(np.asarray(shape, dtype=np.int64)))
    if len(shape) == 0:
        raise ValueError("binary_source: shape must not be empty")
    if any(s < 1 for s in shape):
        raise ValueError(f"binary_source: all dimensions must be >= 1, got {shape}")
    return shape


def binary_source(shape, rng: RngStream, device: bool = False, offset: int = 0):
    """i.i.d. bits (core.py:47-54), bit-exact with the reference's draws.

    Returns numpy uint8 like the reference; `device=True` returns the CUDA
    tensor instead (no host copy).  `offset` (a multiple of 32) starts the
    draw at that bit of the stream, for row chunks of a larger batch.
    """
    shape = _shape(shape)
    out = L.empty(shape, "uint8")
    L.call("ls_binary_source_at", rng.seed & _MASK64, rng.stream_id & _MASK64, int(offset), out.numel(),
           L.ptr(out), L.stream_ptr())
    return out if device else L.to_host(out)


def ebnodb2no(ebno_db: float, bits_per_symbol: int, coderate: float) -> float:
    """core.py:57-68 (scalar host arithmetic, no array work)."""
    if bits_per_symbol < 1:
        raise ValueError("ebnodb2no: bits_per_symbol must be >= 1")
    if not 0.0 < coderate <= 1.0:
        raise ValueError(f"ebnodb2no: coderate must be in (0, 1], got {coderate}")
    ebno = 10.0 ** (float(ebno_db) / 10.0)
    return 1.0 / (ebno * coderate * bits_per_symbol)


def _pair(b, b_hat, name):
    tb, th = L.to_device(b, "uint8"), L.to_device(b_hat, "uint8")
    if tuple(tb.shape) != tuple(th.shape):
        raise ValueError(f"{name}: shape mismatch {tuple(tb.shape)} vs {tuple(th.shape)}")
    return tb, th


def _counts(tb, th):
    counts = L.zeros((2,), "int64")
    rows = tb.shape[0] if tb.dim() else 1
    per = tb.numel() // max(rows, 1)
    L.call("ls_count_errors", L.ptr(tb), L.ptr(th), rows, per, L.ptr(counts), L.stream_ptr())
    c = counts.cpu().tolist()
    return int(c[0]), int(c[1]), rows, tb.numel()


def count_errors(b, b_hat) -> tuple[int, int]:
    """(bit errors, block errors) (core.py:93-99)."""
    tb, th = _pair(b, b_hat, "count_errors")
    bits, blocks, _, _ = _counts(tb, th)
    return bits, blocks


def compute_ber(b, b_hat) -> float:
    """core.py:76-81."""
    tb, th = _pair(b, b_hat, "compute_ber")
    bits, _, _, total = _counts(tb, th)
    return float(bits / total) if total else float("nan")


def compute_bler(b, b_hat) -> float:
    """core.py:84-90."""
    tb, th = _pair(b, b_hat, "compute_bler")
    _, blocks, rows, _ = _counts(tb, th)
    return float(blocks / rows) if rows else float("nan")


def hard_decide(llr):
    """1 iff L > 0 (core.py:102-104): ties and -0.0 decide 0 (k_hard)."""
    was_np = not L.is_tensor(llr)
    torch = L.torch()
    t = L.to_device(llr)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    t = t.contiguous()
    out = L.empty(tuple(t.shape), "uint8")
    L.call("ls_hard_decide", L.ptr(t), int(t.dtype == torch.float64), t.numel(), L.ptr(out), L.stream_ptr())
    return L.to_host(out) if was_np else out
