"""TEST INFRASTRUCTURE ONLY -- CPU parity oracle for the linksim hot path.

A restatement of the reference's (linksim 0.1.0, /root/reference/pkg/src)
coded-link chain, used as the *checker* for the CUDA product:

    binary_source -> ldpc5g_encode -> map_bits -> awgn -> demap_app|maxlog
      -> derate_match -> bp_decode -> count_errors

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  The product package never
does, and never falls back to it.

Pinning: every function here is checked against the golden vectors minted
from the reference itself (tests/golden/make_goldens.py -> tests/golden/*.npz,
see tests/test_oracle_golden.py).  Where the reference's arithmetic lives in
third-party code the restatement names it:
  * numpy 2.3.5 Philox4x64-10 / bounded uint8 draw -> oracle/c/oracle.c
  * numpy 2.3.5 Generator.standard_normal (256-level ziggurat) -> called
    through numpy itself here (same pinned version on the GPU box image) and
    restated bit-exactly in C (oracle/c/oracle.c, orc_standard_normal;
    SURVEY.md A3), both pinned to the reference's draws in tests/golden/rng.npz.
  * scipy 1.18.1 special.logsumexp -> restated in `_lse` below.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

LLR_MAX = 40.0  # core.py:18
MASK64 = (1 << 64) - 1
STREAM_MIX = 0x9E3779B97F4A7C15  # core.py:22
VARIANTS = {"sum-product": 0, "min-sum": 1, "scaled-min-sum": 2}  # ldpc.py:23

_HERE = os.path.dirname(os.path.abspath(__file__))
_GOLDEN = os.path.join(os.path.dirname(_HERE), "tests", "golden")


# ---------------------------------------------------------------- C library
@lru_cache(maxsize=None)
def lib():
    path = os.path.join(_HERE, "_build", "liboracle.so")
    src = os.path.join(_HERE, "c", "oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    L = ctypes.CDLL(path)
    u64, i64, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
    L.orc_philox_raw.argtypes = [u64, u64, u64, i64, vp]
    L.orc_binary_source.argtypes = [u64, u64, i64, vp]
    L.orc_bp_decode.argtypes = [vp, ctypes.c_int, i64, i64, i64, vp, vp, ctypes.c_int,
                                ctypes.c_int, ctypes.c_double, ctypes.c_int, vp, vp, vp]
    L.orc_bp_decode.restype = ctypes.c_int
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- RNG (core.py)
def child_stream(stream_id: int, index: int) -> int:
    """RngStream.child (core.py:41-44)."""
    return ((stream_id * STREAM_MIX) + index + 1) & MASK64


def philox_raw(seed: int, stream_id: int, count: int, first_word: int = 0) -> np.ndarray:
    out = np.empty(count, np.uint64)
    lib().orc_philox_raw(seed & MASK64, stream_id & MASK64, first_word, count, _p(out))
    return out


def binary_source(shape, seed: int, stream_id: int) -> np.ndarray:
    """binary_source (core.py:47-54) via the Philox/Lemire restatement."""
    shape = tuple(int(s) for s in np.atleast_1d(shape))
    out = np.empty(int(np.prod(shape)), np.uint8)
    lib().orc_binary_source(seed & MASK64, stream_id & MASK64, out.size, _p(out))
    return out.reshape(shape)


def standard_normal_pair(shape, seed: int, stream_id: int):
    """The two standard_normal(shape) calls of complex_gaussian (channel.py:27-29).

    Third-party: numpy 2.3.5 ziggurat, called through numpy itself.
    """
    key = ((seed & MASK64) << 64) | (stream_id & MASK64)
    g = np.random.Generator(np.random.Philox(key=key))
    re = g.standard_normal(shape)
    im = g.standard_normal(shape)
    return re, im


def hard_decide(llr):
    """core.py:102-104: 1 iff L > 0."""
    return (np.asarray(llr) > 0).astype(np.uint8)


def exit_mutual_information(llr, bits) -> float:
    """ldpc.py:175-188 restated: 1 - mean(log2(1 + exp(clip(-(2b-1)L, +-40)))),
    clipped to [0, 1]."""
    llr = np.asarray(llr, dtype=np.float64)
    bits = np.asarray(bits)
    if llr.size == 0:
        raise ValueError("exit_mutual_information: empty input")
    if llr.shape != bits.shape:
        raise ValueError("exit_mutual_information: shape mismatch")
    x = np.clip(-(2.0 * bits - 1.0) * llr, -LLR_MAX, LLR_MAX)
    return float(np.clip(1.0 - np.mean(np.log2(1.0 + np.exp(x))), 0.0, 1.0))


def ebnodb2no(ebno_db: float, m: int, coderate: float) -> float:
    """core.py:57-68."""
    return 1.0 / (10.0 ** (float(ebno_db) / 10.0) * coderate * m)


def count_errors(b, b_hat):
    """core.py:93-99: (bit errors, block errors)."""
    d = (np.asarray(b) != np.asarray(b_hat)).reshape(np.asarray(b).shape[0], -1)
    return int(d.sum()), int(d.any(axis=1).sum())


# ---------------------------------------------------------------- base graphs / codes
LIFTING_SIZES = sorted({a << j for a in (2, 3, 5, 7, 9, 11, 13, 15) for j in range(8)
                        if (a << j) <= 384})  # ldpc.py:25-29


@lru_cache(maxsize=None)
def base_graph(bg: int):
    """(entries [nnz,3] sorted by (r,c), m_b, n_b, k_b) from the golden copy of the
    reference's data/ldpc_bg{1,2}.txt (ldpc.py:191-211)."""
    z = np.load(os.path.join(_GOLDEN, "base_graphs.npz"))
    mb, nb, kb = (int(x) for x in z[f"bg{bg}_dims"])
    return z[f"bg{bg}"].astype(np.int64), mb, nb, kb


class Code:
    """LdpcCode5G restated (ldpc.py:214-345)."""

    def __init__(self, k: int, n: int, bg: int | None = None, z: int | None = None):
        if k < 1 or n <= k:
            raise ValueError(f"unsupported (k={k}, n={n}): need 0 < k < n")
        self.k, self.n = k, n
        self.bg = bg if bg is not None else (2 if k <= 292 else 1)
        ent, self.mb, self.nb, self.kb = base_graph(self.bg)
        self.z = z if z is not None else next(zz for zz in LIFTING_SIZES if self.kb * zz >= k)
        Z = self.z
        self.entries = ent
        self.k_full, self.n_full, self.m_full = self.kb * Z, self.nb * Z, self.mb * Z
        self.filler_idx = np.arange(k, self.k_full)
        keep = np.ones(self.n_full, bool)
        keep[self.filler_idx] = False
        keep[: 2 * Z] = False
        buf = np.flatnonzero(keep)
        self.transmit_idx = buf[np.arange(n) % len(buf)]

    @property
    def csr(self):
        """Check-major CSR of the lifted graph: CN r*Z+i <-> VN c*Z+(i+s)%Z."""
        Z = self.z
        rows = [[] for _ in range(self.m_full)]
        i = np.arange(Z)
        for r, c, s in self.entries:
            vs = c * Z + (i + s) % Z
            for ii in range(Z):
                rows[r * Z + ii].append(int(vs[ii]))
        ptr = np.zeros(self.m_full + 1, np.int64)
        ptr[1:] = np.cumsum([len(x) for x in rows])
        var = np.fromiter((v for x in rows for v in sorted(x)), np.int64, count=int(ptr[-1]))
        return ptr, var

    def encode_full(self, bits: np.ndarray) -> np.ndarray:
        """GF(2) encode by rolled-block XORs (restates ldpc.py:298-333 without the GEMM)."""
        bits = np.atleast_2d(np.asarray(bits, np.uint8))
        B, Z, kb = bits.shape[0], self.z, self.kb
        csys = np.zeros((B, self.k_full), np.uint8)
        csys[:, : self.k] = bits
        blk = csys.reshape(B, kb, Z)
        syn = np.zeros((B, self.mb, Z), np.uint8)
        for r, c, s in self.entries:
            if c < kb:
                syn[:, r] ^= np.roll(blk[:, c], -(s % Z), axis=-1)
        tot = syn[:, 0] ^ syn[:, 1] ^ syn[:, 2] ^ syn[:, 3]
        p1 = np.roll(tot, 1, axis=-1)
        p2 = syn[:, 0] ^ tot
        p3 = syn[:, 1] ^ p1 ^ p2
        p4 = syn[:, 2] ^ p3
        core = (p1, p2, p3, p4)
        ext = syn[:, 4:].copy()
        for r, c, s in self.entries:
            if kb <= c < kb + 4 and r >= 4:
                ext[:, r - 4] ^= np.roll(core[c - kb], -(s % Z), axis=-1)
        return np.concatenate([csys, *core, ext.reshape(B, -1)], axis=-1)

    def encode(self, bits):
        return self.encode_full(bits)[:, self.transmit_idx]

    def derate_match(self, llr):
        """ldpc.py:335-345: sequential accumulation from +0.0, fillers -40."""
        llr = np.atleast_2d(np.asarray(llr))
        mother = np.zeros((llr.shape[0], self.n_full), llr.dtype)
        np.add.at(mother, (slice(None), self.transmit_idx), llr)
        mother[:, self.filler_idx] = -LLR_MAX
        return mother


# ---------------------------------------------------------------- mapping (mapping.py)
def qam_points(m: int) -> np.ndarray:
    """Gray QAM, even label bits -> I, odd -> Q, label 0 most positive,
    unit mean energy (mapping.py:33-48, 85-87)."""
    labels = np.arange(1 << m)
    bits = (labels[:, None] >> np.arange(m - 1, -1, -1)) & 1
    na = m // 2
    w = 1 << np.arange(na - 1, -1, -1)

    def gray_inv(g):
        i = g.copy()
        sh = 1
        while sh < 64:
            i ^= i >> sh
            sh *= 2
        return i

    li, lq = gray_inv(bits[:, 0::2] @ w), gray_inv(bits[:, 1::2] @ w)
    M = 1 << na
    pts = ((M - 1) - 2 * li).astype(np.complex128) + 1j * ((M - 1) - 2 * lq)
    return pts / np.sqrt(np.mean(np.abs(pts) ** 2))


def map_bits(bits, points, m):
    """mapping.py:96-107: big-endian m-bit groups index the points."""
    g = np.asarray(bits).reshape(*np.shape(bits)[:-1], -1, m).astype(np.int64)
    return points[g @ (1 << np.arange(m - 1, -1, -1))]


def _lse(a, axis=-1):
    """scipy.special.logsumexp restated: a_max + log1p(sum_{j != argmax} e^(a_j - a_max))."""
    amax = np.max(a, axis=axis, keepdims=True)
    finite = np.isfinite(amax)
    shift = np.where(finite, amax, 0.0)
    e = np.exp(a - shift)
    idx = np.argmax(a, axis=axis)
    e_wo = e.copy()
    np.put_along_axis(e_wo, np.expand_dims(idx, axis), 0.0, axis=axis)
    s = np.sum(e_wo, axis=axis, keepdims=True)
    return np.squeeze(shift + np.log1p(s), axis=axis)


def demap(y, no, points, m, mode="app", prior=None):
    """mapping.py:110-143: LLR ln(p1/p0), f64, optional bit priors."""
    y = np.asarray(y)
    no = np.asarray(no, np.float64)
    if np.any(no <= 0):
        raise ValueError("demap: noise variance must be > 0")
    d2 = np.abs(y[..., None] - points) ** 2
    logits = -d2 / np.broadcast_to(no, y.shape)[..., None]
    lab = (np.arange(1 << m)[:, None] >> np.arange(m - 1, -1, -1)) & 1  # [P, m]
    if prior is not None:  # logit of point p += sum of the priors of its 1-bits
        prior = np.asarray(prior, np.float64)
        if prior.shape != (m,):
            prior = prior.reshape(*y.shape, m)
        logits = logits + prior @ lab.T.astype(np.float64)
    out = np.empty(y.shape + (m,), np.float64)
    for j in range(m):
        one, zero = logits[..., lab[:, j] == 1], logits[..., lab[:, j] == 0]
        if mode == "app":
            out[..., j] = _lse(one) - _lse(zero)
        else:
            out[..., j] = one.max(-1) - zero.max(-1)
    return out.reshape(*y.shape[:-1], -1)


def awgn_single(x_c64, no, seed, stream_id):
    """awgn(x, no, rng) for complex64 x (channel.py:24-40)."""
    if no == 0:
        return x_c64.copy()
    re, im = standard_normal_pair(x_c64.shape, seed, stream_id)
    n = (np.sqrt(no / 2.0) * (re + 1j * im)).astype(np.complex64)
    return x_c64 + n


# ---------------------------------------------------------------- BP (ldpc.py:86-172)
def bp_decode_csr(llr, cptr, cvar, n, num_iter=20, variant="sum-product", scale=0.75,
                  early_stop=True):
    """Exact restatement of bp_decode on a check-major CSR graph.

    Returns (llr_out, hard, iters_used).  Bit-exact vs the reference for the
    min-sum variants; sum-product uses libm tanh/log (the reference uses
    numpy's SIMD versions), so its LLRs agree to a tolerance.
    """
    if variant not in VARIANTS:
        raise ValueError(f"unknown BP variant {variant!r}")
    if num_iter < 1:
        raise ValueError("num_iter must be >= 1")
    llr = np.atleast_2d(np.asarray(llr))
    if llr.dtype not in (np.float32, np.float64):
        llr = llr.astype(np.float64)
    llr = np.ascontiguousarray(llr)
    if llr.shape[-1] != n:
        raise ValueError(f"LLR length {llr.shape[-1]} does not match n={n}")
    B = llr.shape[0]
    out = np.empty_like(llr)
    hard = np.empty(llr.shape, np.uint8)
    iters = np.empty(B, np.int32)
    cptr = np.ascontiguousarray(cptr, np.int64)
    cvar = np.ascontiguousarray(cvar, np.int64)
    lib().orc_bp_decode(_p(llr), int(llr.dtype == np.float64), B, n, len(cptr) - 1, _p(cptr),
                        _p(cvar), num_iter, VARIANTS[variant], float(scale), int(early_stop),
                        _p(out), _p(hard), _p(iters))
    return out, hard, iters


@lru_cache(maxsize=16)
def code(k, n):
    c = Code(k, n)
    c._csr = c.csr
    return c


def decode(llr, c: Code, num_iter=20, variant="sum-product", scale=0.75, early_stop=True):
    """ldpc5g_decode (ldpc.py:354-365) plus the full bp outputs."""
    mother = c.derate_match(llr)
    cptr, cvar = c._csr if hasattr(c, "_csr") else c.csr
    lo, hard, it = bp_decode_csr(mother, cptr, cvar, c.n_full, num_iter, variant, scale,
                                 early_stop)
    return hard[:, : c.k], lo, it


def run_batch(k, n, m, ebno_db, batch, seed, stream_id, variant="sum-product", num_iter=20,
              demapper="app", early_stop=True):
    """Pipeline.run_batch, AWGN + ldpc5g branch, precision 'single'
    (sweep.py:347-364).  Returns (payload, decoded)."""
    c = code(k, n)
    no = ebnodb2no(ebno_db, m, k / n)
    payload = binary_source((batch, k), seed, child_stream(stream_id, 0))
    coded = c.encode(payload)
    pts = qam_points(m)
    x = map_bits(coded, pts, m).astype(np.complex64)
    y = awgn_single(x, no, seed, child_stream(stream_id, 2))
    llr = demap(y, no, pts, m, demapper).astype(np.float32)
    dec, _, _ = decode(llr, c, num_iter, variant, 0.75, early_stop)
    return payload, dec
