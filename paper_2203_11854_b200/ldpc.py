"""Drop-in mirror of linksim.ldpc (ldpc.py:1-365) on the B200 path.

* `LdpcCode5G(k, n)` selects base graph / lifting size / rate matching
  exactly as the reference (ldpc.py:214-272) and owns an ls_code handle.
* `ldpc5g_encode` runs the QC encoder kernel.
* `bp_decode` runs the EXACT-mode GPU decoder on any ParityCheckMatrix:
  bit-identical to the reference for min-sum / scaled-min-sum, and the
  reference's precision pattern for sum-product (LLRs within tolerance).
  On a lifted 5G code's pcm the min-sum variants take the on-chip QC exact
  decoder (bp_qc_exact.cuh), anything else the HBM-streaming CSR engine.
* `ldpc5g_decode(..., mode="exact")` (default) is derate_match + exact BP
  (fused into the on-chip decoder for min-sum on f32 LLRs); `mode="fast"`
  is the on-chip QC decoder fused with rate matching, hard decision and
  error counting: fp16x2 by default ("auto"; two codewords per 32-bit lane,
  dead extension rows pruned), or precision "fp32-full" (f32 messages, all
  rows) / "fp32" (legacy f32 kernel) -- statistically equivalent, hard
  decisions identical on every block that converges.
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib as L
from .alist import ParityCheckMatrix
from .basegraph import base_graph

BP_VARIANTS = ("sum-product", "min-sum", "scaled-min-sum")
_VARIANT_ID = {v: i for i, v in enumerate(BP_VARIANTS)}

_LIFT_BASES = (2, 3, 5, 7, 9, 11, 13, 15)
LIFTING_SIZES = sorted({a * (1 << j) for a in _LIFT_BASES for j in range(8) if a * (1 << j) <= 384})


def _base(bg: int):
    ent, mb, nb, kb = base_graph(bg)
    return {(int(r), int(c)): int(s) for r, c, s in ent}, mb, nb, kb


class _CodeHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h and L._lib is not None:
                L._lib.ls_code_destroy(self.h)
        except Exception:  # pragma: no cover
            pass


class LdpcCode5G:
    """5G-style lifted LDPC code with rate matching (ldpc.py:214-345)."""

    def __init__(self, k: int, n: int, *, base_graph: int | None = None, z: int | None = None):
        self.k, self.n = int(k), int(n)
        if self.k < 1 or self.n <= self.k:
            raise ValueError(f"unsupported (k={self.k}, n={self.n}): need 0 < k < n")
        # BG2 iff k <= 292, smallest Z with k_b*Z >= k (ldpc.py:232-238).  The
        # keyword overrides lift any graph at any Z for the decoder-only sweep
        # (BG2 with Z >= 32 is unreachable otherwise).
        self.base_graph = base_graph if base_graph is not None else (2 if self.k <= 292 else 1)
        entries, mb, nb, kb = _base(self.base_graph)
        if self.k > kb * 384:
            raise ValueError(f"k={self.k} too large for both base graphs")
        if z is None:
            z = next((zz for zz in LIFTING_SIZES if kb * zz >= self.k), None)
            if z is None:
                raise ValueError(f"no lifting size supports k={self.k}")
        elif kb * z < self.k:
            raise ValueError(f"lifting size {z} too small for k={self.k}")
        self.z = int(z)
        self._entries = entries
        self._mb, self._nb, self._kb = mb, nb, kb
        Z = self.z
        self.k_full, self.n_full, self.m_full = kb * Z, nb * Z, mb * Z
        self.num_fillers = self.k_full - self.k
        self.filler_idx = np.arange(self.k, self.k_full)
        keep = np.ones(self.n_full, dtype=bool)
        keep[self.filler_idx] = False
        keep[: 2 * Z] = False
        buffer = np.flatnonzero(keep)
        self.transmit_idx = buffer[np.arange(self.n) % len(buffer)]
        self._ext_parity = [(r, c - kb, s % Z) for (r, c), s in entries.items()
                            if kb <= c < kb + 4 and r >= 4]
        self._pcm = None
        self._handle = None

    @property
    def coderate(self) -> float:
        return self.k / self.n

    # ------------------------------------------------------------ device handle
    @property
    def handle(self):
        if self._handle is None:
            ent = np.array(sorted((r, c, s) for (r, c), s in self._entries.items()), dtype=np.int32)
            h = ctypes.c_void_p()
            L.call("ls_code_create", self.base_graph, self.z, self.k, self.n, self._mb, self._nb,
                   self._kb, ent.ctypes.data, len(ent), ctypes.byref(h))
            self._handle = _CodeHandle(h)
        return self._handle.h

    @property
    def pcm(self) -> ParityCheckMatrix:
        """Lifted mother-code matrix: CN r*Z+i <-> VN c*Z+(i+s)%Z (ldpc.py:278-296)."""
        if self._pcm is None:
            Z = self.z
            i = np.arange(Z)
            rows, cols = [], []
            for (r, c), s in self._entries.items():
                rows.append(r * Z + i)
                cols.append(c * Z + (i + s) % Z)
            rows = np.concatenate(rows)
            cols = np.concatenate(cols)
            order = np.lexsort((cols, rows))
            rows, cols = rows[order], cols[order]
            ptr = np.zeros(self.m_full + 1, np.int64)
            ptr[1:] = np.cumsum(np.bincount(rows, minlength=self.m_full))
            self._pcm = ParityCheckMatrix._trusted(self.n_full, self.m_full, ptr, cols)
            # lets bp_decode(llr, code.pcm) take the on-chip QC exact decoder
            self._pcm._qc_code = weakref.ref(self)
        return self._pcm

    # ------------------------------------------------------------ encoder
    def encode_full(self, bits, device: bool = False):
        """Mother codeword [batch, n_full] (ldpc.py:298-333)."""
        return _encode(bits, self, full=True, device=device)

    def derate_match(self, llr, device: bool = False):
        """Rate-matched LLRs -> mother positions (ldpc.py:335-345)."""
        was_np = not L.is_tensor(llr)
        t = L.to_device(llr)
        if t.dim() == 1:
            t = t.unsqueeze(0)
        torch = L.torch()
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if t.shape[-1] != self.n:
            raise ValueError(f"expected {self.n} LLRs, got {t.shape[-1]}")
        out = L.empty((t.shape[0], self.n_full), "float64" if t.dtype == torch.float64 else "float32")
        L.call("ls_derate", self.handle, L.ptr(t), int(t.dtype == torch.float64), t.shape[0],
               L.ptr(out), L.stream_ptr())
        return L.to_host(out) if (was_np and not device) else out


def _encode(bits, code: LdpcCode5G, full: bool, device: bool):
    was_np = not L.is_tensor(bits)
    t = L.to_device(bits, "uint8")
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.shape[-1] != code.k:
        raise ValueError(f"expected {code.k} info bits, got {t.shape[-1]}")
    B = t.shape[0]
    out = L.empty((B, code.n_full if full else code.n), "uint8")
    L.call("ls_encode", code.handle, L.ptr(t), B, None if full else L.ptr(out),
           L.ptr(out) if full else None, L.stream_ptr())
    return L.to_host(out) if (was_np and not device) else out


def ldpc5g_encode(bits, code: LdpcCode5G, device: bool = False):
    """[batch, k] info bits -> rate-matched [batch, n] (ldpc.py:348-351)."""
    return _encode(bits, code, full=False, device=device)


def _check_variant(variant: str, num_iter: int):
    if variant not in BP_VARIANTS:
        raise ValueError(f"unknown BP variant {variant!r}")
    if num_iter < 1:
        raise ValueError("num_iter must be >= 1")


def _qc_exact_code(pcm, variant: str, dtype):
    """The LdpcCode5G behind `pcm` when the on-chip exact QC decoder serves
    this call (min-sum / scaled-min-sum on f32 LLRs), else None."""
    ref = getattr(pcm, "_qc_code", None)
    code = ref() if ref is not None else None
    if code is None or variant == "sum-product" or dtype != L.torch().float32:
        return None
    return code if qc_has_kernel(code, precision="exact") else None


def bp_decode(llr, pcm: ParityCheckMatrix, num_iter: int = 20, variant: str = "sum-product",
              scale: float = 0.75, early_stop: bool = True, *, return_iters: bool = False,
              device: bool = False, engine: str = "auto"):
    """Flooding BP (ldpc.py:86-172), exact mode, on the GPU.

    Returns (llr_out, hard) [batch, n] like the reference; with
    return_iters=True also the per-row iteration counts.

    engine: "qc" is the on-chip decoder of a lifted 5G code's pcm
    (bp_qc_exact.cuh; min-sum / scaled-min-sum on f32 LLRs), "csr" the
    HBM-streaming decoder for any ParityCheckMatrix (bp_exact.cu); "auto"
    takes "qc" when it serves the call.  Both are bit-identical to the
    reference.
    """
    _check_variant(variant, num_iter)
    was_np = not L.is_tensor(llr)
    torch = L.torch()
    t = L.to_device(llr)
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    if t.shape[-1] != pcm.n:
        raise ValueError(f"LLR length {t.shape[-1]} does not match n={pcm.n}")
    B = t.shape[0]
    if engine not in ("auto", "qc", "csr"):
        raise ValueError(f"unknown bp_decode engine {engine!r}")
    code = _qc_exact_code(pcm, variant, t.dtype) if engine != "csr" else None
    if engine == "qc" and code is None:
        raise ValueError("bp_decode: the on-chip QC exact decoder does not serve this call")
    if code is not None:
        r = qc_decode(t, code, num_iter, variant, scale, early_stop=early_stop, want_llr=True,
                      want_iters=True, precision="exact", mother=True)
        out, hard, iters = r["llr"], r["hard"], r["iters"]
        if was_np and not device:
            res = (L.to_host(out), L.to_host(hard))
            return res + (L.to_host(iters),) if return_iters else res
        return (out, hard, iters) if return_iters else (out, hard)
    is64 = t.dtype == torch.float64
    out = L.empty((B, pcm.n), "float64" if is64 else "float32")
    hard = L.empty((B, pcm.n), "uint8")
    iters = L.empty((B,), "int32")
    L.call("ls_bp_decode", pcm.device_graph(), L.ptr(t), int(is64), B, int(num_iter), _VARIANT_ID[variant],
           float(scale), int(bool(early_stop)), L.ptr(out), L.ptr(hard), L.ptr(iters), L.stream_ptr())
    if was_np and not device:
        res = (L.to_host(out), L.to_host(hard))
        return res + (L.to_host(iters),) if return_iters else res
    return (out, hard, iters) if return_iters else (out, hard)


def ldpc5g_decode(llr, code: LdpcCode5G, num_iter: int = 20, variant: str = "sum-product",
                  scale: float = 0.75, *, mode: str = "exact", early_stop: bool = True,
                  device: bool = False, precision: str = "auto"):
    """BP-decode rate-matched LLRs -> [batch, k] info bits (ldpc.py:354-365)."""
    _check_variant(variant, num_iter)
    if mode == "exact":
        f32_in = (llr.dtype == L.torch().float32) if L.is_tensor(llr) else (np.asarray(llr).dtype == np.float32)
        if f32_in and variant != "sum-product" and qc_has_kernel(code, precision="exact"):
            # on-chip exact decoder with derate_match fused in
            host_in = not L.is_tensor(llr) or not llr.is_cuda
            if host_in and not device:
                return _decode_host_pipelined(llr, code, num_iter, variant, scale, early_stop, "exact")
            t = L.to_device(llr)
            if t.dim() == 1:
                t = t.unsqueeze(0)
            out = qc_decode(t, code, num_iter, variant, scale, early_stop=early_stop,
                            precision="exact")["hard"]
            return L.to_host(out) if (not L.is_tensor(llr) and not device) else out
        mother = code.derate_match(llr, device=True)
        _, hard = bp_decode(mother, code.pcm, num_iter, variant, scale, early_stop, device=True)
        out = hard[:, : code.k].contiguous()
        return L.to_host(out) if (not L.is_tensor(llr) and not device) else out
    if mode != "fast":
        raise ValueError(f"unknown decoder mode {mode!r}")
    if precision == "auto":
        precision = "fp16x2"  # specialised instance, else the runtime-geometry fp16x2 kernel
    host_in = not L.is_tensor(llr) or not llr.is_cuda
    if host_in and not device:
        return _decode_host_pipelined(llr, code, num_iter, variant, scale, early_stop, precision)
    res = qc_decode(llr, code, num_iter, variant, scale, early_stop=early_stop, precision=precision)
    return L.to_host(res["hard"]) if (not L.is_tensor(llr) and not device) else res["hard"]


def _decode_host_pipelined(llr, code, num_iter, variant, scale, early_stop, precision, chunk=2048):
    """Host LLRs [B, n] -> host bits [B, k]: row chunks copied in on a copy
    stream, decoded on the compute stream and copied out, so the PCIe
    transfers overlap the decoder.  Small chunks keep the un-overlapped tail
    (the last chunk's decode) short: on a B200 the 65,536-codeword config-2
    batch runs at 6.5 Gbit/s with 2,048-row chunks against 6.0 with 8,192,
    close to the 55.6 GB/s pinned H2D ceiling (tools/prof_hostdecode.py)."""
    torch = L.torch()
    src = llr if L.is_tensor(llr) else torch.from_numpy(np.ascontiguousarray(np.asarray(llr, np.float32)))
    if src.dtype != torch.float32:
        src = src.to(torch.float32)
    if src.dim() == 1:
        src = src.unsqueeze(0)
    if src.shape[-1] != code.n:
        raise ValueError(f"expected {code.n} LLRs, got {src.shape[-1]}")
    B = src.shape[0]
    out = torch.empty((B, code.k), dtype=torch.uint8, pin_memory=True)
    main = torch.cuda.current_stream()
    h2d, d2h = L.side_stream("h2d"), L.side_stream("d2h")
    dev = L.device()
    for lo in range(0, B, chunk):
        hi = min(B, lo + chunk)
        with torch.cuda.stream(h2d):
            x = src[lo:hi].to(dev, non_blocking=True)
        main.wait_stream(h2d)
        x.record_stream(main)
        hard = qc_decode(x, code, num_iter, variant, scale, early_stop=early_stop, precision=precision)["hard"]
        d2h.wait_stream(main)
        with torch.cuda.stream(d2h):
            out[lo:hi].copy_(hard, non_blocking=True)
        hard.record_stream(d2h)
    d2h.synchronize()
    return out.numpy() if not L.is_tensor(llr) else out


LS_QC_PRUNE, LS_QC_GENERIC, LS_QC_FP16, LS_QC_SP, LS_QC_EXACT, LS_QC_MOTHER, LS_QC_FULL32 = 1, 2, 4, 8, 16, 32, 64


def qc_has_kernel(code: LdpcCode5G, precision: str = "fp32", prune: bool = True,
                  variant: str = "min-sum") -> bool:
    """Whether a compile-time specialised fast decoder exists for this code
    (the sum-product fast decoder exists only as such instances; min-sum codes
    without one run the runtime-geometry fp16x2 or the runtime-Z fp32 kernel).
    precision "exact" asks for the on-chip exact decoder (min-sum variants)."""
    if precision == "exact":
        return variant != "sum-product" and bool(L.lib().ls_qc_has_kernel(code.handle, LS_QC_EXACT))
    if precision == "fp32-full":
        sp = LS_QC_SP | (LS_QC_PRUNE if prune else 0) if variant == "sum-product" else 0
        return bool(L.lib().ls_qc_has_kernel(code.handle, LS_QC_FULL32 | sp))
    flags = (LS_QC_PRUNE if prune else 0) | (LS_QC_FP16 if precision == "fp16x2" else 0)
    if variant == "sum-product":
        flags |= LS_QC_SP
    return bool(L.lib().ls_qc_has_kernel(code.handle, flags))


def qc_decode(llr, code: LdpcCode5G, num_iter: int = 20, variant: str = "min-sum", scale: float = 0.75,
              *, early_stop: bool = True, ref_bits=None, want_hard: bool = True, want_llr: bool = False,
              want_iters: bool = False, counts=None, prune: bool | None = None, generic: bool = False,
              precision: str = "fp32", mother: bool = False):
    """Fast-mode fused decoder: rate-matched f32 LLRs [B, n] on the device ->
    dict(hard [B,k] uint8, llr [B,n_full] f32 mother LLRs, iters [B] int32,
    counts [2] int64 (bit, block) errors vs ref_bits), each only if asked.

    prune (default: on unless mother LLRs are requested) skips the dead
    extension rows whose parity bit is never transmitted.  precision
    "fp16x2" selects the packed two-codewords-per-lane kernel.  generic forces
    the runtime-geometry kernel of that precision instead of a compile-time
    specialised instance.  precision "exact" is the on-chip bit-exact decoder
    (bp_qc_exact.cuh: whole mother graph, reference arithmetic; min-sum and
    scaled-min-sum) and "fp32-full" the same decoder with f32 messages (fast
    mode, all rows); with mother=True the input is mother LLRs [B, n_full]
    and `hard` covers all n_full positions (bp_decode on code.pcm)."""
    if precision not in ("fp32", "fp16x2", "exact", "fp32-full"):
        raise ValueError(f"unknown decoder precision {precision!r}")
    if mother and precision not in ("exact", "fp32-full"):
        raise ValueError("mother-length input needs precision='exact' or 'fp32-full'")
    if precision == "exact" or (precision == "fp32-full" and variant != "sum-product"):
        prune = False
    elif prune is None:
        # f32 sum-product messages fit in shared memory only with the dead rows pruned
        prune = (not want_llr) or (precision == "fp32-full" and variant == "sum-product")
    flags = ((LS_QC_PRUNE if prune else 0) | (LS_QC_GENERIC if generic else 0)
             | (LS_QC_FP16 if precision == "fp16x2" else 0) | (LS_QC_EXACT if precision == "exact" else 0)
             | (LS_QC_FULL32 if precision == "fp32-full" else 0) | (LS_QC_MOTHER if mother else 0))
    _check_variant(variant, num_iter)
    t = L.to_device(llr, "float32")
    if t.dim() == 1:
        t = t.unsqueeze(0)
    n_in = code.n_full if mother else code.n
    if t.shape[-1] != n_in:
        raise ValueError(f"expected {n_in} LLRs, got {t.shape[-1]}")
    B = t.shape[0]
    res = {}
    hard = L.empty((B, code.n_full if mother else code.k), "uint8") if want_hard else None
    lo = L.empty((B, code.n_full), "float32") if want_llr else None
    it = L.empty((B,), "int32") if want_iters else None
    ref = L.to_device(ref_bits, "uint8") if ref_bits is not None else None
    if ref is not None and counts is None:
        counts = L.zeros((2,), "int64")
    L.call("ls_qc_decode", code.handle, L.ptr(t), B, int(num_iter), _VARIANT_ID[variant], float(scale),
           int(bool(early_stop)), flags, L.ptr(hard), L.ptr(lo), L.ptr(it), L.ptr(ref), L.ptr(counts),
           L.stream_ptr())
    res.update(hard=hard, llr=lo, iters=it, counts=counts)
    return res


def exit_mutual_information(llr, bits) -> float:
    """I = 1 - E[log2(1 + exp(-(2b-1) L))] clipped to [0, 1] (ldpc.py:175-188),
    f64 on the GPU (k_mi_partial / k_mi_final)."""
    tl = L.to_device(llr, "float64").contiguous()
    tb = L.to_device(bits, "float64").contiguous()
    if tl.numel() == 0:
        raise ValueError("exit_mutual_information: empty input")
    if tuple(tl.shape) != tuple(tb.shape):
        raise ValueError("exit_mutual_information: shape mismatch")
    out = L.empty((1,), "float64")
    L.call("ls_exit_mutual_information", L.ptr(tl), L.ptr(tb), tl.numel(), L.ptr(out), L.stream_ptr())
    return float(out.cpu()[0])
