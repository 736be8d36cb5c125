"""ctypes binding of liblinksim_b200.so (include/linksim_b200.h) and the
torch plumbing the Python mirror uses for device buffers and streams.

There is no CPU fallback: if the library or a CUDA device is missing, every
array entry point raises.  PyTorch provides only device memory, streams and
host<->device copies; all arithmetic of the hot path runs in the library.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liblinksim_b200.so")

LS_OK, LS_EINVAL, LS_ECUDA, LS_ENOMEM = 0, 1, 2, 3

_lock = threading.Lock()
_lib = None

c_i32p = ctypes.POINTER(ctypes.c_int32)
_vp, _i64, _u64, _int, _dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double

# name -> argtypes (all return int status)
_SIGS = {
    "ls_version": [],
    "ls_code_create": [_int, _int, _int, _int, _int, _int, _int, _vp, _int, _vp],
    "ls_code_destroy": [_vp],
    "ls_code_transmit_idx": [_vp, _vp],
    "ls_graph_create": [_i64, _i64, _vp, _vp, _vp],
    "ls_graph_from_code": [_vp, _vp],
    "ls_graph_destroy": [_vp],
    "ls_binary_source": [_u64, _u64, _i64, _vp, _vp],
    "ls_map_bits": [_vp, _i64, _int, _vp, _vp, _vp],
    "ls_map_bits64": [_vp, _i64, _int, _vp, _vp, _vp],
    "ls_awgn_numpy64": [_vp, _i64, _dbl, _u64, _u64, _vp, _vp],
    "ls_demap64": [_vp, _i64, _dbl, _vp, _vp, _vp, _int, _int, _vp, _vp, _vp],
    "ls_demap_qam64": [_vp, _i64, _dbl, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp, _vp],
    "ls_awgn": [_vp, _i64, _dbl, _u64, _u64, _vp, _vp],
    "ls_demap": [_vp, _i64, _dbl, _vp, _vp, _vp, _int, _int, _vp, _vp, _vp],
    "ls_demap_qam": [_vp, _i64, _dbl, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp, _vp],
    "ls_modem_qam": [_vp, _i64, _int, _vp, _vp, _vp, _dbl, _u64, _u64, _int, _vp, _vp],
    "ls_binary_source_at": [_u64, _u64, _i64, _i64, _vp, _vp],
    "ls_standard_normal": [_u64, _u64, _i64, _vp, _vp],
    "ls_awgn_numpy": [_vp, _i64, _dbl, _u64, _u64, _vp, _vp],
    "ls_awgn_at": [_vp, _i64, _i64, _dbl, _u64, _u64, _vp, _vp],
    "ls_modem_qam_at": [_vp, _i64, _i64, _int, _vp, _vp, _vp, _dbl, _u64, _u64, _int, _vp, _vp],
    "ls_encode": [_vp, _vp, _i64, _vp, _vp, _vp],
    "ls_derate": [_vp, _vp, _int, _i64, _vp, _vp],
    "ls_bp_decode": [_vp, _vp, _int, _i64, _int, _int, _dbl, _int, _vp, _vp, _vp, _vp],
    "ls_qc_decode": [_vp, _vp, _i64, _int, _int, _dbl, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp],
    "ls_qc_live_rows": [_vp],
    "ls_qc_has_kernel": [_vp, _int],
    "ls_count_errors": [_vp, _vp, _i64, _i64, _vp, _vp],
    "ls_hard_decide": [_vp, _int, _i64, _vp, _vp],
    "ls_exit_mutual_information": [_vp, _vp, _i64, _vp, _vp],
}


class CudaPathError(RuntimeError):
    """The B200 CUDA path is unavailable (library not built or no GPU)."""


def lib():
    """Load liblinksim_b200.so once; raise loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaPathError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2203_11854_b200._build` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = ctypes.c_int
            L.ls_last_error.argtypes = []
            L.ls_last_error.restype = ctypes.c_char_p
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == LS_OK:
        return
    msg = (lib().ls_last_error() or b"").decode()
    if rc == LS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"linksim_b200 error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


# ---------------------------------------------------------------- torch plumbing
def torch():
    import torch as _t

    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise CudaPathError("no CUDA device: the linksim_b200 hot path runs on the GPU only")
    lib()
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


_NP2T = {np.dtype(np.uint8): "uint8", np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
         np.dtype(np.complex64): "complex64", np.dtype(np.complex128): "complex128",
         np.dtype(np.int32): "int32", np.dtype(np.int64): "int64"}


def is_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


def to_device(x, dtype=None):
    """numpy/array-like or tensor -> contiguous CUDA tensor of `dtype`.

    Host tensors are copied as they are (asynchronously when pinned) and
    converted on the device; numpy arrays are converted on the host (never
    widening the transfer) and copied from pageable memory -- pinning a fresh
    staging buffer per call costs more than it saves.
    """
    t = torch()
    dev = device()
    if is_tensor(x):
        y = x
        if y.device != dev:
            y = y.to(dev, non_blocking=True)
        if dtype is not None and y.dtype != getattr(t, dtype):
            y = y.to(getattr(t, dtype))
        return y.contiguous()
    a = np.asarray(x)
    if dtype is not None:
        a = a.astype(dtype, copy=False)
    return t.from_numpy(np.ascontiguousarray(a)).to(dev)


_side_streams: dict = {}


def side_stream(name: str):
    """A long-lived side stream per (device, name).  Reusing it across calls
    keeps the caching allocator's per-stream blocks reusable (a fresh stream
    per call would strand them and force new device allocations)."""
    t = torch()
    key = (t.cuda.current_device(), name)
    st = _side_streams.get(key)
    if st is None:
        with _lock:
            st = _side_streams.get(key)
            if st is None:
                st = _side_streams[key] = t.cuda.Stream()
    return st


def to_host(t):
    """CUDA tensor -> numpy (synchronising on the current stream)."""
    return t.cpu().numpy()


def empty(shape, dtype: str):
    t = torch()
    return t.empty(tuple(int(s) for s in shape), dtype=getattr(t, dtype), device=device())


def zeros(shape, dtype: str):
    t = torch()
    return t.zeros(tuple(int(s) for s in shape), dtype=getattr(t, dtype), device=device())
