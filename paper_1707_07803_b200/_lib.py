"""ctypes binding of the sm_100a C-ABI library (include/mpo_b200.h).

This is the only way the package reaches the device: there is no CPU
fallback.  If ``lib/libmpo_b200.so`` is missing or no CUDA device is
visible, every compute entry point raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MPO_B200_LIB: alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("MPO_B200_LIB") or os.path.join(HERE, "lib", "libmpo_b200.so")

MPO_OK, MPO_EVALUE, MPO_ECUDA, MPO_ENOMEM, MPO_EINTERNAL = range(5)

_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_DP = C.POINTER(C.c_double)

# name -> (restype, argtypes); mirrors include/mpo_b200.h one to one
SIGNATURES = {
    "mpo_b200_last_error": (C.c_char_p, []),
    "mpo_b200_abi_version": (C.c_int, []),
    "mpo_b200_launch_count": (C.c_ulonglong, []),
    "mpo_b200_round_paths": (C.c_int, [C.POINTER(C.c_ulonglong)]),
    "mpo_b200_profile_enable": (C.c_int, [C.c_int]),
    "mpo_b200_profile_read": (C.c_int, [C.c_int, _DP, _DP, C.POINTER(C.c_ulonglong)]),
    "mpo_ctx_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "mpo_ctx_set_stream": (C.c_int, [_P, _P]),
    "mpo_ctx_synchronize": (C.c_int, [_P]),
    "mpo_ctx_destroy": (C.c_int, [_P]),
    "mpo_dev_create": (C.c_int, [_P, C.c_int, _I64P, C.POINTER(_P), C.c_int, C.POINTER(_P)]),
    "mpo_dev_create_packed": (C.c_int, [_P, C.c_int, _I64P, _P, C.c_int, C.POINTER(_P)]),
    "mpo_dev_copy_all": (C.c_int, [_P, _P, _P, C.c_int]),
    "mpo_dev_num_cores": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "mpo_dev_shapes": (C.c_int, [_P, _I64P]),
    "mpo_dev_core_ptr": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "mpo_dev_copy_core": (C.c_int, [_P, _P, C.c_int, _P, C.c_int]),
    "mpo_dev_free": (C.c_int, [_P]),
    "mpo_matmul": (C.c_int, [_P, _P, C.c_int, _P, C.c_int, C.POINTER(_P)]),
    "mpo_transpose": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "mpo_merge_leading_cores": (C.c_int, [_P, _P, C.c_int, C.POINTER(_P)]),
    "mpo_qr": (C.c_int, [_P, _P, C.c_double, C.c_int, C.POINTER(_P), _DP]),
    "mpo_svd": (C.c_int, [_P, _P, C.c_double, C.c_int, _DP, _DP, C.POINTER(_P)]),
    "mpo_subspace_iteration": (C.c_int, [_P, _P, _P, C.c_int, C.c_double, C.c_int,
                                         C.POINTER(_P)]),
    "mpo_tnrsvd": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_double, C.c_int,
                             C.POINTER(_P), _DP, C.POINTER(_P)]),
    "mpo_round": (C.c_int, [_P, _P, C.c_double, C.POINTER(_P)]),
    "mpo_add": (C.c_int, [_P, _P, _P, C.POINTER(_P)]),
    "mpo_sparse_convert": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int, C.c_int, _I64P,
                                     _I64P, C.POINTER(_P)]),
    "mpo_conv_info": (C.c_int, [_P, _I64P, _I64P]),
    "mpo_conv_copy": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, C.c_int]),
    "mpo_conv_ptrs": (C.c_int, [_P, _P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                C.POINTER(_P), C.POINTER(_P)]),
    "mpo_conv_level": (C.c_int, [_P, _P, C.c_int, _P, _P, C.c_int]),
    "mpo_conv_dense_core": (C.c_int, [_P, _P, C.c_int, _P, C.c_int]),
    "mpo_conv_chunk": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.POINTER(_P)]),
    "mpo_conv_free": (C.c_int, [_P]),
    "mpo_keys_unique": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, _I64P]),
    "mpo_keys_lookup": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P]),
    "mpo_keys_search": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int64, C.c_int, _P]),
    "mpo_remap_ids": (C.c_int, [_P, _P, _P, C.c_int64]),
    "mpo_dense_qr": (C.c_int, [_P, C.c_int64, C.c_int64, _P, C.c_int64, _P, C.c_int64, _P,
                               C.c_int64]),
    "mpo_dense_svd": (C.c_int, [_P, C.c_int64, C.c_int64, _P, C.c_int64, _P, _P, C.c_int64, _P,
                                C.c_int64]),
    "mpo_dense_gemm": (C.c_int, [_P, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                 C.c_double, _P, C.c_int64, _P, C.c_int64, C.c_double, _P,
                                 C.c_int64]),
}

_lib = None
_lock = threading.Lock()
_ctx = {}


def load():
    """Load the library (no device needed); raise if it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"CUDA library {LIB_PATH} is missing: build it with `make` "
                        "(or __graft_entry__.build()); there is no CPU fallback")
                lib = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


def check(code: int):
    if code == MPO_OK:
        return
    msg = load().mpo_b200_last_error().decode("utf-8", "replace")
    if code == MPO_EVALUE:
        raise ValueError(msg)
    if code == MPO_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"mpo_b200: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def context(device: int | None = None):
    """Per-(device, stream) context; the stream is torch's current stream
    when torch is loaded with CUDA, else the legacy default stream."""
    stream = None
    dev = 0 if device is None else int(device)
    try:
        import torch  # plumbing only: streams
        if torch.cuda.is_available():
            if device is None:
                dev = torch.cuda.current_device()
            stream = torch.cuda.current_stream(dev).cuda_stream
    except ImportError:  # pragma: no cover
        pass
    key = (dev, stream)
    ctx = _ctx.get(key)
    if ctx is None:
        h = C.c_void_p()
        call("mpo_ctx_create", dev, C.c_void_p(stream), C.byref(h))
        ctx = h
        _ctx[key] = ctx
    return ctx


def launch_count() -> int:
    return int(load().mpo_b200_launch_count())


def round_paths() -> dict:
    """Counts of the truncation-step rounding paths taken so far."""
    out = (C.c_ulonglong * 5)()
    call("mpo_b200_round_paths", out)
    return dict(zip(("cert", "cert_tall", "tail", "tail_tall", "svd"), (int(x) for x in out)))


def host_empty(shape, dtype=np.float64, order="C"):
    """Host array for a download.  Backed by page-locked memory from torch's
    caching host allocator when CUDA is up (the D2H copy runs at full link
    speed and the pages are recycled across calls instead of faulted in
    afresh); plain numpy for small arrays or without CUDA."""
    shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    n = int(np.prod(shape)) if shape else 1
    try:
        import torch  # plumbing only: the pinned host allocator
        if n >= (1 << 16) and torch.cuda.is_available():
            tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64}[np.dtype(dtype)]
            return torch.empty(n, dtype=tdt, pin_memory=True).numpy().reshape(shape, order=order)
    except (ImportError, KeyError):  # pragma: no cover
        pass
    return np.empty(shape, dtype=dtype, order=order)


def as_i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)
