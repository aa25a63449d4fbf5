"""ctypes binding of the C ABI in include/mirrorbreak_b200.h.

The library is built in-tree (``paper_2604_21908_b200/_lib``) by
``__graft_entry__.build()``. There is no fallback: if the library is missing
or no CUDA device is usable, every chain operation raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libmirrorbreak_b200.so"

MB_C128, MB_C64 = 0, 1
SIDE = {"left": 0, "right": 1, "both": 2}
DTYPES = {"complex128": MB_C128, "complex64": MB_C64}


class NativeError(RuntimeError):
    """A call into libmirrorbreak_b200 failed (message from mb_last_error)."""


_lib = None
_ready = False

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)

_SIGS = {
    "mb_last_error": (C.c_char_p, []),
    "mb_version": (_i, []),
    "mb_init": (_i, [_i]),
    "mb_stream": (_p, []),
    "mb_synchronize": (_i, []),
    "mb_launch_count": (C.c_longlong, []),
    "mb_profile_begin": (_i, []),
    "mb_profile_end": (_i, [_dp, C.POINTER(C.c_longlong), _dp]),
    "mb_counters": (_i, [C.POINTER(C.c_longlong)]),
    "mb_identity_mpo": (_p, [_i, _i]),
    "mb_chain_from_host": (_p, [_i, _i, _i, _i64p, _dp, _d, _i]),
    "mb_chain_clone": (_p, [_p]),
    "mb_chain_free": (None, [_p]),
    "mb_chain_info": (_i, [_p, _ip, _ip, _ip, _dp, _ip]),
    "mb_chain_bonds": (_i, [_p, _i64p]),
    "mb_total_elements": (_i64, [_p]),
    "mb_chain_to_host": (_i, [_p, _dp]),
    "mb_absorb_1q": (_i, [_p, _i, _dp, _i]),
    "mb_absorb_2q": (_i, [_p, _i, _dp, _i, _d, _i64]),
    "mb_move_center": (_i, [_p, _i]),
    "mb_pair_swap": (_i, [_p, _i, _i, _i, _d, _i64, _i]),
    "mb_swap_extents": (_i, [_p, _i, _i, _ip, _d, _i64, _i64p]),
    "mb_batch_swap_extents": (_i, [_p, _i, _ip, _ip, _i, _d, _i64, _i64p, _i64p]),
    "mb_compress": (_i, [_p, _d, _i64]),
    "mb_try_bond": (_i, [_p, _i, _i, _ip, _d, _i64, _i, _i64p, _i64p, _ip]),
    "mb_try_bond_run": (_i, [_p, _i, _ip, _i, _d, _i64, _i, _ip, _i64p, _i64p]),
    "mb_trial": (_i, [_p, _i, _ip, _ip, _dp, _i, _d, _i64]),
    "mb_trial_pair": (_i, [_p, _i, _ip, _ip, _dp, _i, _ip, _ip, _dp, _d, _i64,
                           C.POINTER(_p), C.POINTER(_p)]),
    "mb_frobenius_norm": (_i, [_p, _dp]),
    "mb_apply_to_zero": (_p, [_p, _d, _i64]),
    "mb_peak": (_i, [_p, _u8p, _dp]),
    "mb_sample": (_i, [_p, _i64, _dp, _u8p]),
    "mb_svd_truncate": (_i, [_dp, _i64, _i64, _i, _d, _i64, _dp, _dp, _dp, _i64p, _dp]),
    "mb_herm_eig": (_i, [_dp, _i64, _dp, _dp]),
    "mb_debug_fail_svd": (_i, [_i]),
    "mb_profile_eig": (_i, [_dp, _i64p, _dp, _dp]),
    "mb_gemm": (_i, [_dp, _dp, _i64, _i64, _i64, _i, _i, _dp]),
}


def exported_symbols():
    """Names every binding expects (checked against include/*.h by the tests)."""
    return tuple(_SIGS)


def load(init: bool = True):
    """Load the library (and initialize the device unless init=False)."""
    global _lib, _ready
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"CUDA library missing at {LIB_PATH}; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if init and not _ready:
        # one process per GPU: bind the rank's local device
        dev = int(os.environ.get("MB_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        rc = _lib.mb_init(dev)
        if rc != 0:
            raise NativeError(f"mb_init failed: {_lib.mb_last_error().decode()}")
        _ready = True
    return _lib


class SvdConvergenceError(NativeError):
    """The SVD failed even after a perturbed retry (the reference's
    tensor.SvdConvergenceError, tensor.py:26)."""


ERR_NUMERIC = -3


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = f"{what}: {_lib.mb_last_error().decode()}"
        if rc == ERR_NUMERIC and "converge" in msg:
            raise SvdConvergenceError(msg)
        raise NativeError(msg)


def handle(h, what: str):
    if not h:
        raise NativeError(f"{what}: {_lib.mb_last_error().decode()}")
    return h


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def u8ptr(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def complex_buffer(a) -> np.ndarray:
    """Contiguous complex128 view suitable for a double* argument."""
    return np.ascontiguousarray(a, dtype=np.complex128)


def launch_count() -> int:
    return int(load().mb_launch_count())


def counters() -> dict:
    out = (C.c_longlong * 8)()
    load().mb_counters(out)
    keys = ("svd_small", "svd_large", "large_sweeps", "host_syncs", "svd_not_converged", "max_p",
            "h2d_bytes", "d2h_bytes")
    return dict(zip(keys, (int(x) for x in out)))


PROFILE_CLASSES = ("gemm", "gate", "svd_small", "svd_large", "emit", "other", "svd_jacobi")


def profile_begin() -> None:
    check(load().mb_profile_begin(), "mb_profile_begin")


def profile_end() -> dict:
    ms = (C.c_double * 7)()
    n = (C.c_longlong * 7)()
    fl = (C.c_double * 7)()
    check(load().mb_profile_end(ms, n, fl), "mb_profile_end")
    return {k: {"ms": ms[i], "launch_groups": int(n[i]), "flops": fl[i]}
            for i, k in enumerate(PROFILE_CLASSES)}


EIG_STAGES = ("gram", "trd_panel", "trd_symv", "trd_update", "dc", "backtransform", "xv")


def profile_eig() -> dict:
    """Per-stage device time, launches, algorithmic bytes and flops of the
    large-SVD Gram path over the last profiled region (mb_profile_eig)."""
    ms = (C.c_double * 7)()
    n = (C.c_longlong * 7)()
    by = (C.c_double * 7)()
    fl = (C.c_double * 7)()
    check(load().mb_profile_eig(ms, n, by, fl), "mb_profile_eig")
    return {k: {"ms": ms[i], "launches": int(n[i]), "bytes": by[i], "flops": fl[i]}
            for i, k in enumerate(EIG_STAGES)}


def stream_handle() -> int:
    return int(load().mb_stream() or 0)


def synchronize() -> None:
    check(load().mb_synchronize(), "mb_synchronize")
