"""Truncated SVD on the device (reference tensor.py:84-136).

``svd_truncate`` runs the engine's Jacobi SVD kernels on the matricized
tensor and applies the reference's truncation rule on the device; the host
only receives the kept factors.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C
import numpy as np

from . import _native as nat
from ._native import SvdConvergenceError  # noqa: F401  (reference name, tensor.py:26)

TIE_TOLERANCE = 1e-12


class ZeroTensorError(ValueError):
    """Raised when an SVD is requested for an all-zero tensor."""


@dataclass(frozen=True)
class TruncatedSVD:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    discarded_weight: float

    @property
    def rank(self) -> int:
        return len(self.s)


def truncation_rank(s: np.ndarray, epsilon: float, chi_max: int) -> int:
    """Kept rank of a descending spectrum under the relative cutoff: smallest
    r with discarded squared weight <= eps^2 of the total, grown across ties
    at the boundary, capped at chi_max, at least 1 (tensor.py:119-136). The
    device applies the same rule inside the SVD kernels; this host copy
    serves callers that already hold a spectrum."""
    w = np.asarray(s, dtype=np.float64) ** 2
    budget = epsilon * epsilon * float(w.sum())
    tail = np.concatenate([np.cumsum(w[::-1])[::-1], [0.0]])
    ok = np.nonzero(tail[1:] <= budget)[0]
    r = int(ok[0]) + 1 if len(ok) else len(w)
    edge = s[r - 1]
    while r < len(s) and s[r] >= edge - TIE_TOLERANCE:
        r += 1
    return min(r, chi_max)


def svd_truncate(t: np.ndarray, split: int, epsilon: float, chi_max: int,
                 dtype: str = "complex128") -> TruncatedSVD:
    """Truncated SVD of ``t`` matricized between axes [0:split) and
    [split:), computed by the device kernels (tensor.py:84-116)."""
    t = np.asarray(t, dtype=np.complex128)
    if not (1 <= split < t.ndim):
        raise ValueError(f"split {split} must satisfy 1 <= split < rank {t.ndim}")
    if epsilon < 0:
        raise ValueError("epsilon must be >= 0")
    if chi_max < 1:
        raise ValueError("chi_max must be >= 1")
    if not np.all(np.isfinite(t)):
        raise ValueError("tensor contains non-finite amplitudes")
    rows = int(np.prod(t.shape[:split], dtype=np.int64))
    cols = int(np.prod(t.shape[split:], dtype=np.int64))
    a = np.ascontiguousarray(t.reshape(rows, cols))
    if not np.any(a):
        raise ZeroTensorError("cannot decompose an all-zero tensor")
    lib = nat.load()
    k = min(rows, cols)
    u = np.empty((rows, k), dtype=np.complex128)
    s = np.empty(k, dtype=np.float64)
    v = np.empty((k, cols), dtype=np.complex128)
    rank = C.c_int64()
    disc = C.c_double()
    nat.check(lib.mb_svd_truncate(nat.dptr(a), rows, cols, nat.DTYPES[dtype], float(epsilon),
                                  int(chi_max), nat.dptr(u), nat.dptr(s), nat.dptr(v),
                                  C.byref(rank), C.byref(disc)), "mb_svd_truncate")
    r = rank.value
    # the library wrote u as (rows x r) and v as (r x cols), contiguous
    u_k = u.reshape(-1)[: rows * r].reshape(rows, r).copy()
    v_k = v.reshape(-1)[: r * cols].reshape(r, cols).copy()
    return TruncatedSVD(u=u_k, s=s[:r].copy(), v=v_k, discarded_weight=disc.value)


def device_gemm(a: np.ndarray, b: np.ndarray, dtype: str = "complex64",
                tensor_cores: bool = True) -> np.ndarray:
    """C = A @ B on the device (the pair-blob contraction primitive). With
    dtype complex64 and tensor_cores=True this runs the tcgen05 kind::tf32
    kernel (3xTF32 split); otherwise the CUDA-core tile kernel."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    c = np.empty((m, n), dtype=np.complex128)
    lib = nat.load()
    nat.check(lib.mb_gemm(nat.dptr(a), nat.dptr(b), m, n, k, nat.DTYPES[dtype],
                          int(bool(tensor_cores)), nat.dptr(c)), "mb_gemm")
    return c


def device_herm_eig(a: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Eigen-decomposition of a Hermitian matrix by the engine's large-SVD
    eigensolver (Householder tridiagonalization, divide and conquer,
    back-transformation; mb_eig.cu): (w ascending, V with eigenvector
    columns). The Gram eigenproblem behind svd_truncate's large path."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n, n2 = a.shape
    if n != n2:
        raise ValueError("matrix must be square")
    w = np.empty(n, dtype=np.float64)
    v = np.empty((n, n), dtype=np.complex128)
    lib = nat.load()
    nat.check(lib.mb_herm_eig(nat.dptr(a), n, w.ctypes.data_as(C.POINTER(C.c_double)),
                              nat.dptr(v)), "mb_herm_eig")
    return w, v


def truncated_spectrum(t: np.ndarray, split: int, epsilon: float, chi_max: int,
                       dtype: str = "complex128") -> tuple[np.ndarray, float]:
    """Kept singular values and discarded weight from the values-only device
    decomposition that scores unswap candidates (unswap.py:104-112:
    np.linalg.svd(..., compute_uv=False) + truncation_rank)."""
    t = np.asarray(t, dtype=np.complex128)
    rows = int(np.prod(t.shape[:split], dtype=np.int64))
    cols = int(np.prod(t.shape[split:], dtype=np.int64))
    a = np.ascontiguousarray(t.reshape(rows, cols))
    s = np.empty(min(rows, cols), dtype=np.float64)
    rank = C.c_int64()
    disc = C.c_double()
    lib = nat.load()
    nat.check(lib.mb_svd_truncate(nat.dptr(a), rows, cols, nat.DTYPES[dtype], float(epsilon),
                                  int(chi_max), None, nat.dptr(s), None, C.byref(rank),
                                  C.byref(disc)), "mb_svd_truncate")
    return s[: rank.value].copy(), disc.value
