"""TEST INFRASTRUCTURE ONLY — brute-force statevector ground truth.

Restates /root/reference/pkg/src/mirrorbreak/oracle.py: qubit 0 is the least
significant bit of the amplitude index; bitstrings print qubit 0 leftmost.
"""

from __future__ import annotations

import numpy as np

from .mirror_oracle import unitary_of

MAX_QUBITS = 24


def _apply(psi, g, n):
    """oracle.py:425-435: axis j of the [2]*n tensor is qubit n-1-j."""
    u = unitary_of(g)
    if len(g.qubits) == 1:
        ax = n - 1 - g.qubits[0]
        return np.moveaxis(np.tensordot(u, psi, axes=([1], [ax])), 0, ax)
    a, b = g.qubits
    axes = [n - 1 - a, n - 1 - b]
    out = np.tensordot(u.reshape(2, 2, 2, 2), psi, axes=([2, 3], axes))
    return np.moveaxis(out, [0, 1], axes)


def simulate(n, gates):
    """oracle.py:411-422."""
    if n > MAX_QUBITS:
        raise ValueError("statevector capped at 24 qubits")
    psi = np.zeros(2 ** n, dtype=np.complex128)
    psi[0] = 1.0
    psi = psi.reshape([2] * n)
    for g in gates:
        psi = _apply(psi, g, n)
    return psi.reshape(-1)


def circuit_unitary(n, gates):
    """oracle.py:438-448."""
    dim = 2 ** n
    cols = np.eye(dim, dtype=np.complex128).reshape([2] * n + [dim])
    for g in gates:
        cols = _apply(cols, g, n)
    return cols.reshape(dim, dim)


def bits_of(x, n):
    return "".join("1" if (x >> i) & 1 else "0" for i in range(n))


def index_of(bits):
    return sum(1 << i for i, b in enumerate(bits) if b == "1")


def peak(state):
    """oracle.py:460-465 (lowest index on ties)."""
    pr = np.abs(state) ** 2
    n = int(np.log2(len(state)))
    i = int(np.argmax(pr))
    return bits_of(i, n), float(pr[i])


def tvd(p, q):
    return float(0.5 * np.abs(np.asarray(p, float) - np.asarray(q, float)).sum())


def permute_index(mapping, x):
    y = 0
    for i, m in enumerate(mapping):
        if (x >> i) & 1:
            y |= 1 << m
    return y


def permute_vector(mapping, state):
    """oracle.py:497-502."""
    out = np.empty_like(state)
    for x in range(len(state)):
        out[permute_index(mapping, x)] = state[x]
    return out


def permutation_matrix(mapping):
    dim = 2 ** len(mapping)
    mat = np.zeros((dim, dim), dtype=np.complex128)
    for x in range(dim):
        mat[permute_index(mapping, x), x] = 1.0
    return mat
