"""Device-resident matrix product operators and states.

Mirrors /root/reference/pkg/src/mirrorbreak/chains.py. The site tensors live
in HBM inside libmirrorbreak_b200 (one opaque handle per chain); every
operation below is one C-ABI call that runs the reference's numerical
sequence as CUDA kernels on the engine stream. Site axes are (left bond,
top physical, bottom physical, right bond) for operators and (left bond,
physical, right bond) for states; absorbing from the left realizes G.M and
from the right M.G.

Operations are functional like the reference's (chains.py:13-15): they clone
the handle (O(n), sites are copy-on-write on the device) and return a new
chain. ``sites`` downloads the tensors to numpy (a test bridge).
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .circuit import Gate, gate_unitary

DENSE_GUARD_QUBITS = 12


class _Chain:
    _d = 4

    def __init__(self, handle):
        self._h = nat.handle(handle, type(self).__name__)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and nat._lib is not None:
            nat._lib.mb_chain_free(h)
            self._h = None

    # -- inspection -------------------------------------------------------
    def _info(self):
        import ctypes as C

        n, d, dt, c = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        ln = C.c_double()
        nat._lib.mb_chain_info(self._h, C.byref(n), C.byref(d), C.byref(dt), C.byref(ln),
                               C.byref(c))
        return n.value, d.value, dt.value, ln.value, c.value

    @property
    def num_sites(self) -> int:
        return self._info()[0]

    @property
    def log_norm(self) -> float:
        return self._info()[3]

    @property
    def center(self):
        c = self._info()[4]
        return None if c < 0 else c

    @property
    def dtype(self) -> str:
        return "complex64" if self._info()[2] == nat.MB_C64 else "complex128"

    def _bonds(self) -> np.ndarray:
        n = self.num_sites
        b = np.zeros(n + 1, dtype=np.int64)
        nat._lib.mb_chain_bonds(self._h, nat.i64ptr(b))
        return b

    def bond_dims(self) -> tuple[int, ...]:
        """Extents of the N-1 internal bonds (chains.py:53-55)."""
        return tuple(int(x) for x in self._bonds()[1:-1])

    def total_elements(self) -> int:
        return int(nat._lib.mb_total_elements(self._h))

    @property
    def sites(self) -> tuple[np.ndarray, ...]:
        b = self._bonds()
        d = self._d
        sizes = [int(b[i] * d * b[i + 1]) for i in range(len(b) - 1)]
        flat = np.empty(sum(sizes), dtype=np.complex128)
        nat.check(nat._lib.mb_chain_to_host(self._h, nat.dptr(flat)), "mb_chain_to_host")
        out, off = [], 0
        for i, sz in enumerate(sizes):
            shape = (int(b[i]), 2, 2, int(b[i + 1])) if d == 4 else (int(b[i]), 2, int(b[i + 1]))
            out.append(flat[off:off + sz].reshape(shape))
            off += sz
        return tuple(out)

    def _clone_handle(self):
        return nat.handle(nat._lib.mb_chain_clone(self._h), "mb_chain_clone")

    @classmethod
    def from_sites(cls, sites, log_norm: float = 0.0, center=None, dtype: str = "complex128"):
        nat.load()
        sites = [np.asarray(s) for s in sites]
        d = cls._d
        bonds = np.array([s.shape[0] for s in sites] + [sites[-1].shape[-1]], dtype=np.int64)
        for i, s in enumerate(sites):
            want = (bonds[i], 2, 2, bonds[i + 1]) if d == 4 else (bonds[i], 2, bonds[i + 1])
            if s.shape != tuple(want):
                raise ValueError(f"site {i} has bad shape {s.shape}")
        if bonds[0] != 1 or bonds[-1] != 1:
            raise ValueError("boundary bonds must have extent 1")
        flat = np.concatenate([np.ascontiguousarray(s, dtype=np.complex128).ravel() for s in sites])
        h = nat._lib.mb_chain_from_host(len(sites), d, nat.DTYPES[dtype], nat.i64ptr(bonds),
                                        nat.dptr(flat), float(log_norm),
                                        -1 if center is None else int(center))
        return cls(h)


class MatrixProductOperator(_Chain):
    """Chain of (l, 2, 2, r) site tensors in HBM (chains.py:31-55)."""

    _d = 4


class MatrixProductState(_Chain):
    """Chain of (l, 2, r) site tensors in HBM (chains.py:58-80)."""

    _d = 2


def identity_mpo(n: int, dtype: str = "complex128") -> MatrixProductOperator:
    """Identity operator with all bond extents 1 (chains.py:83-88)."""
    if n < 1:
        raise ValueError("need at least one site")
    lib = nat.load()
    return MatrixProductOperator(lib.mb_identity_mpo(n, nat.DTYPES[dtype]))


def total_elements(m: _Chain) -> int:
    return m.total_elements()


def frobenius_norm(m: _Chain) -> float:
    """Norm of the stored chain, log_norm excluded (chains.py:95-102)."""
    import ctypes as C

    out = C.c_double()
    nat.check(nat._lib.mb_frobenius_norm(m._h, C.byref(out)), "mb_frobenius_norm")
    return out.value


def move_center(m: MatrixProductOperator, target: int) -> MatrixProductOperator:
    """Exact move of the orthogonality center (chains.py:128-145)."""
    if not (0 <= target < m.num_sites):
        raise ValueError(f"center target {target} out of range")
    h = m._clone_handle()
    out = MatrixProductOperator(h)
    nat.check(nat._lib.mb_move_center(h, int(target)), "mb_move_center")
    return out


def gate_tensor_ordered(g: Gate) -> np.ndarray:
    """4x4 gate with legs (out_lo, out_hi, in_lo, in_hi) by site index
    (chains.py:148-154), flattened row-major as complex128."""
    u4 = gate_unitary(g).reshape(2, 2, 2, 2)
    if g.qubits[0] > g.qubits[1]:
        u4 = u4.transpose(1, 0, 3, 2)
    return np.ascontiguousarray(u4.reshape(16), dtype=np.complex128)


def absorb_gate_inplace(m: MatrixProductOperator, g: Gate, side: str, epsilon: float,
                        chi_max: int) -> None:
    """In-place variant used by the driver's trial absorptions."""
    if side not in ("left", "right"):
        raise ValueError(f"side must be left or right, got {side!r}")
    lib = nat._lib
    if len(g.qubits) == 1:
        u = np.ascontiguousarray(gate_unitary(g).reshape(4), dtype=np.complex128)
        nat.check(lib.mb_absorb_1q(m._h, g.qubits[0], nat.dptr(u), nat.SIDE[side]), "absorb_1q")
        return
    a, b = g.qubits
    if abs(a - b) != 1:
        raise ValueError(f"two-qubit gate on non-adjacent sites {g.qubits}")
    g16 = gate_tensor_ordered(g)
    nat.check(lib.mb_absorb_2q(m._h, min(a, b), nat.dptr(g16), nat.SIDE[side], float(epsilon),
                               int(chi_max)), "absorb_2q")


def absorb_gate(m: MatrixProductOperator, g: Gate, side: str, epsilon: float,
                chi_max: int) -> MatrixProductOperator:
    """Contract a gate into the chain: ``left`` gives G.M, ``right`` M.G
    (chains.py:174-218). Two-qubit gates re-split their bond with the
    relative cutoff; single-qubit gates are a plain site contraction."""
    if side not in ("left", "right"):
        raise ValueError(f"side must be left or right, got {side!r}")
    out = MatrixProductOperator(m._clone_handle())
    absorb_gate_inplace(out, g, side, epsilon, chi_max)
    return out


def apply_swap_boundary(m: MatrixProductOperator, bond: int, side: str, epsilon: float,
                        chi_max: int) -> MatrixProductOperator:
    """SWAP on sites (bond, bond+1) applied to the top legs (left), bottom
    legs (right) or both, then local re-truncation (chains.py:221-259)."""
    if side not in ("left", "right", "both"):
        raise ValueError(f"side must be left, right or both, got {side!r}")
    if not (0 <= bond <= m.num_sites - 2):
        raise ValueError(f"bond {bond} out of range")
    out = MatrixProductOperator(m._clone_handle())
    nat.check(nat._lib.mb_pair_swap(out._h, bond, int(side in ("left", "both")),
                                    int(side in ("right", "both")), float(epsilon), int(chi_max),
                                    1), "pair_swap")
    return out


def compress(m: MatrixProductOperator, epsilon: float, chi_max: int) -> MatrixProductOperator:
    """Left-to-right orthogonalization then right-to-left truncation; unit
    stored norm with the scale in log_norm, center at 0 (chains.py:262-285)."""
    out = MatrixProductOperator(m._clone_handle())
    nat.check(nat._lib.mb_compress(out._h, float(epsilon), int(chi_max)), "compress")
    return out


def apply_to_zero(m: MatrixProductOperator, epsilon: float, chi_max: int) -> MatrixProductState:
    """All-zero input column, compressed and normalized (chains.py:293-324)."""
    h = nat._lib.mb_apply_to_zero(m._h, float(epsilon), int(chi_max))
    if not h:
        raise ValueError(nat._lib.mb_last_error().decode())
    return MatrixProductState(h)


def sample_uniforms(n: int, shots: int, seed: int) -> np.ndarray:
    """The reference's random stream: one rng.random(shots) per site, in
    site order (chains.py:358-367)."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.random(shots) for _ in range(n)]) if n else np.zeros((0, shots))


def sample(psi: MatrixProductState, shots: int, seed: int) -> list[str]:
    """Exact conditional sampling on the device, qubit 0 leftmost
    (chains.py:347-372); the same seed gives the reference's draws."""
    if shots < 1:
        raise ValueError("shots must be positive")
    n = psi.num_sites
    uni = np.ascontiguousarray(sample_uniforms(n, shots, seed))
    bits = np.empty((shots, n), dtype=np.uint8)
    rc = nat._lib.mb_sample(psi._h, int(shots), nat.dptr(uni), nat.u8ptr(bits))
    if rc != 0:
        raise ValueError(nat._lib.mb_last_error().decode())
    chars = np.where(bits == 1, ord("1"), ord("0")).astype(np.uint8)
    return [row.tobytes().decode() for row in chars]


def extract_peak(psi: MatrixProductState) -> tuple[str, float]:
    """Greedy sequential marginal sweep on the device: at each site keep the
    more probable branch given the chosen prefix. Returns the bitstring
    (qubit 0 leftmost) and its exact probability |<x|psi>|^2.

    This is a *greedy* peak: it is guaranteed to be the argmax only when the
    peak carries more than half the weight (each conditional then exceeds
    1/2). For peaked circuits with a 10% planted peak it can in principle
    differ from the reference's answer, the top count of samples
    (cli.py:167-173); callers that report a match cross-check it against
    sampled counts (bench.py does)."""
    n = psi.num_sites
    bits = np.empty(n, dtype=np.uint8)
    probs = np.empty(n, dtype=np.float64)
    rc = nat._lib.mb_peak(psi._h, nat.u8ptr(bits), nat.dptr(probs))
    if rc != 0:
        raise ValueError(nat._lib.mb_last_error().decode())
    return "".join("1" if b else "0" for b in bits), float(np.prod(probs))


def mpo_to_dense(m: MatrixProductOperator) -> np.ndarray:
    """Exact 2^n x 2^n matrix, qubit 0 least significant (chains.py:380-394)."""
    n = m.num_sites
    if n > DENSE_GUARD_QUBITS:
        raise ValueError(f"dense materialization capped at {DENSE_GUARD_QUBITS} sites")
    sites = m.sites
    cur = sites[0][0]
    for s in sites[1:]:
        cur = np.tensordot(cur, s, axes=(-1, 0))
    cur = cur[..., 0]
    order = [2 * i for i in reversed(range(n))] + [2 * i + 1 for i in reversed(range(n))]
    return cur.transpose(order).reshape(2 ** n, 2 ** n) * math.exp(m.log_norm)


def mps_to_dense(psi: MatrixProductState) -> np.ndarray:
    """Exact 2^n amplitudes, qubit 0 least significant (chains.py:397-407)."""
    n = psi.num_sites
    if n > DENSE_GUARD_QUBITS:
        raise ValueError(f"dense materialization capped at {DENSE_GUARD_QUBITS} sites")
    sites = psi.sites
    cur = sites[0][0]
    for s in sites[1:]:
        cur = np.tensordot(cur, s, axes=(-1, 0))
    cur = cur[..., 0]
    return cur.transpose(tuple(reversed(range(n)))).reshape(-1) * math.exp(psi.log_norm)
