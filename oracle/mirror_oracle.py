"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference contraction path.

See ``oracle/__init__.py``. References below are to
``/root/reference/pkg/src/mirrorbreak/<file>:<line>``. The restatement keeps
the reference's numerical call sequence (same LAPACK routines, same operand
order) so that its outputs match the reference bit for bit; the structure and
names are this repo's own.

Data model (all plain values, never mutated after construction):
  gate    = OGate(kind, qubits, params, routed)       routed=True <=> transpilation swap
  circuit = (n, tuple_of_gates)
  chain   = OChain(sites, log_norm, center)           MPO sites (l, top, bottom, r)
  state   = OChain(sites, log_norm, center)           MPS sites (l, phys, r)
  perm    = tuple mapping wire i -> perm[i]
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

# --------------------------------------------------------------------------
# gates (circuit.py:27-149)
# --------------------------------------------------------------------------

ARITY = {"h": (1, 0), "x": (1, 0), "rx": (1, 1), "ry": (1, 1), "rz": (1, 1),
         "u3": (1, 3), "cx": (2, 0), "rzz": (2, 1), "swap": (2, 0)}


class OGate(NamedTuple):
    kind: str
    qubits: tuple
    params: tuple = ()
    routed: bool = False

    @property
    def two(self) -> bool:
        return len(self.qubits) == 2


def unitary_of(g: OGate) -> np.ndarray:
    """circuit.py:94-132 — same matrices, same basis convention (first listed
    qubit is the most significant bit of the 2-qubit index)."""
    k, p = g.kind, g.params
    if k == "h":
        return np.array([[1, 1], [1, -1]], dtype=complex) / math.sqrt(2)
    if k == "x":
        return np.array([[0, 1], [1, 0]], dtype=complex)
    if k in ("rx", "ry"):
        c, s = math.cos(p[0] / 2), math.sin(p[0] / 2)
        if k == "rx":
            return np.array([[c, -1j * s], [-1j * s, c]], dtype=complex)
        return np.array([[c, -s], [s, c]], dtype=complex)
    if k == "rz":
        return np.array([[np.exp(-0.5j * p[0]), 0], [0, np.exp(0.5j * p[0])]], dtype=complex)
    if k == "u3":
        th, ph, lam = p
        c, s = math.cos(th / 2), math.sin(th / 2)
        return np.array([[c, -np.exp(1j * lam) * s],
                         [np.exp(1j * ph) * s, np.exp(1j * (ph + lam)) * c]], dtype=complex)
    if k == "cx":
        return np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    if k == "rzz":
        a, b = np.exp(-0.5j * p[0]), np.exp(0.5j * p[0])
        return np.diag([a, b, b, a]).astype(complex)
    if k == "swap":
        return np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)
    raise ValueError(k)


def adjoint_gate(g: OGate) -> OGate:
    """circuit.py:135-144."""
    if g.kind in ("rx", "ry", "rz", "rzz"):
        return g._replace(params=(-g.params[0],))
    if g.kind == "u3":
        th, ph, lam = g.params
        return g._replace(params=(-th, -lam, -ph))
    return g


def split_midpoint(gates):
    """circuit.py:152-182: first half gets floor(T/2) two-qubit gates; the
    cut falls right after the last of them."""
    gates = tuple(gates)
    total = sum(1 for g in gates if g.two)
    if total == 0:
        cut = len(gates) // 2
    else:
        want, seen, cut = total // 2, 0, 0
        if want:
            for idx, g in enumerate(gates):
                seen += g.two
                if g.two and seen == want:
                    cut = idx + 1
                    break
    return gates[:cut], gates[cut:]


# --------------------------------------------------------------------------
# permutations and routing (routing.py)
# --------------------------------------------------------------------------


def p_identity(n):
    return tuple(range(n))


def p_compose(a, b):
    """routing.py:308-315: (a . b)[i] = a[b[i]]."""
    return tuple(a[x] for x in b)


def p_inverse(a):
    out = [0] * len(a)
    for i, m in enumerate(a):
        out[m] = i
    return tuple(out)


def p_transposition(n, i, j):
    m = list(range(n))
    m[i], m[j] = m[j], m[i]
    return tuple(m)


def p_apply_bits(a, bits: str) -> str:
    """routing.py:317-321."""
    out = ["0"] * len(a)
    for i, b in enumerate(bits):
        out[a[i]] = b
    return "".join(out)


def p_factorization(a):
    """routing.py:323-339: bubble sort of the one-line notation."""
    arr, swaps, dirty = list(a), [], True
    while dirty:
        dirty = False
        for x in range(len(arr) - 1):
            if arr[x] > arr[x + 1]:
                arr[x], arr[x + 1] = arr[x + 1], arr[x]
                swaps.append((x, x + 1))
                dirty = True
    return tuple(swaps)


def p_advance(layout, wa, wb):
    """routing.py:460-463."""
    return p_compose(p_transposition(len(layout), wa, wb), layout)


class _Wires:
    """logical<->wire bookkeeping (routing.py:357-372)."""

    def __init__(self, n, l2p=None):
        self.l2p = list(l2p) if l2p is not None else list(range(n))
        self.p2l = [0] * n
        for lg, w in enumerate(self.l2p):
            self.p2l[w] = lg

    def swap(self, w1, w2):
        a, b = self.p2l[w1], self.p2l[w2]
        self.p2l[w1], self.p2l[w2] = b, a
        self.l2p[a], self.l2p[b] = w2, w1


def route(n, gates, direction="forward"):
    """routing.py:385-420. Returns (gates, input_layout, output_layout)."""
    wires = _Wires(n)
    out = []
    seq = gates if direction == "forward" else tuple(reversed(gates))
    for g in seq:
        if len(g.qubits) == 1:
            out.append(g._replace(qubits=(wires.l2p[g.qubits[0]],)))
            continue
        a, b = g.qubits
        pa, pb = wires.l2p[a], wires.l2p[b]
        if abs(pa - pb) != 1:
            lo, hi = min(pa, pb), max(pa, pb)
            for w in range(hi, lo + 1, -1):
                out.append(OGate("swap", (w - 1, w), (), True))
                wires.swap(w - 1, w)
            pa, pb = wires.l2p[a], wires.l2p[b]
        out.append(g._replace(qubits=(pa, pb)))
    if direction == "forward":
        return tuple(out), p_identity(n), tuple(wires.l2p)
    return tuple(reversed(out)), tuple(wires.l2p), p_identity(n)


def strip_routing(n, gates, initial=None):
    """routing.py:423-443."""
    wires = _Wires(n, initial)
    out = []
    for g in gates:
        if g.routed:
            wires.swap(*g.qubits)
            continue
        out.append(OGate(g.kind, tuple(wires.p2l[q] for q in g.qubits), g.params, False))
    return tuple(out)


def relabel(gates, perm):
    """routing.py:446-457."""
    return tuple(g._replace(qubits=tuple(perm[q] for q in g.qubits)) for g in gates)


# --------------------------------------------------------------------------
# truncated SVD (tensor.py:84-150)
# --------------------------------------------------------------------------

TIE = 1e-12


def kept_rank(s, eps, chi_max):
    """tensor.py:119-136: smallest r with relative discarded weight <= eps^2,
    grown across near-ties at the boundary, capped at chi_max, >= 1."""
    w = s * s
    total = float(w.sum())
    tail = np.concatenate([np.cumsum(w[::-1])[::-1], [0.0]])
    budget = eps * eps * total
    r = len(s)
    for k in range(1, len(s) + 1):
        if tail[k] <= budget:
            r = k
            break
    edge = s[r - 1]
    while r < len(s) and s[r] >= edge - TIE:
        r += 1
    return min(r, chi_max)


def _lapack_svd(m):
    """tensor.py:139-150 (gesdd, one perturbed retry)."""
    try:
        return np.linalg.svd(m, full_matrices=False)
    except np.linalg.LinAlgError:
        pert = m + 1e-14 * np.linalg.norm(m) * np.random.default_rng(0).standard_normal(m.shape)
        return np.linalg.svd(pert, full_matrices=False)


def tsvd(t, split, eps, chi_max):
    """tensor.py:84-116. Returns (u, s, v, discarded_weight)."""
    t = np.asarray(t, dtype=np.complex128)
    rows = int(np.prod(t.shape[:split], dtype=np.int64))
    mat = t.reshape(rows, -1)
    if not np.any(mat):
        raise ValueError("cannot decompose an all-zero tensor")
    u, s, v = _lapack_svd(mat)
    r = kept_rank(s, eps, chi_max)
    w = s * s
    disc = float(w[r:].sum() / float(w.sum()))
    return u[:, :r], s[:r].copy(), v[:r, :], disc


# --------------------------------------------------------------------------
# chains (chains.py)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class OChain:
    sites: tuple
    log_norm: float = 0.0
    center: int | None = None

    def bonds(self):
        return tuple(s.shape[-1] for s in self.sites[:-1])

    def elements(self):
        return sum(s.size for s in self.sites)


def identity_chain(n):
    """chains.py:83-88."""
    eye = np.eye(2, dtype=np.complex128).reshape(1, 2, 2, 1)
    return OChain(tuple(eye.copy() for _ in range(n)), 0.0, None)


def chain_norm(c: OChain):
    """chains.py:95-102."""
    if c.center is not None:
        return float(np.linalg.norm(c.sites[c.center]))
    env = np.ones((1, 1), dtype=np.complex128)
    for s in c.sites:
        env = np.einsum("ab,atpr,btpq->rq", env, np.conj(s), s)
    return float(math.sqrt(abs(env[0, 0].real)))


def _push_right(sites, i):
    """chains.py:110-116: left-orthogonalize site i."""
    l, t, b, r = sites[i].shape
    q, rem = np.linalg.qr(sites[i].reshape(l * t * b, r))
    sites[i] = q.reshape(l, t, b, q.shape[1])
    sites[i + 1] = np.tensordot(rem, sites[i + 1], axes=(1, 0))


def _push_left(sites, i):
    """chains.py:119-125: right-orthogonalize site i (QR of the transpose)."""
    l, t, b, r = sites[i].shape
    q, rem = np.linalg.qr(sites[i].reshape(l, t * b * r).T)
    sites[i] = q.T.reshape(q.shape[1], t, b, r)
    sites[i - 1] = np.tensordot(sites[i - 1], rem.T, axes=(3, 0))


def recenter(c: OChain, target):
    """chains.py:128-145."""
    n = len(c.sites)
    sites = list(c.sites)
    if c.center is None:
        for i in range(target):
            _push_right(sites, i)
        for i in range(n - 1, target, -1):
            _push_left(sites, i)
    elif c.center < target:
        for i in range(c.center, target):
            _push_right(sites, i)
    else:
        for i in range(c.center, target, -1):
            _push_left(sites, i)
    return OChain(tuple(sites), c.log_norm, target)


def _ordered_gate4(g: OGate):
    """chains.py:148-154: (out_lo, out_hi, in_lo, in_hi) by site index."""
    u = unitary_of(g).reshape(2, 2, 2, 2)
    return u.transpose(1, 0, 3, 2) if g.qubits[0] > g.qubits[1] else u


def _resplit(theta, eps, chi_max):
    """chains.py:157-167: singular values go to the right factor."""
    l, t1, b1, t2, b2, r = theta.shape
    u, s, v, _ = tsvd(theta, 3, eps, chi_max)
    k = len(s)
    return u.reshape(l, t1, b1, k), (s[:, None] * v).reshape(k, t2, b2, r)


def _blob(sites, i):
    """chains.py:170-171."""
    return np.tensordot(sites[i], sites[i + 1], axes=(3, 0))


def absorb(c: OChain, g: OGate, side, eps, chi_max):
    """chains.py:174-218."""
    if len(g.qubits) == 1:
        u = unitary_of(g)
        q = g.qubits[0]
        sites = list(c.sites)
        if side == "left":
            sites[q] = np.einsum("tk,lkbr->ltbr", u, sites[q])
        else:
            sites[q] = np.einsum("ltkr,kb->ltbr", sites[q], u)
        return OChain(tuple(sites), c.log_norm, c.center)
    i = min(g.qubits)
    c = recenter(c, i)
    sites = list(c.sites)
    theta = _blob(sites, i)
    u4 = _ordered_gate4(g)
    if side == "left":
        theta = np.einsum("xytu,ltbuar->lxbyar", u4, theta)
    else:
        theta = np.einsum("ltbuar,baxy->ltxuyr", theta, u4)
    sites[i], sites[i + 1] = _resplit(theta, eps, chi_max)
    return OChain(tuple(sites), c.log_norm, i + 1)


def _exchange(theta, top, bottom):
    if top:
        theta = theta.transpose(0, 3, 2, 1, 4, 5)
    if bottom:
        theta = theta.transpose(0, 1, 4, 3, 2, 5)
    return theta


def swap_bond(c: OChain, bond, side, eps, chi_max):
    """chains.py:221-259 (apply_swap_boundary / _pair_swap)."""
    c = recenter(c, bond)
    sites = list(c.sites)
    theta = _exchange(_blob(sites, bond), side in ("left", "both"), side in ("right", "both"))
    sites[bond], sites[bond + 1] = _resplit(theta, eps, chi_max)
    return OChain(tuple(sites), c.log_norm, bond + 1)


def compress(c: OChain, eps, chi_max):
    """chains.py:262-285."""
    n = len(c.sites)
    sites = list(c.sites)
    for i in range(n - 1):
        _push_right(sites, i)
    for i in range(n - 1, 0, -1):
        l, t, b, r = sites[i].shape
        u, s, v, _ = tsvd(sites[i], 1, eps, chi_max)
        sites[i] = v.reshape(len(s), t, b, r)
        sites[i - 1] = np.tensordot(sites[i - 1], u * s[None, :], axes=(3, 0))
    f = float(np.linalg.norm(sites[0]))
    if f == 0.0:
        raise ValueError("compress reached an all-zero chain")
    sites[0] = sites[0] / f
    return OChain(tuple(sites), c.log_norm + math.log(f), 0)


def to_zero_state(c: OChain, eps, chi_max):
    """chains.py:293-324."""
    scale = chain_norm(c)
    sites = [s[:, :, 0, :] for s in c.sites]
    n = len(sites)
    for i in range(n - 1):
        l, p, r = sites[i].shape
        q, rem = np.linalg.qr(sites[i].reshape(l * p, r))
        sites[i] = q.reshape(l, p, q.shape[1])
        sites[i + 1] = np.tensordot(rem, sites[i + 1], axes=(1, 0))
    for i in range(n - 1, 0, -1):
        l, p, r = sites[i].shape
        u, s, v, _ = tsvd(sites[i], 1, eps, chi_max)
        sites[i] = v.reshape(len(s), p, r)
        sites[i - 1] = np.tensordot(sites[i - 1], u * s[None, :], axes=(2, 0))
    f = float(np.linalg.norm(sites[0]))
    if f < 1e-12 * (scale / (2 ** (n / 2))):
        raise ValueError("all-zero column norm collapsed")
    sites[0] = sites[0] / f
    return OChain(tuple(sites), c.log_norm + math.log(f), 0)


def _state_right_canonical(psi: OChain):
    """chains.py:327-344."""
    sites = list(psi.sites)
    n = len(sites)
    start = psi.center if psi.center is not None else n - 1
    if psi.center is None:
        for i in range(n - 1):
            l, p, r = sites[i].shape
            q, rem = np.linalg.qr(sites[i].reshape(l * p, r))
            sites[i] = q.reshape(l, p, q.shape[1])
            sites[i + 1] = np.tensordot(rem, sites[i + 1], axes=(1, 0))
    for i in range(start, 0, -1):
        l, p, r = sites[i].shape
        q, rem = np.linalg.qr(sites[i].reshape(l, p * r).T)
        sites[i] = q.T.reshape(q.shape[1], p, r)
        sites[i - 1] = np.tensordot(sites[i - 1], rem.T, axes=(2, 0))
    return sites, float(np.linalg.norm(sites[0]))


def sample_state(psi: OChain, shots, seed):
    """chains.py:347-372 (same RNG stream: one rng.random(shots) per site)."""
    sites, nrm = _state_right_canonical(psi)
    if abs(nrm - 1.0) > 1e-6:
        raise ValueError("state is not normalized")
    rng = np.random.default_rng(seed)
    env = np.ones((shots, 1), dtype=np.complex128)
    bits = np.empty((shots, len(sites)), dtype=np.int8)
    rows = np.arange(shots)
    for i, s in enumerate(sites):
        amp = np.einsum("sl,lpr->spr", env, s)
        pr = np.sum(np.abs(amp) ** 2, axis=2)
        p1 = pr[:, 1] / pr.sum(axis=1)
        pick = (rng.random(shots) < p1).astype(np.int8)
        bits[:, i] = pick
        env = amp[rows, pick, :] / np.sqrt(pr[rows, pick])[:, None]
    return ["".join("1" if b else "0" for b in row) for row in bits]


def greedy_peak(psi: OChain):
    """Peak extraction by a sequential marginal sweep (the product's
    ``extract_peak``; no reference counterpart beyond sampling, chains.py:347).

    Right-canonicalize, then walk left to right keeping the conditional
    environment of the chosen prefix; at each site take the branch with the
    larger conditional probability (ties -> 0). Returns (bits, probability
    of the returned bitstring, marginal probabilities of each choice).
    """
    sites, _ = _state_right_canonical(psi)
    env = np.ones(1, dtype=np.complex128)
    bits, prob = [], 1.0
    for s in sites:
        amp = np.einsum("l,lpr->pr", env, s)
        pr = np.sum(np.abs(amp) ** 2, axis=1)
        tot = pr[0] + pr[1]
        pick = 1 if pr[1] > pr[0] else 0
        bits.append(pick)
        prob *= pr[pick] / tot
        env = amp[pick] / math.sqrt(pr[pick])
    return "".join(str(b) for b in bits), prob


def chain_dense(c: OChain):
    """chains.py:380-394 (qubit 0 = least significant bit)."""
    n = len(c.sites)
    cur = c.sites[0][0]
    for s in c.sites[1:]:
        cur = np.tensordot(cur, s, axes=(-1, 0))
    cur = cur[..., 0]
    order = [2 * i for i in range(n)][::-1] + [2 * i + 1 for i in range(n)][::-1]
    return cur.transpose(order).reshape(2 ** n, 2 ** n) * math.exp(c.log_norm)


def state_dense(psi: OChain):
    """chains.py:397-407."""
    n = len(psi.sites)
    cur = psi.sites[0][0]
    for s in psi.sites[1:]:
        cur = np.tensordot(cur, s, axes=(-1, 0))
    cur = cur[..., 0]
    return cur.transpose(tuple(range(n))[::-1]).reshape(-1) * math.exp(psi.log_norm)


# --------------------------------------------------------------------------
# unswapping (unswap.py)
# --------------------------------------------------------------------------

_CYCLE = (("both", 0), ("both", 1), ("left", 0), ("left", 1), ("right", 0), ("right", 1))


class _Factor:
    """unswap.py:67-92: chain + accumulated outer permutations."""

    def __init__(self, c: OChain):
        n = len(c.sites)
        self.c, self.left, self.right, self.accepted = c, p_identity(n), p_identity(n), 0
        self.log = []  # (bond, side) of accepted swaps, in order

    def accept(self, c, bond, side):
        tau = p_transposition(len(c.sites), bond, bond + 1)
        if side in ("left", "both"):
            self.left = p_compose(self.left, tau)
        if side in ("right", "both"):
            self.right = p_compose(tau, self.right)
        self.c = c
        self.accepted += 1
        self.log.append((bond, side))


def swap_extent(c: OChain, bond, side, eps, chi_max):
    """unswap.py:104-112: values-only SVD of the swapped blob."""
    theta = _exchange(_blob(c.sites, bond), side in ("left", "both"), side in ("right", "both"))
    s = np.linalg.svd(theta.reshape(theta.shape[0] * 4, -1), compute_uv=False)
    return kept_rank(s, eps, chi_max)


def _commit_swap(c: OChain, bond, side, eps, chi_max):
    """unswap.py:115-121."""
    sites = list(c.sites)
    theta = _exchange(_blob(sites, bond), side in ("left", "both"), side in ("right", "both"))
    sites[bond], sites[bond + 1] = _resplit(theta, eps, chi_max)
    return OChain(tuple(sites), c.log_norm, bond + 1)


def _retruncate(c: OChain, bond, eps, chi_max):
    """unswap.py:124-134."""
    c = recenter(c, bond)
    sites = list(c.sites)
    sites[bond], sites[bond + 1] = _resplit(_blob(sites, bond), eps, chi_max)
    return OChain(tuple(sites), c.log_norm, bond + 1), sites[bond].shape[3]


def _attempt(st: _Factor, bond, sides, eps, chi_max, relaxed, seen):
    """unswap.py:137-167."""
    c, base = _retruncate(st.c, bond, eps, chi_max)
    st.c = c
    best = None
    for side in sides:
        if seen is not None and (bond, side) in seen:
            continue
        ext = swap_extent(c, bond, side, eps, chi_max)
        if best is None or ext < best[1]:
            best = (side, ext)
    if best is None:
        return False
    side, ext = best
    if ext < base or (relaxed and ext == base):
        if seen is not None:
            seen.add((bond, side))
        st.accept(_commit_swap(c, bond, side, eps, chi_max), bond, side)
        return True
    return False


def unswap_sequential(c: OChain, eps, chi_max, relaxed=False, max_outer=20):
    """unswap.py:170-211."""
    st = _Factor(c)
    before = c.elements()
    n = len(c.sites)
    limit = max_outer * max(1, n - 1) * 3 * 16
    evals = 0
    for _ in range(max_outer):
        avail = set(range(n - 1))
        seen = set() if relaxed else None
        took = 0
        while avail:
            evals += 1
            if evals > limit:
                raise RuntimeError("unswap exceeded its evaluation budget")
            dims = st.c.bonds()
            bond = max(avail, key=lambda i: (dims[i], -i))
            if _attempt(st, bond, ("left", "right", "both"), eps, chi_max, relaxed, seen):
                took += 1
                avail.discard(bond)
                if bond >= 1:
                    avail.add(bond - 1)
                if bond + 1 <= n - 2:
                    avail.add(bond + 1)
            else:
                avail.discard(bond)
        if took == 0:
            break
    return st, before


def unswap_parallel(c: OChain, eps, chi_max, relaxed=False, max_outer=20):
    """unswap.py:214-240."""
    st = _Factor(c)
    before = c.elements()
    n = len(c.sites)
    for _ in range(max_outer):
        shrank = False
        for side, parity in _CYCLE:
            for bond in range(parity, n - 1, 2):
                was = st.c.bonds()[bond]
                if _attempt(st, bond, (side,), eps, chi_max, relaxed, None):
                    if st.c.bonds()[bond] < was:
                        shrank = True
        if not shrank:
            break
    return st, before


# --------------------------------------------------------------------------
# driver (driver.py)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class OConfig:
    """driver.py:50-88 defaults (paper App. A.4)."""
    epsilon: float = 2e-3
    chi_max: int = 8192
    tau: int = 1_000_000
    max_unswap_iterations: int = 20
    acceptance: str = "strict"
    unswap_strategy: str = "parity-parallel"
    side_mode: str = "adaptive"
    stall_limit: int = 3

    @property
    def every(self):
        return None if self.side_mode == "adaptive" else int(self.side_mode.split(":", 1)[1])


class OStall(RuntimeError):
    def __init__(self, elements, reductions, trace):
        super().__init__(f"no exploitable mirror structure ({elements} elements)")
        self.elements, self.reductions, self.trace = elements, reductions, trace


def pop_layer(gates, from_back):
    """driver.py:137-156: maximal brick layer of innermost gates."""
    order = range(len(gates) - 1, -1, -1) if from_back else range(len(gates))
    blocked, taken, layer = set(), set(), []
    for idx in order:
        g = gates[idx]
        if blocked.isdisjoint(g.qubits):
            taken.add(idx)
            layer.append(g)
        blocked.update(g.qubits)
    return layer, [g for i, g in enumerate(gates) if i not in taken]


class _Half:
    """driver.py:127-134."""

    def __init__(self, gates, front, back):
        self.gates, self.front, self.back = list(gates), front, back


def _trial(c, half: _Half, which, cfg: OConfig, hooks=None):
    """driver.py:178-191."""
    layer, rest = pop_layer(half.gates, which == "right")
    for g in layer:
        c = absorb(c, g, which, cfg.epsilon, cfg.chi_max)
    c = compress(c, cfg.epsilon, cfg.chi_max)
    return c, layer, rest


def _pick_side(left: _Half, right: _Half, c, cfg: OConfig, step):
    """driver.py:194-223."""
    if not left.gates:
        return ("right",) + _trial(c, right, "right", cfg)
    if not right.gates:
        return ("left",) + _trial(c, left, "left", cfg)
    k = cfg.every
    if k is not None:
        which = "left" if (step // k) % 2 == 0 else "right"
        return (which,) + _trial(c, left if which == "left" else right, which, cfg)
    tl = _trial(c, left, "left", cfg)
    tr = _trial(c, right, "right", cfg)
    if tl[0].elements() <= tr[0].elements():
        return ("left",) + tl
    return ("right",) + tr


def _rewire_left(pi_out, half: _Half, extracted, n):
    """driver.py:226-235."""
    logical = strip_routing(n, half.gates, half.front)
    sigma = p_compose(p_inverse(half.front), extracted)
    gates, _, drift = route(n, relabel(logical, p_inverse(sigma)), "forward")
    pi_out = p_compose(p_compose(p_compose(pi_out, half.back), sigma), p_inverse(drift))
    return pi_out, _Half(gates, p_identity(n), drift)


def _rewire_right(pi_in, half: _Half, extracted, n):
    """driver.py:238-247."""
    logical = strip_routing(n, half.gates, half.front)
    sigma = p_compose(extracted, half.back)
    gates, drift, _ = route(n, relabel(logical, sigma), "reverse")
    pi_in = p_compose(p_compose(p_compose(drift, sigma), p_inverse(half.front)), pi_in)
    return pi_in, _Half(gates, drift, p_identity(n))


@dataclass
class OResult:
    state: OChain
    pi_out: tuple
    pi_in: tuple
    trace: list          # (phase, unitaries_consumed, elements)
    final_elements: int
    chi_saturations: int
    unswap_logs: list    # per unswap call: list of accepted (bond, side)
    consumed_source: int = 0


def contract(n, gates, cfg: OConfig = OConfig(), max_steps=None, on_record=None):
    """driver.py:250-346. ``max_steps`` bounds the number of absorption steps
    (used only by the bounded CPU baseline; None = run to completion).
    ``on_record(record, chain)`` is called after every trace record (used by
    the long-run golden generator to stream the trace)."""
    if not gates:
        raise ValueError("circuit has no gates")
    if cfg.tau < 4 * n:
        raise ValueError("tau below the identity chain size")
    routed, _, out_layout = route(n, tuple(gates), "forward")
    first, second = split_midpoint(routed)
    cut = p_identity(n)
    for g in first:
        if g.routed:
            cut = p_advance(cut, *g.qubits)
    pi_out, pi_in = p_inverse(out_layout), p_identity(n)
    left = _Half(second, cut, out_layout)
    right = _Half(first, p_identity(n), cut)
    c = identity_chain(n)
    trace, logs = [], []
    consumed = consumed_src = step = sat = 0
    src_total = sum(1 for g in gates if g.two)
    stalls = []
    strat = unswap_sequential if cfg.unswap_strategy == "sequential" else unswap_parallel
    while left.gates or right.gates:
        progressed = False
        while (c.elements() < cfg.tau or not progressed) and (left.gates or right.gates):
            which, c, layer, rest = _pick_side(left, right, c, cfg, step)
            half = left if which == "left" else right
            for g in layer:
                if g.routed:
                    if which == "right":
                        half.back = p_advance(half.back, *g.qubits)
                    else:
                        half.front = p_advance(half.front, *g.qubits)
            half.gates = rest
            consumed += sum(1 for g in layer if g.two)
            consumed_src += sum(1 for g in layer if g.two and not g.routed)
            if any(not g.routed for g in layer):
                progressed = True
            step += 1
            if any(d >= cfg.chi_max for d in c.bonds()):
                sat += 1
            trace.append(("absorb", consumed, c.elements()))
            if on_record is not None:
                on_record(trace[-1], c)
            if max_steps is not None and step >= max_steps:
                return OResult(None, pi_out, pi_in, trace, c.elements(), sat, logs, consumed_src)
        if not (left.gates or right.gates):
            break
        before = c.elements()
        st, _ = strat(c, cfg.epsilon, cfg.chi_max, cfg.acceptance == "relaxed",
                      cfg.max_unswap_iterations)
        logs.append(list(st.log))
        c = compress(st.c, cfg.epsilon, cfg.chi_max)
        after = c.elements()
        trace.append(("unswap", consumed, after))
        if on_record is not None:
            on_record(trace[-1], c)
        red = (before - after) / before if before else 0.0
        if after >= cfg.tau and red < 0.01:
            stalls.append(red)
            if len(stalls) >= cfg.stall_limit:
                raise OStall(after, stalls, trace)
        else:
            stalls = []
        pi_out, left = _rewire_left(pi_out, left, st.left, n)
        pi_in, right = _rewire_right(pi_in, right, st.right, n)
    if consumed_src != src_total:
        raise AssertionError("layer accounting bug")
    psi = to_zero_state(c, cfg.epsilon, cfg.chi_max)
    return OResult(psi, pi_out, pi_in, trace, c.elements(), sat, logs, consumed_src)


def sample_result(res: OResult, shots, seed):
    """driver.py:349-355."""
    raw = sample_state(res.state, shots, seed)
    if res.pi_out == p_identity(len(res.pi_out)):
        return raw
    return [p_apply_bits(res.pi_out, b) for b in raw]


def peak_result(res: OResult):
    """Greedy marginal peak of the output state, relabeled through pi_out."""
    bits, p = greedy_peak(res.state)
    return p_apply_bits(res.pi_out, bits), p


def result_dense(res: OResult):
    """driver.py:358-361."""
    from .statevector import permute_vector
    return permute_vector(res.pi_out, state_dense(res.state))


# --------------------------------------------------------------------------
# serialized-circuit reader (the subset circuit.py:407-419 emits)
# --------------------------------------------------------------------------


def read_qasm(text):
    """Parse the one-gate-per-line OpenQASM 2.0 that the reference's
    serializer writes (circuit.py:407-419). Returns (n, gates)."""
    import re

    n, gates = None, []
    for line in text.splitlines():
        line = line.strip()
        if not line or line.startswith(("OPENQASM", "include")):
            continue
        if line.startswith("qreg"):
            n = int(re.search(r"\[(\d+)\]", line).group(1))
            continue
        m = re.fullmatch(r"([a-z0-9]+)(?:\(([^)]*)\))?\s+(.+);", line)
        kind, params, ops = m.group(1), m.group(2), m.group(3)
        qs = tuple(int(x) for x in re.findall(r"q\[(\d+)\]", ops))
        ps = tuple(float(p) for p in params.split(",")) if params else ()
        gates.append(OGate(kind, qs, ps, False))
    return n, tuple(gates)
