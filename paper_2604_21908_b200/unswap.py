"""Greedy extraction of hidden permutations from a device-resident chain:
input = P_left . reduced . P_right (reference unswap.py).

The control flow (availability set, parity cycle, tie rules, acceptance) is
host logic identical to the reference; the numerics per bond are device
calls: the bond re-truncation is ``mb_pair_swap(recenter=1)`` with no swap,
the left/right/both candidate extents are ONE batched ``mb_swap_extents``
call (values-only decompositions, one CTA per candidate), and the accepted
candidate is re-split in place with ``mb_pair_swap(recenter=0)``.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .chains import MatrixProductOperator, total_elements
from .routing import QubitPermutation
from .sharding import Comm, unswap_parity_batched

_EVALUATION_SLACK = 16

# MB_BOND_RUN=0: drive each bond step of a parity batch from Python instead
_BOND_RUN = os.environ.get("MB_BOND_RUN", "1") != "0"
PARALLEL_CYCLE = (("both", 0), ("both", 1), ("left", 0), ("left", 1), ("right", 0), ("right", 1))


@dataclass(frozen=True)
class UnswapConfig:
    """unswap.py:38-54 (paper App. A.1, A.2, A.4)."""

    epsilon: float
    chi_max: int
    acceptance: str = "strict"
    strategy: str = "sequential"
    max_outer_iterations: int = 20

    def __post_init__(self):
        if self.acceptance not in ("strict", "relaxed"):
            raise ValueError(f"acceptance must be strict or relaxed, got {self.acceptance!r}")
        if self.strategy not in ("sequential", "parity-parallel", "parity-batched"):
            raise ValueError(
                "strategy must be sequential, parity-parallel or parity-batched, "
                f"got {self.strategy!r}")
        if self.max_outer_iterations < 1:
            raise ValueError("max_outer_iterations must be >= 1")


@dataclass(frozen=True)
class UnswapResult:
    reduced: MatrixProductOperator
    left_perm: QubitPermutation
    right_perm: QubitPermutation
    accepted_swaps: int
    elements_before: int
    elements_after: int


class _Work:
    """The chain being reduced (mutated in place on the device) plus the
    accumulated outer permutations (unswap.py:67-92)."""

    def __init__(self, m: MatrixProductOperator, cfg: UnswapConfig):
        self.m = MatrixProductOperator(m._clone_handle())
        n = m.num_sites
        self.n = n
        self.left = QubitPermutation.identity(n)
        self.right = QubitPermutation.identity(n)
        self.accepted = 0
        self.cfg = cfg
        self.bonds = list(m.bond_dims())
        self.log: list[tuple[int, str]] = []

    def refresh(self):
        # host-side metadata read (no device sync); a center move can shrink
        # any bond it crosses, so refresh them all
        self.bonds = [int(x) for x in self.m._bonds()[1:-1]]

    def normalize(self, bond: int) -> int:
        """Move the center to the bond and re-truncate it (unswap.py:124-134)."""
        nat.check(nat._lib.mb_pair_swap(self.m._h, bond, 0, 0, self.cfg.epsilon,
                                        self.cfg.chi_max, 1), "normalize bond")
        self.refresh()
        return self.bonds[bond]

    def extents(self, bond: int, sides) -> list[int]:
        """Values-only candidate extents, batched (unswap.py:104-112)."""
        codes = (C.c_int * len(sides))(*(nat.SIDE[s] for s in sides))
        out = np.zeros(len(sides), dtype=np.int64)
        nat.check(nat._lib.mb_swap_extents(self.m._h, bond, len(sides), codes, self.cfg.epsilon,
                                           self.cfg.chi_max, nat.i64ptr(out)), "swap extents")
        return [int(x) for x in out]

    def try_bond(self, bond: int, sides) -> int:
        """Normalize + score + accept in one device call; returns the index
        of the accepted side in ``sides`` or -1 (baseline/extents kept in
        ``last_scores`` for tracing)."""
        codes = (C.c_int * max(1, len(sides)))(*(nat.SIDE[s] for s in sides))
        base = C.c_int64()
        ext = np.zeros(3, dtype=np.int64)
        acc = C.c_int()
        nat.check(nat._lib.mb_try_bond(self.m._h, bond, len(sides), codes, self.cfg.epsilon,
                                       self.cfg.chi_max, int(self.cfg.acceptance == "relaxed"),
                                       C.byref(base), nat.i64ptr(ext), C.byref(acc)), "try bond")
        self.last_scores = (int(base.value), [int(x) for x in ext[:len(sides)]])
        if acc.value < 0:
            self.refresh()
        return int(acc.value)

    def score_batch(self, bonds, mine, side):
        """Device batch scoring of one (side, parity) batch (this rank's shard)."""
        nb = len(bonds)
        b_arr = (C.c_int * nb)(*bonds)
        m_arr = (C.c_int * nb)(*mine)
        base = np.full(nb, -1, dtype=np.int64)
        ext = np.full(nb, -1, dtype=np.int64)
        nat.check(nat._lib.mb_batch_swap_extents(self.m._h, nb, b_arr, m_arr, nat.SIDE[side],
                                                 self.cfg.epsilon, self.cfg.chi_max,
                                                 nat.i64ptr(base), nat.i64ptr(ext)),
                  "batch swap extents")
        self.refresh()
        return base, ext

    def accept_recenter(self, bond: int, side: str) -> None:
        """Apply a batch-accepted swap with the center moved onto the bond."""
        nat.check(nat._lib.mb_pair_swap(self.m._h, bond, int(side in ("left", "both")),
                                        int(side in ("right", "both")), self.cfg.epsilon,
                                        self.cfg.chi_max, 1), "apply batched candidate")
        self._record(bond, side)

    def try_bond_run(self, bonds, side: str):
        """One (side, parity) batch of single-side bond steps in one engine
        call (mb_try_bond_run): per bond (accepted, dim before, dim after)."""
        nb = len(bonds)
        b_arr = (C.c_int * max(1, nb))(*bonds)
        acc = (C.c_int * max(1, nb))()
        was = np.zeros(max(1, nb), dtype=np.int64)
        now = np.zeros(max(1, nb), dtype=np.int64)
        nat.check(nat._lib.mb_try_bond_run(self.m._h, nb, b_arr, nat.SIDE[side], self.cfg.epsilon,
                                           self.cfg.chi_max, int(self.cfg.acceptance == "relaxed"),
                                           acc, nat.i64ptr(was), nat.i64ptr(now)), "try bond run")
        self.refresh()
        return [bool(acc[i]) for i in range(nb)], was[:nb].tolist(), now[:nb].tolist()

    def _record(self, bond: int, side: str, refresh: bool = True) -> None:
        if refresh:
            self.refresh()
        tau = QubitPermutation.transposition(self.n, bond, bond + 1)
        if side in ("left", "both"):
            self.left = self.left.compose(tau)
        if side in ("right", "both"):
            self.right = tau.compose(self.right)
        self.accepted += 1
        self.log.append((bond, side))

    def accept(self, bond: int, side: str) -> None:
        """Materialize the candidate and record the swap (unswap.py:84-92, 115-121)."""
        nat.check(nat._lib.mb_pair_swap(self.m._h, bond, int(side in ("left", "both")),
                                        int(side in ("right", "both")), self.cfg.epsilon,
                                        self.cfg.chi_max, 0), "apply candidate")
        self.refresh()
        tau = QubitPermutation.transposition(self.n, bond, bond + 1)
        if side in ("left", "both"):
            self.left = self.left.compose(tau)
        if side in ("right", "both"):
            self.right = tau.compose(self.right)
        self.accepted += 1
        self.log.append((bond, side))


def _try_bond(w: _Work, bond: int, sides, seen) -> bool:
    """unswap.py:137-167: normalize the bond, score the candidate sides on the
    normalized split, accept the best (ties prefer earlier sides: left,
    right, both) iff it shrinks the bond (relaxed: does not grow it). One
    engine call (mb_try_bond), one host round trip."""
    todo = [s for s in sides if seen is None or (bond, s) not in seen]
    chosen = w.try_bond(bond, todo)
    if chosen < 0:
        return False
    side = todo[chosen]
    if seen is not None:
        seen.add((bond, side))
    w._record(bond, side)
    return True


def _result(w: _Work, before: int) -> UnswapResult:
    return UnswapResult(reduced=w.m, left_perm=w.left, right_perm=w.right,
                        accepted_swaps=w.accepted, elements_before=before,
                        elements_after=total_elements(w.m))


def unswap_sequential(m: MatrixProductOperator, cfg: UnswapConfig) -> UnswapResult:
    """Availability-set loop over bonds ranked by extent, lowest index on
    ties; acceptance re-enables the neighbours (unswap.py:170-211)."""
    w = _Work(m, cfg)
    before = total_elements(m)
    n = w.n
    budget = cfg.max_outer_iterations * max(1, n - 1) * 3 * _EVALUATION_SLACK
    evals = 0
    for _ in range(cfg.max_outer_iterations):
        avail = set(range(n - 1))
        seen = set() if cfg.acceptance == "relaxed" else None
        took = 0
        while avail:
            evals += 1
            if evals > budget:
                raise RuntimeError("unswap exceeded its evaluation budget")
            bond = max(avail, key=lambda i: (w.bonds[i], -i))
            if _try_bond(w, bond, ("left", "right", "both"), seen):
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
    return _result(w, before)


def unswap_parallel(m: MatrixProductOperator, cfg: UnswapConfig) -> UnswapResult:
    """Parity-batched variant cycling (both, left, right) x (even, odd);
    stops after a cycle with no bond reduction (unswap.py:214-240)."""
    w = _Work(m, cfg)
    before = total_elements(m)
    n = w.n
    for _ in range(cfg.max_outer_iterations):
        reduced = False
        for side, parity in PARALLEL_CYCLE:
            bonds = list(range(parity, n - 1, 2))
            if not _BOND_RUN:
                for bond in bonds:
                    was = w.bonds[bond]
                    if _try_bond(w, bond, (side,), None) and w.bonds[bond] < was:
                        reduced = True
                continue
            # the same steps in the same order, driven from C++ (one call)
            acc, was, now = w.try_bond_run(bonds, side)
            for bond, a, b0, b1 in zip(bonds, acc, was, now):
                if a:
                    w._record(bond, side, refresh=False)
                    if b1 < b0:
                        reduced = True
        if not reduced:
            break
    return _result(w, before)


def unswap_batched(m: MatrixProductOperator, cfg: UnswapConfig,
                   comm: Comm | None = None) -> UnswapResult:
    """Parity batches scored in one batched device pass each, optionally
    sharded over the ranks of ``comm`` (sharding.py). Not bit-identical to the
    reference's bond-by-bond re-truncation order, which ``parity-parallel``
    keeps; see DESIGN.md."""
    w = _Work(m, cfg)
    before = total_elements(m)
    unswap_parity_batched(w, cfg.acceptance == "relaxed", cfg.max_outer_iterations,
                          comm or Comm())
    return _result(w, before)


def unswap(m: MatrixProductOperator, cfg: UnswapConfig, comm: Comm | None = None) -> UnswapResult:
    if cfg.strategy == "sequential":
        return unswap_sequential(m, cfg)
    if cfg.strategy == "parity-batched":
        return unswap_batched(m, cfg, comm)
    return unswap_parallel(m, cfg)
