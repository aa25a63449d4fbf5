"""Sharded unswap candidate scoring across the GPUs of one box.

North-star subsystem 3 (reference unswap.py:214-240, paper App. A.1): within
a (side, parity) batch the candidate swaps act on disjoint bond pairs, so
their scores are independent. Each rank keeps a full replica of the chain
(all ranks apply the same accepted swaps, so the replicas stay identical),
scores only its shard of the batch's bonds (bond t of the batch belongs to
rank t mod world), and ONE all-reduce(MAX) over a 2 x nbonds int64 vector
merges the shards (unscored entries are -1). That vector is the only data
that crosses NVLink; the chain never moves.

The loop is written against a small protocol so the same code drives the
device chain (``unswap._Work``) and, in the CPU tests, an oracle-backed chain
under a gloo process group.
"""

from __future__ import annotations

from typing import Protocol

import numpy as np

PARITY_CYCLE = (("both", 0), ("both", 1), ("left", 0), ("left", 1), ("right", 0), ("right", 1))


class Comm:
    """Rank/world plus the one collective; single-process when torch.distributed
    is not initialized (or ``group`` is None and world is 1)."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.rank, self.world = 0, 1
        self.device = device
        try:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized():
                self.rank = dist.get_rank(group)
                self.world = dist.get_world_size(group)
        except ImportError:  # pragma: no cover - torch is always present here
            pass

    def allreduce_max(self, arr: np.ndarray) -> np.ndarray:
        if self.world == 1:
            return arr
        import torch
        import torch.distributed as dist

        dev = self.device
        if dev is None:
            dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()


class BatchWork(Protocol):
    n: int
    bonds: list

    def score_batch(self, bonds, mine, side) -> tuple[np.ndarray, np.ndarray]: ...

    def accept_recenter(self, bond: int, side: str) -> None: ...


def shard_mask(nbonds: int, rank: int, world: int) -> list[int]:
    """Bond t of a batch is scored by rank t mod world."""
    return [1 if t % world == rank else 0 for t in range(nbonds)]


def unswap_parity_batched(work: BatchWork, relaxed: bool, max_outer: int, comm: Comm) -> int:
    """Parity-batched unswapping with batch-level scoring (App. A.1): for each
    (side, parity) batch all candidate extents and baselines are scored on the
    same chain state (sharded over ranks, merged with one all-reduce), then
    every admissible swap (extent < baseline; relaxed: <=) is applied in bond
    order. Stops after a cycle with no bond reduction. Returns the number of
    accepted swaps."""
    n = work.n
    accepted = 0
    for _ in range(max_outer):
        reduced = False
        for side, parity in PARITY_CYCLE:
            bonds = list(range(parity, n - 1, 2))
            if not bonds:
                continue
            mine = shard_mask(len(bonds), comm.rank, comm.world)
            base, ext = work.score_batch(bonds, mine, side)
            merged = comm.allreduce_max(np.concatenate([base, ext]).astype(np.int64))
            base, ext = merged[: len(bonds)], merged[len(bonds):]
            for b, bl, ex in zip(bonds, base, ext):
                if ex < bl or (relaxed and ex == bl):
                    before = work.bonds[b]
                    work.accept_recenter(b, side)
                    accepted += 1
                    if work.bonds[b] < before:
                        reduced = True
        if not reduced:
            break
    return accepted
