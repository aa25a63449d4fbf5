"""Multi-rank path of the sharded unswap scoring (paper_2604_21908_b200/
sharding.py) on CPU: world_size 2 over gloo, with the oracle as the chain
backend, must take exactly the decisions of the single-process run."""

import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mirror_oracle as mo
from paper_2604_21908_b200.sharding import Comm, shard_mask, unswap_parity_batched

EPS, CHI = 1e-10, 4096


class OracleWork:
    """BatchWork over an oracle chain (numpy), same protocol as unswap._Work."""

    def __init__(self, chain):
        self.c = chain
        self.n = len(chain.sites)
        self.bonds = list(chain.bonds())
        self.log = []

    def score_batch(self, bonds, mine, side):
        base = np.full(len(bonds), -1, dtype=np.int64)
        ext = np.full(len(bonds), -1, dtype=np.int64)
        for t, b in enumerate(bonds):
            if not mine[t]:
                continue
            self.c = mo.recenter(self.c, b)
            theta = mo._blob(self.c.sites, b)
            s = np.linalg.svd(theta.reshape(theta.shape[0] * 4, -1), compute_uv=False)
            base[t] = mo.kept_rank(s, EPS, CHI)
            ext[t] = mo.swap_extent(self.c, b, side, EPS, CHI)
        self.c = mo.recenter(self.c, bonds[-1])
        return base, ext

    def accept_recenter(self, bond, side):
        self.c = mo.swap_bond(self.c, bond, side, EPS, CHI)
        self.bonds = list(self.c.bonds())
        self.log.append([bond, side])


def _perm_chain(seed):
    rng = np.random.default_rng(seed)
    perm = tuple(int(x) for x in rng.permutation(7))
    c = mo.identity_chain(7)
    for i, j in reversed(mo.p_factorization(perm)):
        c = mo.absorb(c, mo.OGate("swap", (i, j)), "left", 1e-12, 4096)
    return mo.compress(c, 1e-12, 4096)


def _run(seed, comm):
    w = OracleWork(_perm_chain(seed))
    acc = unswap_parity_batched(w, relaxed=False, max_outer=20, comm=comm)
    return {"accepted": acc, "log": w.log, "bonds": list(w.c.bonds())}


def _worker(rank, world, port, out_dir, seed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run(seed, Comm())
        with open(os.path.join(out_dir, f"r{rank}.json"), "w") as fh:
            json.dump(res, fh)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_mask_partitions_the_batch():
    for world in (1, 2, 3, 8):
        masks = [shard_mask(27, r, world) for r in range(world)]
        assert all(sum(col) == 1 for col in zip(*masks))


def test_single_process_batched_reduces_permutation_to_bond_one():
    res = _run(3, Comm())
    assert res["accepted"] > 0
    assert all(b == 1 for b in res["bonds"])


@pytest.mark.parametrize("seed", [3, 11])
def test_two_rank_gloo_matches_single_process(tmp_path, seed):
    single = _run(seed, Comm())
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), seed), nprocs=2, join=True)
    for r in range(2):
        got = json.loads((tmp_path / f"r{r}.json").read_text())
        assert got == json.loads(json.dumps(single)), r
