"""GPU: sharded unswap scoring through the device path with two ranks.

Two processes (gloo process group over 127.0.0.1) share cuda:0, each holding
a device replica of the chain; the parity-batched unswap shards every
(side, parity) batch's candidate decompositions over the ranks and merges
them with one all-reduce (sharding.py, mb_batch_swap_extents). The ranks'
kernels never wait on each other (the collective runs on host tensors), so
one GPU stands in for two without cross-rank device dependencies.

Asserted: both ranks end with bit-identical results (trace, permutations,
MPS amplitudes), equal to the single-process parity-batched run — i.e. the
sharding changes who computes a decomposition, never a decision — and the
peak is the planted one.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["MB_ROOT"])
import torch.distributed as dist
from paper_2604_21908_b200 import _native as nat
from paper_2604_21908_b200.driver import ContractionConfig, run, dense_output, peak_output
from paper_2604_21908_b200.peaked import generate
from paper_2604_21908_b200.sharding import Comm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
if world > 1:
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["MB_PORT"],
                            rank=rank, world_size=world)
nat.load()
inst = generate(n=12, depth=120, peak_weight=0.2, obfuscation_swaps=24, seed=5)
cfg = ContractionConfig(epsilon=1e-8, chi_max=4096, tau=4000, stall_limit=40,
                        unswap_strategy="parity-batched")
res = run(inst.circuit, cfg, Comm() if world > 1 else None)
vec = dense_output(res)
bits, p = peak_output(res)
out = {"trace": [[t.phase, t.unitaries_consumed, t.elements] for t in res.trace],
       "pi_out": list(res.output_permutation.mapping), "pi_in": list(res.input_permutation.mapping),
       "bits": bits, "planted": inst.peak, "p": p}
np.save(os.environ["MB_OUT"] + f".{rank}.npy", vec)
open(os.environ["MB_OUT"] + f".{rank}.json", "w").write(json.dumps(out))
if world > 1:
    dist.destroy_process_group()
'''


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(world, out, port):
    env = dict(os.environ, MB_ROOT=str(ROOT), MB_OUT=str(out), MB_PORT=str(port),
               WORLD_SIZE=str(world), OMP_NUM_THREADS="1")
    procs = [subprocess.Popen([sys.executable, "-c", WORKER], env=dict(env, RANK=str(r)))
             for r in range(world)]
    for p in procs:
        assert p.wait(timeout=600) == 0


def test_two_ranks_match_single_process(tmp_path):
    _launch(1, tmp_path / "single", _free_port())
    _launch(2, tmp_path / "pair", _free_port())
    ref = json.loads((tmp_path / "single.0.json").read_text())
    ref_vec = np.load(tmp_path / "single.0.npy")
    assert ref["bits"] == ref["planted"]
    for r in range(2):
        got = json.loads((tmp_path / f"pair.{r}.json").read_text())
        assert got["trace"] == ref["trace"], f"rank {r} trace differs"
        assert got["pi_out"] == ref["pi_out"] and got["pi_in"] == ref["pi_in"]
        assert got["bits"] == ref["bits"]
        np.testing.assert_array_equal(np.load(tmp_path / f"pair.{r}.npy"), ref_vec)
