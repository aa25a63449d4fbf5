"""Per-call host wall time of the small-chain engine operations (the latency
floor of absorb_2q / compress / trial on chains with tiny bonds).

    python tools/micro_absorb.py [n_sites] [calls]
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_21908_b200 import _native as nat  # noqa: E402
from paper_2604_21908_b200.chains import absorb_gate_inplace, identity_mpo  # noqa: E402
from paper_2604_21908_b200.circuit import Gate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 400
nat.load()
rng = np.random.default_rng(0)
m = identity_mpo(n)
gates = [Gate("rzz", (int(a), int(a) + 1), (float(t),)) for a, t in
         zip(rng.integers(0, n - 1, calls), rng.uniform(-3, 3, calls))]
for g in gates[:20]:
    absorb_gate_inplace(m, g, "left", 2e-3, 8192)
nat.synchronize()
t0 = time.perf_counter()
for g in gates:
    absorb_gate_inplace(m, g, "left", 2e-3, 8192)
nat.synchronize()
t1 = time.perf_counter()
for _ in range(50):
    nat.check(nat._lib.mb_compress(m._h, 2e-3, 8192), "compress")
nat.synchronize()
t2 = time.perf_counter()
c0 = nat.counters()
print({"sites": n, "bonds": m.bond_dims(), "absorb_2q_us": round((t1 - t0) / calls * 1e6, 1),
       "compress_us": round((t2 - t1) / 50 * 1e6, 1), "launches": nat.launch_count(), "counters": c0})
