"""Run the tcgen05 complex64 GEMM (3xTF32) once at a size above the routing
threshold and report achieved throughput (for the ncu tensor-pipe capture).

    python tools/tc_gemm_probe.py [m n k]
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_21908_b200 import _native as nat  # noqa: E402
from paper_2604_21908_b200.tensor import device_gemm  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 2048, 2048)
nat.load()
rng = np.random.default_rng(0)
a = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
ref = a @ b
c = device_gemm(a, b, "complex64", tensor_cores=True)
err = float(np.abs(c - ref).max() / np.abs(ref).max())
t0 = time.perf_counter()
for _ in range(3):
    device_gemm(a, b, "complex64", tensor_cores=True)
dt = (time.perf_counter() - t0) / 3
print({"m": m, "n": n, "k": k, "rel_err": err, "host_s_incl_copies": dt})
