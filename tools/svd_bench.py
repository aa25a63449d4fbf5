"""Device truncated-SVD timing on random complex matrices (engine counters +
host wall clock), fp64 and fp32, plus accuracy against the known spectrum.

    python tools/svd_bench.py [--kind graded|gauss|mpo] [--dtypes c128,c64] n1 n2 ...
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_21908_b200 as pb  # noqa: E402
from paper_2604_21908_b200 import _native as nat  # noqa: E402
from paper_2604_21908_b200.tensor import truncation_rank  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("sizes", nargs="*", type=int, default=[128, 512, 1024])
ap.add_argument("--kind", default="graded")
ap.add_argument("--dtypes", default="complex128,complex64")
a = ap.parse_args()
nat.load()
rng = np.random.default_rng(0)


def haar(n):
    return np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))[0]


for n in a.sizes:
    if a.kind == "gauss":
        s = np.sort(rng.chisquare(2, n))[::-1] ** 0.5
    elif a.kind == "mpo":  # degenerate plateaus + exact zeros (permutation-like)
        s = np.repeat([1.0, 0.5, 0.25, 0.125], n // 8)
        s = np.concatenate([s, np.zeros(n - len(s))])
    else:  # geometric decay + exact null space
        s = np.exp(-np.arange(n) / (n / 16))
        s[n // 2:] = 0
    mat = (haar(n) * s) @ haar(n)
    ref = np.sort(s)[::-1]
    for dt in a.dtypes.split(","):
        pb.svd_truncate(mat, 1, 2e-3, 10**6, dtype=dt)
        c0 = nat.counters()
        t0 = time.perf_counter()
        dec = pb.svd_truncate(mat, 1, 2e-3, 10**6, dtype=dt)
        secs = time.perf_counter() - t0
        c1 = nat.counters()
        k = dec.rank
        print(json.dumps({"kind": a.kind, "n": n, "dtype": dt, "seconds": round(secs, 4),
                          "rank": k, "ref_rank": truncation_rank(ref, 2e-3, 10**6),
                          "max_sigma_err_rel": float(np.max(np.abs(dec.s - ref[:k])) / ref[0]),
                          "sweeps": c1["large_sweeps"] - c0["large_sweeps"],
                          "not_converged": c1["svd_not_converged"] - c0["svd_not_converged"]}),
              flush=True)
