"""Time the large-SVD Gram path per stage (CUDA events around every launch)
on synthetic pair blobs of the contraction's shapes.

    python tools/eig_bench.py [--sizes 512 1024 2048 4096] [--dtype complex128]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_21908_b200 import _native as nat  # noqa: E402
from paper_2604_21908_b200.tensor import svd_truncate  # noqa: E402


def blob(rng, p, kind):
    if kind == "lowrank":  # pair blob through a middle bond of p/4
        k = max(1, p // 4)
        a = (rng.standard_normal((p, k)) + 1j * rng.standard_normal((p, k))) @ \
            (rng.standard_normal((k, p)) + 1j * rng.standard_normal((k, p)))
    else:
        a = rng.standard_normal((p, p)) + 1j * rng.standard_normal((p, p))
    return a / np.linalg.norm(a)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[512, 1024, 2048, 4096])
    ap.add_argument("--dtype", default="complex128")
    ap.add_argument("--kind", default="lowrank")
    a = ap.parse_args()
    nat.load()
    rng = np.random.default_rng(0)
    for p in a.sizes:
        m = blob(rng, p, a.kind)
        svd_truncate(m, 1, 2e-3, 8192, dtype=a.dtype)  # warm-up (allocations)
        nat.synchronize()
        t0 = time.perf_counter()
        svd_truncate(m, 1, 2e-3, 8192, dtype=a.dtype)
        nat.synchronize()
        wall_plain = time.perf_counter() - t0
        nat.profile_begin()
        t0 = time.perf_counter()
        res = svd_truncate(m, 1, 2e-3, 8192, dtype=a.dtype)
        nat.synchronize()
        wall = time.perf_counter() - t0
        nat.profile_end()
        st = nat.profile_eig()
        tot = sum(v["ms"] for v in st.values())
        out = {"p": p, "dtype": a.dtype, "kind": a.kind, "rank": len(res.s), "wall_ms": wall * 1e3, "wall_ms_unprofiled": wall_plain * 1e3,
               "stages_ms": {k: round(v["ms"], 3) for k, v in st.items()},
               "stage_total_ms": round(tot, 3),
               "launches": {k: v["launches"] for k, v in st.items()},
               "gbs": {k: round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) for k, v in st.items() if v["ms"] > 0},
               "tflops": {k: round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2) for k, v in st.items() if v["ms"] > 0}}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
