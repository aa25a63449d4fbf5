"""Device truncated-SVD timing on random complex matrices (CUDA events on the
engine stream), fp64 and fp32, plus accuracy against numpy."""
import sys, time, json
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_21908_b200 as pb
from paper_2604_21908_b200 import _native as nat

nat.load()
sizes = [int(x) for x in (sys.argv[1:] or ["128", "512", "1024", "2048"])]
rng = np.random.default_rng(0)
for n in sizes:
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    # MPO-like spectrum: geometric decay + exact zeros
    u = np.linalg.qr(a)[0]
    v = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))[0]
    s = np.exp(-np.arange(n) / (n / 16))
    s[n // 2:] = 0
    a = (u * s) @ v
    for dt in ("complex128", "complex64"):
        pb.svd_truncate(a, 1, 2e-3, 10**6, dtype=dt)
        c0 = nat.counters()
        t0 = time.perf_counter()
        dec = pb.svd_truncate(a, 1, 2e-3, 10**6, dtype=dt)
        dt_s = time.perf_counter() - t0
        c1 = nat.counters()
        ref = np.sort(s)[::-1] if n > 2048 else np.linalg.svd(a, compute_uv=False)
        k = dec.rank
        err = float(np.max(np.abs(dec.s - ref[:k])) / ref[0])
        print(json.dumps({"n": n, "dtype": dt, "seconds": round(dt_s, 4), "rank": k,
                          "ref_rank": int(pb.tensor.truncation_rank(ref, 2e-3, 10**6)),
                          "max_sigma_err_rel": err,
                          "sweeps": c1["large_sweeps"] - c0["large_sweeps"],
                          "not_converged": c1["svd_not_converged"] - c0["svd_not_converged"]}), flush=True)
