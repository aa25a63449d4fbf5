"""Profile one contraction on the device: per-kernel-class CUDA-event time,
engine counters, trace summary. Used for the profiles/ summaries.

    python tools/profile_run.py --config c20 [--dtype complex64] [--max-steps K] [--chi X]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import CONFIGS, _instance  # noqa: E402
from paper_2604_21908_b200 import Contraction, ContractionConfig, _native as nat  # noqa: E402
from paper_2604_21908_b200.driver import peak_output  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c20", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="complex128")
    ap.add_argument("--max-steps", type=int, default=None)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--side", default="adaptive")
    ap.add_argument("--chi", type=int, default=8192)
    ap.add_argument("--deadline", type=float, default=None, help="stop after this many seconds")
    ap.add_argument("--chunk", type=int, default=8)
    ap.add_argument("--serial", action="store_true", help="sequential adaptive trials")
    ap.add_argument("--trace-out", default=None, help="write the trace records (JSON lines)")
    ap.add_argument("--seed", type=int, default=None, help="instance seed override")
    a = ap.parse_args()
    if a.seed is not None:
        from paper_2604_21908_b200.peaked import generate
        n, depth, w, obf, _, hidden = CONFIGS[a.config]
        inst = generate(n, depth, w, obf, a.seed, hidden_permutation=hidden)
    else:
        inst = _instance(a.config)
    nat.load()
    c0 = nat.counters()
    l0 = nat.launch_count()
    if a.profile:
        nat.profile_begin()
    t0 = time.perf_counter()
    job = Contraction(inst.circuit, ContractionConfig(dtype=a.dtype, side_mode=a.side, chi_max=a.chi,
                                                          concurrent_trials=not a.serial))
    last = t0
    done = False
    while not done:
        done = job.advance(max_steps=a.chunk if a.max_steps is None else min(a.chunk, a.max_steps))
        now = time.perf_counter()
        tr = job.trace[-1] if job.trace else None
        print(f"t={now - t0:8.2f}s steps={job.step} consumed={job.consumed} "
              f"elements={tr.elements if tr else 0} bonds_max={max(job.m.bond_dims() or (1,))} "
              f"unswaps={job.unswap_calls} dt={now - last:.2f}s large={nat.counters()['svd_large']}", flush=True)
        last = now
        if a.max_steps is not None and job.step >= a.max_steps:
            break
        if a.deadline is not None and now - t0 > a.deadline:
            break
    out = {}
    if done:
        res = job.finish()
        out["peak"] = peak_output(res)
        out["planted"] = inst.peak
    nat.synchronize()
    wall = time.perf_counter() - t0
    if a.profile:
        out["profile"] = nat.profile_end()
        out["profile_eig"] = nat.profile_eig()
    c1 = nat.counters()
    out["wall_s"] = wall
    out["launches"] = nat.launch_count() - l0
    out["counters"] = {k: c1[k] - c0.get(k, 0) if k != "max_p" else c1[k] for k in c1}
    out["steps"] = job.step
    out["consumed"] = job.consumed
    out["unswap_calls"] = job.unswap_calls
    out["max_elements"] = max(t.elements for t in job.trace) if job.trace else 0
    if a.trace_out:
        with open(a.trace_out, "w") as f:
            for t in job.trace:
                f.write(json.dumps([t.phase, t.unitaries_consumed, t.elements, round(t.wall_time_s, 3)]) + "\n")
    print(json.dumps(out, indent=1, default=str))


if __name__ == "__main__":
    main()
