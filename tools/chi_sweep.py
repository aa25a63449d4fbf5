#!/usr/bin/env python
"""Max-bond-dimension sweep (BASELINE configs[2]/[4]): contract a bench
instance to its peak with chi_max capped, one JSON line per (config, dtype,
chi_max) point, each bounded by a wall-clock deadline.

    python tools/chi_sweep.py --config c36 --chi 64 128 256 --dtype complex128 complex64
                              [--deadline 120] [--tau 1000000]

A point reports whether the contraction finished inside the deadline, the
wall-clock to peak, the source two-qubit gates absorbed, the largest MPO seen,
the extracted peak against the planted one and its probability (the planted
weight is 0.1: p_peak / 0.1 is the run's fidelity proxy). A capped chain can
stay above tau after an unswap; the driver's stall rule then raises
StallError, reported as such.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402  (instance table)


def point(name, dtype, chi, tau, deadline, stall_limit):
    from paper_2604_21908_b200 import Contraction, ContractionConfig, peak_output, _native as nat
    from paper_2604_21908_b200.driver import StallError

    inst = bench._instance(name)
    cfg = ContractionConfig(dtype=dtype, chi_max=chi, tau=tau, stall_limit=stall_limit)
    nat.synchronize()
    t0 = time.perf_counter()
    job = Contraction(inst.circuit, cfg)
    status, max_el = "timeout", 0
    try:
        while time.perf_counter() - t0 < deadline:
            if job.advance(max_steps=8):
                status = "done"
                break
            max_el = max(max_el, job.m.total_elements())
    except StallError:
        status = "stall"
    out = {"config": name, "qubits": inst.circuit.num_qubits, "dtype": dtype, "chi_max": chi,
           "tau": tau, "status": status, "source_gates": job.consumed_source,
           "source_gates_total": job.source_two_qubit, "unswap_calls": job.unswap_calls,
           "accepted_swaps": job.accepted_swaps, "chi_saturations": job.chi_saturations}
    if job.trace:
        max_el = max(max_el, max(t.elements for t in job.trace))
    out["max_elements"] = max_el
    if status == "done":
        res = job.finish()
        bits, p = peak_output(res)
        nat.synchronize()
        out.update({"peak_bits": bits, "planted": inst.peak, "match": bits == inst.peak,
                    "peak_probability": p})
    nat.synchronize()
    out["seconds"] = time.perf_counter() - t0
    out["gates_per_s"] = job.consumed_source / out["seconds"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c36", choices=sorted(bench.CONFIGS))
    ap.add_argument("--chi", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--dtype", nargs="+", default=["complex128"])
    ap.add_argument("--tau", type=int, default=1_000_000)
    ap.add_argument("--deadline", type=float, default=120.0)
    ap.add_argument("--stall-limit", type=int, default=3)
    a = ap.parse_args()
    for dtype in a.dtype:
        for chi in a.chi:
            print(json.dumps(point(a.config, dtype, chi, a.tau, a.deadline, a.stall_limit)),
                  flush=True)


if __name__ == "__main__":
    main()
