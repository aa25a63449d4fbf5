#!/usr/bin/env python
"""fp32-vs-fp64 fidelity check of the middle MPO (BASELINE configs[2]).

Runs the same contraction prefix in complex64 and complex128 and reports the
normalized Hilbert-Schmidt overlap of the two operators,

    F = |Tr(M32^H M64)|^2 / (Tr(M32^H M32) Tr(M64^H M64)),

computed as a transfer-matrix sweep over the sites (E <- sum_d A_d^H E B_d,
renormalized per site) with torch complex128 matmuls — a checker, not the
product path. F = 1 means the two runs hold the same operator up to a
global scalar.

    python tools/mpo_fidelity.py --config c36 --steps 160
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def hs_overlap(sa, sb, device="cpu"):
    """(log|<A,B>|, phase) of Tr(A^H B) for two MPOs given as host site lists
    of shape (l, 2, 2, r); bond dims of A and B may differ."""
    import numpy as np
    import torch

    e = torch.ones((1, 1), dtype=torch.complex128, device=device)
    logscale = 0.0
    for a, b in zip(sa, sb):
        ta = torch.from_numpy(np.ascontiguousarray(a).reshape(a.shape[0], 4, a.shape[-1])).to(device)
        tb = torch.from_numpy(np.ascontiguousarray(b).reshape(b.shape[0], 4, b.shape[-1])).to(device)
        # E'[ra, rb] = sum_{la, d} conj(A[la, d, ra]) (E B)[la, d, rb]
        eb = (e @ tb.reshape(tb.shape[0], -1)).reshape(e.shape[0], 4, tb.shape[-1])
        e = ta.conj().reshape(-1, ta.shape[-1]).T @ eb.reshape(-1, tb.shape[-1])
        s = float(e.abs().max())
        if s == 0.0:
            return float("-inf"), 1.0
        e = e / s
        logscale += np.log(s)
    v = complex(e[0, 0])
    return logscale + np.log(abs(v)), v / abs(v)


def fidelity(ma, mb, device="cpu") -> float:
    import numpy as np

    sa, sb = ma.sites, mb.sites
    lab, _ = hs_overlap(sa, sb, device)
    laa, _ = hs_overlap(sa, sa, device)
    lbb, _ = hs_overlap(sb, sb, device)
    return float(np.exp(2 * lab - laa - lbb))


def run_pair(name: str, steps: int, device: str):
    from bench import _instance
    from paper_2604_21908_b200 import Contraction, ContractionConfig

    out = {"config": name, "steps": steps}
    jobs = {}
    for dt in ("complex64", "complex128"):
        t0 = time.perf_counter()
        job = Contraction(_instance(name).circuit, ContractionConfig(dtype=dt))
        job.advance(max_steps=steps)
        out[f"seconds_{dt}"] = round(time.perf_counter() - t0, 2)
        jobs[dt] = job
    t32 = [(t.phase, t.unitaries_consumed, t.elements) for t in jobs["complex64"].trace]
    t64 = [(t.phase, t.unitaries_consumed, t.elements) for t in jobs["complex128"].trace]
    out["same_trace"] = t32 == t64
    out["records"] = len(t64)
    out["elements"] = [jobs["complex64"].m.total_elements(), jobs["complex128"].m.total_elements()]
    out["max_bond"] = max(jobs["complex128"].m.bond_dims())
    out["fidelity"] = fidelity(jobs["complex64"].m, jobs["complex128"].m, device)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c36")
    ap.add_argument("--steps", type=int, nargs="+", default=[40, 80, 160])
    ap.add_argument("--device", default="cuda")
    a = ap.parse_args()
    for s in a.steps:
        print(json.dumps(run_pair(a.config, s, a.device)), flush=True)


if __name__ == "__main__":
    main()
