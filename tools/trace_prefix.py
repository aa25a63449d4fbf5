"""Dump the (phase, unitaries_consumed, elements) trace of the first K
absorption steps of a bench config on the device, for comparison with the
oracle's trace of the same prefix.

    python tools/trace_prefix.py --config c36 --steps 160 --out trace.json
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _instance  # noqa: E402
from paper_2604_21908_b200 import Contraction, ContractionConfig, _native as nat  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c36")
ap.add_argument("--steps", type=int, default=160)
ap.add_argument("--dtype", default="complex128")
ap.add_argument("--out", default="trace.json")
a = ap.parse_args()
nat.load()
inst = _instance(a.config)
job = Contraction(inst.circuit, ContractionConfig(dtype=a.dtype))
job.advance(max_steps=a.steps)
json.dump([(t.phase, t.unitaries_consumed, t.elements) for t in job.trace], open(a.out, "w"))
print(len(job.trace))
