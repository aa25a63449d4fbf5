"""Stream the oracle's trace of a bench instance (the bit-exact restatement
of the reference algorithm, pinned by test_oracle_golden.py) record by
record, with each record's bond dimensions and CPU wall time, into a JSON
Lines file. Used to extend the large-bond parity fixtures past the c36
prefix: run it unattended for hours, then cut a fixture from its output
with --fixture.

    python tests/golden/make_long_trace.py --config c36 --out /tmp/c36_oracle.jsonl
    python tests/golden/make_long_trace.py --fixture /tmp/c36_oracle.jsonl --steps N
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def stream(config, out):
    import bench
    from oracle import mirror_oracle as mo

    n, gates = bench._oracle_circuit(config)
    t0 = time.perf_counter()
    with open(out, "w") as f:
        def rec(r, c):
            f.write(json.dumps({"rec": list(r), "bonds": [int(b) for b in c.bonds()],
                                "t": round(time.perf_counter() - t0, 3)}) + "\n")
            f.flush()
        res = mo.contract(n, gates, mo.OConfig(), on_record=rec)
        f.write(json.dumps({"done": True, "peak": mo.peak_result(res)[0],
                            "t": time.perf_counter() - t0}) + "\n")


def fixture(src, steps, config):
    rows = [json.loads(x) for x in open(src) if x.strip()]
    recs = [r for r in rows if "rec" in r]
    absorbs = 0
    keep = []
    for r in recs:
        if r["rec"][0] == "absorb":
            absorbs += 1
            if absorbs > steps:
                break
        keep.append(r)
    out = {"config": config, "steps": absorbs if absorbs <= steps else steps,
           "trace": [r["rec"] for r in keep], "max_bond": max(max(r["bonds"]) for r in keep)}
    dst = Path(__file__).parent / f"{config}_prefix{out['steps']}_trace.json"
    dst.write_text(json.dumps(out))
    print(dst, len(keep), out["max_bond"])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c36")
    ap.add_argument("--out")
    ap.add_argument("--fixture")
    ap.add_argument("--steps", type=int, default=0)
    a = ap.parse_args()
    if a.fixture:
        fixture(a.fixture, a.steps, a.config)
    else:
        stream(a.config, a.out)
