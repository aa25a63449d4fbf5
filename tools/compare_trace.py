"""Compare a device trace (profile_run.py --trace-out) with the oracle's
streamed trace (tests/golden/make_long_trace.py): first divergent record.

    python tools/compare_trace.py device.jsonl oracle.jsonl
"""
import json
import sys


def load(path):
    out = []
    for line in open(path):
        if not line.strip():
            continue
        r = json.loads(line)
        if isinstance(r, dict):
            if "rec" not in r:
                continue
            r = r["rec"]
        out.append(tuple(r[:3]))
    return out


def main():
    dev, orc = load(sys.argv[1]), load(sys.argv[2])
    n = min(len(dev), len(orc))
    for i in range(n):
        if dev[i] != orc[i]:
            print(f"first divergence at record {i}: device {dev[i]} oracle {orc[i]}")
            print(f"records compared: {n}; identical prefix {i}")
            return 1
    print(f"identical over {n} records (device {len(dev)}, oracle {len(orc)})")
    return 0


if __name__ == "__main__":
    sys.exit(main())
