"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: count, share of summed device time, mean per launch.

    python tools/summarize_launches.py launches.csv "command line" > summary.txt
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
cmd = sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    name = re.sub(r"^void ", "", r[4])
    name = re.sub(r"\(.*$", "", name)
    agg[name][0] += 1
    agg[name][1] += float(r[14].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none")
print(f"command: {cmd}")
print("per-launch times are cold-cache and serialised: compare SHARES, not absolutes")
print(f"launches={len(rows)} total_ns={tot:.0f}")
print(f"{'kernel':60s} {'n':>7s} {'share':>6s} {'avg_us':>9s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {n:7d} {t / tot:6.3f} {t / n / 1e3:9.2f}")
