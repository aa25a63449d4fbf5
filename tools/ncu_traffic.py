"""Per-kernel DRAM traffic from an `ncu --set full` report, next to the
kernel's algorithmic bytes, for profiles/r02_kernel_traffic.json (the bench
line's roofline `traffic` field).

    ncu -i gpurun_out/prof.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_traffic.py raw.csv --out profiles/r02_kernel_traffic.json --p 4096

Algorithmic bytes per launch (what the kernel must move at minimum):
  k_symv_tiles  : one 64 x 64 complex128 tile per CTA -> grid * 64 KiB
                  (diagonal tiles read half; counted in full: an upper bound)
  k_gemm_cm     : reported as dram / flop-equivalent only (compute-bound)
  other kernels : dram bytes only
"""
import argparse
import csv
import json
import re
import statistics
from collections import defaultdict


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--out", required=True)
    ap.add_argument("--p", type=int, default=None, help="problem size of the capture")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    need = ["Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]
    for k in need:
        if k not in idx:
            raise SystemExit(f"missing column {k}")
    grid_col = next((h for h in hdr if h in ("launch__grid_size", "Grid Size")), None)
    units = rows[1]
    scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    scale_t = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
    fb_r = scale_b.get(units[idx["dram__bytes_read.sum"]], 1)
    fb_w = scale_b.get(units[idx["dram__bytes_write.sum"]], 1)
    ft = scale_t.get(units[idx["gpu__time_duration.sum"]], 1)
    per = defaultdict(list)
    for r in rows[2:]:  # row 1 holds units
        if len(r) < len(hdr):
            continue
        name = r[idx["Kernel Name"]]
        short = re.sub(r"[<(].*", "", re.sub(r"^void ", "", name)).strip()
        rd, wr = num(r[idx["dram__bytes_read.sum"]]), num(r[idx["dram__bytes_write.sum"]])
        t = num(r[idx["gpu__time_duration.sum"]])
        rd = rd * fb_r if rd is not None else None
        wr = wr * fb_w if wr is not None else None
        t = t * ft if t is not None else None
        grid = num(r[idx[grid_col]]) if grid_col else None
        if rd is None or wr is None:
            continue
        per[short].append((rd + wr, t, grid, name))
    out = {"source": "ncu --set full --clock-control none", "problem_p": a.p, "kernels": {}}
    for k, v in per.items():
        dram = statistics.mean(x[0] for x in v)
        ent = {"launches_captured": len(v), "dram_bytes_per_launch": dram,
               "gpu_time_ns_mean": statistics.mean(x[1] for x in v if x[1] is not None) if v else None,
               "example": v[0][3][:160]}
        if k == "k_symv_tiles" and v[0][2]:
            alg = statistics.mean(x[2] * 64 * 64 * 16 for x in v)
            ent["algorithmic_bytes_per_launch"] = alg
            ent["dram_over_algorithmic"] = dram / alg if alg else None
        out["kernels"][k] = ent
    open(a.out, "w").write(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
