#!/usr/bin/env python
"""Benchmark: middle-MPO contraction of a peaked circuit to its peak
bitstring on B200 (BASELINE.json metric).

Default workload: configs[1], the 20-qubit peaked circuit with swap
insertion (the largest configuration whose full contraction both the B200
arm and the CPU reference arm complete; its trace is golden-verified against
the reference). ``--config c56`` runs the 56-qubit H2-scale instance
(configs[3]) — see DESIGN.md for its status.

One step = contract the whole circuit (route, split, absorb/unswap/rewire
loop, apply to |0..0>) and extract the peak on the device. ``value`` is
source two-qubit gates absorbed per second over the K timed steps (the
metric's "gates absorbed/s"); ``ms_per_step`` is the wall-clock to peak.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c56|c36|c20|c12] [--dtype complex128|complex64]

Under torchrun (N>1) every rank holds a replica of the chain and the
unswap candidate scoring of each parity batch is sharded over the ranks,
merged by one NCCL all-reduce (sharding.py): one contraction per step,
scaling "strong", value = its gates / max-over-ranks time. ``--impl reference`` times the CPU
reference arm (the oracle restatement of the reference algorithm, bit-exact
with it) on a bounded prefix of the same contraction, on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (n, depth, peak_weight, obfuscation_swaps, seed, hidden_permutation)
    "c12": (12, 120, 0.1, 0, 7, False),
    "c20": (20, 200, 0.1, 20, 1, True),
    "c36": (36, 700, 0.1, 40, 1, True),
    "c56": (56, 1917, 0.1, 60, 1, True),
}
METRIC = "wall-clock to peak for 56q circuit (1 B200); gates absorbed/s; TC util & HBM GB/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c20")
    ap.add_argument("--dtype", choices=["complex128", "complex64"], default="complex128")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0,
                    help="CPU work per reference-arm sample (seconds, approx.)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def _instance(name):
    from paper_2604_21908_b200.peaked import generate

    n, depth, w, obf, seed, hidden = CONFIGS[name]
    return generate(n, depth, w, obf, seed, hidden_permutation=hidden)


def _workload(name, dtype):
    n, depth, w, obf, seed, hidden = CONFIGS[name]
    return {"workload": f"{n}q peaked circuit, middle-MPO contraction + peak extraction",
            "config": name, "qubits": n, "depth_budget": depth, "obfuscation_swaps": obf,
            "seed": seed, "epsilon": 2e-3, "chi_max": 8192, "tau": 1_000_000,
            "side_mode": "adaptive", "dtype": dtype,
            "l2": "working set re-created every step (fresh MPO per contraction)"}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self):
        self.rows, self._stop, self._t = [], threading.Event(), None

    def start(self):
        def loop():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    dev = os.environ.get("MB_DEVICE", os.environ.get("LOCAL_RANK", "0"))
                    out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", dev],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    row = [x.strip() for x in out.split(",")] if out else []
                    if len(row) >= 7:
                        self.rows.append(row)
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def _oracle_circuit(name):
    from oracle import mirror_oracle as mo

    inst = _instance(name)
    gates = tuple(mo.OGate(g.kind, g.qubits, g.params, g.origin != "source")
                  for g in inst.circuit.gates)
    return inst.circuit.num_qubits, gates


def cpu_prefix_steps(name, budget_s):
    """Number of absorption steps of the CPU reference arm that costs about
    budget_s seconds (doubling search; untimed). None = the whole job fits."""
    from oracle import mirror_oracle as mo

    n, gates = _oracle_circuit(name)
    steps = 4
    while True:
        t0 = time.perf_counter()
        res = mo.contract(n, gates, mo.OConfig(), max_steps=steps)
        spent = time.perf_counter() - t0
        if res.state is not None:
            return None
        if spent >= budget_s / 2.5 or steps >= 1 << 14:
            return steps
        steps *= 2


def cpu_reference(name, steps):
    """Time the CPU reference arm (the oracle: the reference's algorithm and
    numpy/OpenBLAS calls, bit-exact with it) on the first `steps` absorption
    steps of the same contraction (or the whole job if steps is None)."""
    from oracle import mirror_oracle as mo

    n, gates = _oracle_circuit(name)
    # every host thread (torchrun sets OMP_NUM_THREADS=1 for its ranks);
    # report what the BLAS pool actually runs with
    threads = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_info, threadpool_limits

        ctx = threadpool_limits(limits=threads, user_api="blas")
        info = [p for p in threadpool_info() if p.get("user_api") == "blas"]
        if info:
            threads = int(info[0].get("num_threads", threads))
    except ImportError:  # pragma: no cover - threadpoolctl is in the image
        ctx = None
    t0 = time.perf_counter()
    res = mo.contract(n, gates, mo.OConfig(), max_steps=steps)
    spent = time.perf_counter() - t0
    if ctx is not None:
        ctx.restore_original_limits()
    return {"seconds": spent, "absorb_steps": steps, "source_gates": res.consumed_source,
            "value": res.consumed_source / spent if spent > 0 else 0.0, "threads": threads,
            "complete": res.state is not None}


def gpu_prefix(name, dtype, steps):
    """The same bounded prefix on the device (for an apples-to-apples line)."""
    from paper_2604_21908_b200 import Contraction, ContractionConfig, _native as nat

    inst = _instance(name)
    job = Contraction(inst.circuit, ContractionConfig(dtype=dtype))
    nat.synchronize()
    t0 = time.perf_counter()
    job.advance(max_steps=steps)
    nat.synchronize()
    dt = time.perf_counter() - t0
    return {"seconds": dt, "source_gates": job.consumed_source,
            "value": job.consumed_source / dt if dt > 0 else 0.0}


def _sample_text(name, r):
    what = (f"first {r['absorb_steps']} absorption steps" if r["absorb_steps"] is not None
            else "the complete contraction")
    return (f"{what} ({r['source_gates']} source two-qubit gates) of the {name} contraction, "
            f"{r['seconds']:.1f} s, numpy/OpenBLAS {r['threads']} threads")


def run_reference(args, rank, world):
    if rank != 0:
        return
    steps = cpu_prefix_steps(args.config, args.cpu_sample_s)
    timed = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference(args.config, steps)
        if i >= args.warmup:
            timed.append(r)
    val = statistics.mean(r["value"] for r in timed)
    ms = statistics.mean(r["seconds"] for r in timed) * 1e3
    line = {"metric": METRIC, "value": val, "unit": "source 2q gates absorbed/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (reference generator, seeded)",
            "config": _workload(args.config, "complex128"),
            "cpu_baseline": {"value": val, "unit": "source 2q gates absorbed/s",
                             "cores": timed[-1]["threads"], "kind": "port",
                             "sample": _sample_text(args.config, timed[-1])},
            "e2e": {"value": val, "unit": "source 2q gates absorbed/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


_CLASS_KERNEL = {"svd_small": "k_sweep", "svd_large": "k_jacobi_pair_cl", "gemm": "k_gemm"}


def _traffic(cls):
    """DRAM bytes per launch of the class's dominant kernel, from the committed
    ncu --set full capture (profiles/r01_kernel_traffic.json), else None."""
    p = ROOT / "profiles" / "r01_kernel_traffic.json"
    try:
        k = json.loads(p.read_text())["kernels"].get(_CLASS_KERNEL.get(cls, ""))
    except (OSError, ValueError, KeyError):
        return None
    return None if k is None else {"kernel": _CLASS_KERNEL[cls], "dram_bytes_per_launch": k["mean"]}


def _phase_seconds(trace):
    """Host wall time per phase of one contraction, from the trace's
    cumulative stamps (absorb steps vs unswap calls)."""
    out = {"absorb": 0.0, "unswap": 0.0}
    prev = 0.0
    for t in trace:
        out[t.phase] = out.get(t.phase, 0.0) + (t.wall_time_s - prev)
        prev = t.wall_time_s
    return {k: round(v, 4) for k, v in out.items()}


def main():
    args = _args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_

        dist = dist_
        backend = "gloo" if args.impl == "reference" else os.environ.get("MB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("MB_DEVICE", local)))
        dist.init_process_group(backend=backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.destroy_process_group()
        return

    import torch

    from paper_2604_21908_b200 import Contraction, ContractionConfig, _native as nat
    from paper_2604_21908_b200.circuit import parse_qasm, serialize_qasm
    from paper_2604_21908_b200.driver import peak_output

    from paper_2604_21908_b200.sharding import Comm

    torch.cuda.set_device(int(os.environ.get("MB_DEVICE", local)))
    nat.load()
    stream = torch.cuda.ExternalStream(nat.stream_handle())
    inst = _instance(args.config)
    qasm = serialize_qasm(inst.circuit)
    # N = 1: the reference's bond-by-bond unswap order (golden-trace parity).
    # N > 1: every rank holds a replica of the chain and the parity batches'
    # candidate scoring is sharded over ranks, merged by one NCCL all-reduce.
    comm = Comm() if world > 1 else None
    cfg = ContractionConfig(dtype=args.dtype,
                            unswap_strategy="parity-batched" if world > 1 else "parity-parallel")
    n2q = inst.circuit.two_qubit_count()

    def one_step():
        job = Contraction(inst.circuit, cfg, comm)
        job.advance()
        res = job.finish()
        return job, peak_output(res)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        nat.synchronize()

    for _ in range(args.warmup):
        one_step()
    barrier()

    # ---- timed region: device-resident path (circuit already loaded) ----
    clocks = Clocks()
    clocks.start()
    launches0 = nat.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    peaks, jobs = [], []
    for _ in range(args.steps):
        job, pk = one_step()
        peaks.append(pk)
        jobs.append(job)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    dev_ms = ev0.elapsed_time(ev1)
    launches = nat.launch_count() - launches0
    t_dev = "cuda" if not dist or dist.get_backend() == "nccl" else "cpu"
    t_max = torch.tensor([dev_ms], dtype=torch.float64, device=t_dev)
    if dist:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    dev_ms = float(t_max.item())
    total_gates = n2q * args.steps  # one (replicated) contraction per step
    value = total_gates / (dev_ms / 1e3)

    # ---- e2e: through the public API from QASM text to the host bitstring ----
    from paper_2604_21908_b200 import peak_output as _po
    c0 = nat.counters()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        circ = parse_qasm(qasm)
        job = Contraction(circ, cfg, comm)
        job.advance()
        bits, p = _po(job.finish())
    e1.record(stream)
    barrier()
    c1 = nat.counters()
    e2e_ms = e0.elapsed_time(e1)
    t_e2e = torch.tensor([e2e_ms], dtype=torch.float64, device=t_dev)
    if dist:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_ms = float(t_e2e.item())
    h2d = (c1["h2d_bytes"] - c0["h2d_bytes"]) // args.steps + len(qasm)
    d2h = (c1["d2h_bytes"] - c0["d2h_bytes"]) // args.steps

    # ---- one profiled (untimed) step: per-kernel-class device time ----
    nat.profile_begin()
    one_step()
    prof = nat.profile_end()
    hbm, bf16, src = _peaks()
    dom = max(prof, key=lambda k: prof[k]["ms"])
    tot_ms = sum(v["ms"] for v in prof.values())
    d = prof[dom]
    achieved_tf = d["flops"] / (d["ms"] / 1e3) / 1e12 if d["ms"] > 0 else 0.0

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "source 2q gates absorbed/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "c128" if args.dtype == "complex128" else "c64",
            "data": "synthetic (reference generator, seeded)",
            "config": dict(_workload(args.config, args.dtype),
                           parallelism=(f"sharded unswap scoring x{world} (NCCL all-reduce)"
                                        if world > 1 else "1 GPU"),
                           unswap_order="parity-batched" if world > 1 else "parity-parallel"),
            "peak": {"bits": peaks[-1][0], "probability": peaks[-1][1],
                     "planted": inst.peak, "match": peaks[-1][0] == inst.peak},
            "two_qubit_gates": n2q,
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": {"value": total_gates / (e2e_ms / 1e3), "unit": "source 2q gates absorbed/s",
                    "ms_per_step": e2e_ms / args.steps,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "roofline": {"bound": "tensor", "kernel_class": dom, "achieved": achieved_tf,
                         "peak": bf16, "unit": "TFLOP/s", "frac": achieved_tf / bf16,
                         "traffic": _traffic(dom), "peak_source": src,
                         "share_of_device_time": d["ms"] / tot_ms if tot_ms else None,
                         "note": "fp64/fp32 CUDA-core Jacobi + GEMM vs the bf16 tensor peak"},
            "profile_ms": {k: round(v["ms"], 3) for k, v in prof.items()},
            "contraction": {"trace_records": len(jobs[-1].trace), "unswap_calls": jobs[-1].unswap_calls,
                            "phase_s": _phase_seconds(jobs[-1].trace),
                            "accepted_swaps": jobs[-1].accepted_swaps,
                            "max_elements": max(t.elements for t in jobs[-1].trace)},
            "counters": nat.counters(),
        }
        if not args.no_cpu_baseline and world == 1:
            steps = cpu_prefix_steps(args.config, args.cpu_sample_s)
            ref = cpu_reference(args.config, steps)
            pre = gpu_prefix(args.config, args.dtype, steps)
            line["cpu_baseline"] = {"value": ref["value"], "unit": "source 2q gates absorbed/s",
                                    "cores": ref["threads"], "kind": "port",
                                    "sample": _sample_text(args.config, ref),
                                    "b200_same_sample": pre["value"],
                                    "b200_same_sample_speedup": pre["value"] / ref["value"]
                                    if ref["value"] else None}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
