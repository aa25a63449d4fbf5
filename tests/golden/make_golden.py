"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``mirrorbreak`` from /root/reference/pkg/src, runs it on seeded
inputs and writes ``golden.json`` + ``golden.npz`` next to this file. The
fixtures are committed; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF))

import mirrorbreak.driver as driver  # noqa: E402
import mirrorbreak.peaked as peaked  # noqa: E402
import mirrorbreak.routing as routing  # noqa: E402
import mirrorbreak.tensor as tensor  # noqa: E402
import mirrorbreak.unswap  # noqa: E402,F401
unswap = sys.modules["mirrorbreak.unswap"]
from mirrorbreak.circuit import Circuit, Gate, inverse_circuit, serialize_qasm  # noqa: E402
from mirrorbreak.oracle import peak_of, simulate  # noqa: E402
from tests.oracles import random_circuit  # noqa: E402  (reference test helper)
from tests.test_unswap import permutation_mpo  # noqa: E402

OUT = Path(__file__).resolve().parent
arrays: dict[str, np.ndarray] = {}


def cfg_dict(cfg):
    return {k: getattr(cfg, k) for k in ("epsilon", "chi_max", "tau", "max_unswap_iterations",
                                         "acceptance", "unswap_strategy", "side_mode",
                                         "stall_limit")}


def unobfuscated_mirror(n, depth, peak_weight, seed):
    """configs[0]: U U^dagger with a planted peak, no hidden permutation and no
    swaps; built from the reference generator's own pieces."""
    rng = np.random.default_rng(seed)
    peak = "".join("1" if rng.random() < 0.5 else "0" for _ in range(n))
    fwd = peaked._random_brickwork(n, max(n // 2, depth // 2), rng)
    dil = []
    if peak_weight < 1.0:
        ang = 2.0 * np.arccos(peak_weight ** (1.0 / (2 * n)))
        for q in range(n):
            kind = "rx" if rng.random() < 0.5 else "ry"
            sign = 1.0 if rng.random() < 0.5 else -1.0
            dil.append(Gate(kind, (q,), (float(sign * ang),)))
    xs = [Gate("x", (q,)) for q in range(n) if peak[q] == "1"]
    gates = tuple(fwd) + inverse_circuit(Circuit(n, tuple(fwd))).gates + tuple(xs) + tuple(dil)
    return Circuit(n, gates), peak


def run_case(name, circuit, cfg, peak=None, dense=True):
    res = driver.run(circuit, cfg)
    case = {
        "name": name,
        "qasm": serialize_qasm(circuit),
        "config": cfg_dict(cfg),
        "trace": [[r.phase, r.unitaries_consumed, r.elements] for r in res.trace],
        "final_elements": res.final_elements,
        "chi_saturation_events": res.chi_saturation_events,
        "pi_out": list(res.output_permutation.mapping),
        "pi_in": list(res.input_permutation.mapping),
        "state_bonds": list(res.state.bond_dims()),
        "state_log_norm": res.state.log_norm,
        "samples_seed9": driver.sample_output(res, 200, seed=9),
        "planted_peak": peak,
    }
    shots = driver.sample_output(res, 1000, seed=3)
    counts = {}
    for s in shots:
        counts[s] = counts.get(s, 0) + 1
    case["top1000_seed3"] = sorted(counts.items(), key=lambda kv: (-kv[1], kv[0]))[0]
    if circuit.num_qubits <= 12 and dense:
        vec = driver.dense_output(res)
        arrays[f"{name}__dense"] = vec
        ref = simulate(circuit)
        case["oracle_peak"], case["oracle_peak_prob"] = peak_of(ref)
        case["fidelity_vs_statevector"] = float(abs(np.vdot(ref, vec)) ** 2)
    print(name, "trace", len(case["trace"]), "final", res.final_elements, flush=True)
    return case


def main():
    gold = {"svd": [], "circuits": [], "unswap": [], "routing": [], "generator": []}

    # ---- truncated SVD (tensor.py:84) -------------------------------------
    rng = np.random.default_rng(123)
    shapes = [(8, 8), (6, 10), (12, 5), (64, 64), (100, 37), (37, 100)]
    for k, shp in enumerate(shapes):
        a = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
        arrays[f"svd{k}"] = a
        s_all = np.linalg.svd(a, compute_uv=False)
        rows = []
        for eps, chi in [(0.0, 10**6), (1e-10, 10**6), (0.3, 10**6), (0.6, 3), (0.05, 10**6)]:
            dec = tensor.svd_truncate(a, 1, eps, chi)
            rows.append({"eps": eps, "chi": chi, "rank": dec.rank,
                         "discarded": dec.discarded_weight})
        gold["svd"].append({"key": f"svd{k}", "s": s_all.tolist(), "cuts": rows})
    # degenerate spectrum straddling the cut (ties kept together)
    s = np.array([1.0, 0.5, 0.5, 0.5, 1e-9])
    u = np.linalg.qr(rng.standard_normal((5, 5)))[0]
    v = np.linalg.qr(rng.standard_normal((5, 5)))[0]
    a = ((u * s) @ v).astype(complex)
    arrays["svd_deg"] = a
    eps = float(np.sqrt((0.5 ** 2 + 1e-18) / (s ** 2).sum()) * 1.001)
    dec = tensor.svd_truncate(a, 1, eps, 5)
    gold["svd"].append({"key": "svd_deg", "s": np.linalg.svd(a, compute_uv=False).tolist(),
                        "cuts": [{"eps": eps, "chi": 5, "rank": dec.rank,
                                  "discarded": dec.discarded_weight}]})

    # ---- routing (routing.py:385) -----------------------------------------
    for k in range(12):
        r2 = np.random.default_rng(500 + k)
        n = int(r2.integers(3, 9))
        c = random_circuit(n, int(r2.integers(4, 16)), r2)
        fw = routing.route_linear(c, "forward")
        rv = routing.route_linear(c, "reverse")
        gold["routing"].append({
            "qasm": serialize_qasm(c),
            "forward": [[g.kind, list(g.qubits), g.origin] for g in fw.circuit.gates],
            "forward_out": list(fw.output_layout.mapping),
            "reverse": [[g.kind, list(g.qubits), g.origin] for g in rv.circuit.gates],
            "reverse_in": list(rv.input_layout.mapping),
        })

    # ---- unswapping on permutation chains (unswap.py:170, 214) --------------
    cfgs = {"sequential": unswap.UnswapConfig(epsilon=1e-10, chi_max=4096),
            "parity-parallel": unswap.UnswapConfig(epsilon=1e-10, chi_max=4096,
                                                   strategy="parity-parallel")}
    for k in range(10):
        r2 = np.random.default_rng(1900 + k)
        n = int(r2.integers(3, 8))
        perm = routing.QubitPermutation(tuple(int(x) for x in r2.permutation(n)))
        side = "left" if k % 2 == 0 else "right"
        m = permutation_mpo(perm, side)
        for strat, cfg in cfgs.items():
            res = unswap.unswap(m, cfg)
            gold["unswap"].append({
                "perm": list(perm.mapping), "side": side, "strategy": strat,
                "accepted": res.accepted_swaps, "left": list(res.left_perm.mapping),
                "right": list(res.right_perm.mapping),
                "bonds_before": list(m.bond_dims()), "bonds_after": list(res.reduced.bond_dims()),
                "elements_before": res.elements_before, "elements_after": res.elements_after,
            })

    # ---- generator (peaked.py:574) ------------------------------------------
    for args in [(5, 20, 0.4, 3, 9), (12, 120, 0.1, 40, 11), (20, 200, 0.1, 20, 1),
                 (36, 700, 0.1, 40, 1), (56, 1917, 0.1, 60, 1)]:
        inst = peaked.generate(*args)
        text = serialize_qasm(inst.circuit)
        gold["generator"].append({
            "args": list(args), "peak": inst.peak, "sha256": hashlib.sha256(text.encode()).hexdigest(),
            "two_qubit": inst.circuit.two_qubit_count(), "gates": len(inst.circuit.gates),
            "achieved_weight": inst.achieved_weight,
            "qasm": text if args[0] <= 12 else None,
        })

    # ---- end-to-end driver runs (driver.py:250) -------------------------------
    C = driver.ContractionConfig
    tight = C(epsilon=1e-10, chi_max=4096)
    g = random_circuit(6, 20, np.random.default_rng(2001), adjacent_only=True)
    mirror = Circuit(6, g.gates + inverse_circuit(g).gates)
    gold["circuits"].append(run_case("mirror6", mirror, tight))

    c = random_circuit(5, 12, np.random.default_rng(2101))
    gold["circuits"].append(run_case("random5_longrange", c, tight))

    c = random_circuit(5, 10, np.random.default_rng(2300))
    gold["circuits"].append(run_case("random5_forced_unswap", c,
                                     C(epsilon=1e-10, chi_max=4096, tau=150, stall_limit=50)))

    for strat in ("sequential", "parity-parallel"):
        inst = peaked.generate(n=6, depth=30, peak_weight=0.3, obfuscation_swaps=8, seed=2200)
        gold["circuits"].append(run_case(
            f"peaked6_{strat}", inst.circuit,
            C(epsilon=1e-10, chi_max=4096, tau=240, unswap_strategy=strat, stall_limit=50),
            inst.peak))
    inst = peaked.generate(n=6, depth=30, peak_weight=0.3, obfuscation_swaps=8, seed=2201)
    gold["circuits"].append(run_case(
        "peaked6_relaxed", inst.circuit,
        C(epsilon=1e-10, chi_max=4096, tau=240, acceptance="relaxed", stall_limit=50), inst.peak))

    inst = peaked.generate(n=10, depth=80, peak_weight=0.35, obfuscation_swaps=30, seed=77)
    gold["circuits"].append(run_case("peaked10_tau4000", inst.circuit,
                                     C(epsilon=1e-10, chi_max=4096, tau=4000, stall_limit=25),
                                     inst.peak))

    inst = peaked.generate(n=12, depth=120, peak_weight=0.3, obfuscation_swaps=30, seed=5)
    gold["circuits"].append(run_case("peaked12_sawtooth", inst.circuit,
                                     C(epsilon=1e-8, chi_max=4096, tau=5000, stall_limit=25),
                                     inst.peak))

    circ, pk = unobfuscated_mirror(12, 120, 0.1, 7)
    gold["circuits"].append(run_case("config0_mirror12", circ, C(), pk))

    inst = peaked.generate(n=20, depth=200, peak_weight=0.1, obfuscation_swaps=20, seed=1)
    gold["circuits"].append(run_case("config1_peaked20", inst.circuit, C(stall_limit=40),
                                     inst.peak, dense=False))

    (OUT / "golden.json").write_text(json.dumps(gold, indent=1, sort_keys=True) + "\n")
    np.savez_compressed(OUT / "golden.npz", **arrays)
    print("wrote", OUT / "golden.json")


if __name__ == "__main__":
    main()
