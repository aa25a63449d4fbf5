"""CPU-only checks: host-side logic of the product package against the
reference's golden outputs, and the C-ABI library's exported surface."""

import ctypes
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2604_21908_b200 import _native as nat
from paper_2604_21908_b200.circuit import (
    Circuit,
    Gate,
    QasmError,
    gate_unitary,
    inverse_circuit,
    parse_qasm,
    serialize_qasm,
    split_at_midpoint,
)
from paper_2604_21908_b200.peaked import generate
from paper_2604_21908_b200.routing import (
    QubitPermutation,
    compose_transpositions,
    reindex,
    route_linear,
    strip_transpilation_swaps,
)
from paper_2604_21908_b200.tensor import truncation_rank
from oracle import mirror_oracle as mo
from oracle import statevector as sv

ROOT = Path(__file__).resolve().parents[1]


def _to_oracle(c: Circuit):
    return c.num_qubits, tuple(mo.OGate(g.kind, g.qubits, g.params, g.origin != "source")
                               for g in c.gates)


# ---- C ABI -------------------------------------------------------------------

def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "mirrorbreak_b200.h").read_text()
    declared = set(re.findall(r"\b(mb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = nat.load(init=False)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared but not exported"
    assert declared == set(nat.exported_symbols())
    assert lib.mb_version() == 1


def test_library_is_sm100a():
    data = nat.LIB_PATH.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


# ---- circuit IR -----------------------------------------------------------------

def test_qasm_round_trip_matches_reference_serializer(golden):
    for case in golden["circuits"]:
        c = parse_qasm(case["qasm"])
        assert serialize_qasm(c) == case["qasm"]


def test_qasm_errors():
    with pytest.raises(QasmError, match="OPENQASM"):
        parse_qasm("qreg q[2];")
    with pytest.raises(QasmError, match="acts on 2"):
        parse_qasm("OPENQASM 2.0;\nqreg q[4];\nrzz(0.5) q[0];")
    with pytest.raises(QasmError, match="out of register"):
        parse_qasm("OPENQASM 2.0;\nqreg q[2];\nh q[2];")
    with pytest.raises(QasmError, match="unsupported"):
        parse_qasm("OPENQASM 2.0;\nqreg q[2];\nccx q[0],q[1];")
    c = parse_qasm("OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[2];\ncreg c[2];\n"
                   "rx(pi/2) q[0];\nbarrier q[0],q[1];\nmeasure q[0] -> c[0];\n")
    assert c.gates == (Gate("rx", (0,), (np.pi / 2,)),)


def test_gate_matrices_match_oracle():
    rng = np.random.default_rng(3)
    for kind, (nq, npar) in mo.ARITY.items():
        for _ in range(20):
            ps = tuple(float(x) for x in rng.uniform(-7, 7, npar))
            qs = (0, 1) if nq == 2 else (0,)
            a = gate_unitary(Gate(kind, qs, ps))
            b = mo.unitary_of(mo.OGate(kind, qs, ps))
            assert a.tobytes() == b.tobytes()
            assert np.allclose(a.conj().T @ a, np.eye(len(a)), atol=1e-12)


def test_split_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(2, 7))
        gates = []
        for _ in range(int(rng.integers(1, 12))):
            if rng.random() < 0.5:
                gates.append(Gate("h", (int(rng.integers(n)),)))
            else:
                a, b = rng.choice(n, 2, replace=False)
                gates.append(Gate("cx", (int(a), int(b))))
        c = Circuit(n, tuple(gates))
        first, second = split_at_midpoint(c)
        o1, o2 = mo.split_midpoint(_to_oracle(c)[1])
        assert len(first.gates) == len(o1) and first.gates + second.gates == c.gates


# ---- routing ---------------------------------------------------------------------

def test_routing_matches_reference(golden):
    for case in golden["routing"]:
        c = parse_qasm(case["qasm"])
        fw = route_linear(c, "forward")
        assert [[g.kind, list(g.qubits), g.origin] for g in fw.circuit.gates] == case["forward"]
        assert list(fw.output_layout.mapping) == case["forward_out"]
        rv = route_linear(c, "reverse")
        assert [[g.kind, list(g.qubits), g.origin] for g in rv.circuit.gates] == case["reverse"]
        assert list(rv.input_layout.mapping) == case["reverse_in"]
        assert strip_transpilation_swaps(fw.circuit).gates == c.gates
        assert strip_transpilation_swaps(rv.circuit, rv.input_layout).gates == c.gates


def test_routed_unitary_equivalence():
    rng = np.random.default_rng(11)
    for _ in range(10):
        n = int(rng.integers(3, 6))
        gates = []
        for _ in range(8):
            a, b = rng.choice(n, 2, replace=False)
            gates.append(Gate("rzz", (int(a), int(b)), (float(rng.uniform(-3, 3)),)))
            gates.append(Gate("u3", (int(a),), tuple(float(x) for x in rng.uniform(-3, 3, 3))))
        c = Circuit(n, tuple(gates))
        r = route_linear(c)
        nn, og = _to_oracle(r.circuit)
        u_r = sv.circuit_unitary(nn, og)
        u_c = sv.circuit_unitary(*_to_oracle(c))
        p_out = sv.permutation_matrix(r.output_layout.mapping)
        assert np.abs(u_r - p_out @ u_c).max() < 1e-10


def test_permutation_algebra():
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = QubitPermutation(tuple(int(x) for x in rng.permutation(5)))
        b = QubitPermutation(tuple(int(x) for x in rng.permutation(5)))
        lhs = sv.permutation_matrix(a.mapping) @ sv.permutation_matrix(b.mapping)
        assert np.array_equal(lhs, sv.permutation_matrix(a.compose(b).mapping))
        assert compose_transpositions(5, a.factorization).mapping == a.mapping
        assert a.compose(a.inverse()).is_identity()
    c = Circuit(3, (Gate("h", (0,)), Gate("cx", (0, 2))))
    p = QubitPermutation((2, 0, 1))
    assert reindex(reindex(c, p), p.inverse()).gates == c.gates


# ---- generator ----------------------------------------------------------------------

def test_generator_is_byte_identical_to_reference(golden):
    for case in golden["generator"]:
        inst = generate(*case["args"])
        text = serialize_qasm(inst.circuit)
        assert hashlib.sha256(text.encode()).hexdigest() == case["sha256"], case["args"]
        assert inst.peak == case["peak"]
        assert inst.circuit.two_qubit_count() == case["two_qubit"]


def test_generator_planted_peak_small():
    inst = generate(n=8, depth=60, peak_weight=0.1, obfuscation_swaps=8, seed=4)
    vec = sv.simulate(*_to_oracle(inst.circuit))
    bits, p = sv.peak(vec)
    assert bits == inst.peak and p >= 0.08


def test_unobfuscated_mirror_is_exact_peak():
    inst = generate(n=6, depth=30, peak_weight=1.0, obfuscation_swaps=0, seed=2,
                    hidden_permutation=False)
    assert not any(g.kind == "swap" for g in inst.circuit.gates)
    vec = sv.simulate(*_to_oracle(inst.circuit))
    assert sv.peak(vec) == (inst.peak, pytest.approx(1.0, abs=1e-12))


# ---- truncation rule -----------------------------------------------------------------

def test_truncation_rank_matches_oracle(golden, golden_arrays):
    for case in golden["svd"]:
        s = np.asarray(case["s"])
        for cut in case["cuts"]:
            assert truncation_rank(s, cut["eps"], cut["chi"]) == cut["rank"]
            assert mo.kept_rank(s, cut["eps"], cut["chi"]) == cut["rank"]


def test_trial_layer_encoding():
    """mb_trial / mb_trial_pair gate arrays: kind, lower site, matrix slot."""
    from paper_2604_21908_b200.chains import gate_tensor_ordered
    from paper_2604_21908_b200.circuit import gate_unitary
    from paper_2604_21908_b200.driver import _encode_layer

    layer = [Gate("h", (3,)), Gate("cx", (5, 4)), Gate("rzz", (1, 2), (0.3,))]
    kinds, sites, mats = _encode_layer(layer)
    assert list(kinds) == [1, 2, 2] and list(sites) == [3, 4, 1]
    np.testing.assert_array_equal(mats[0, :4], gate_unitary(layer[0]).reshape(4))
    np.testing.assert_array_equal(mats[0, 4:], 0)
    np.testing.assert_array_equal(mats[1], gate_tensor_ordered(layer[1]).reshape(16))
    with pytest.raises(ValueError):
        _encode_layer([Gate("cx", (0, 2))])
    k0, s0, m0 = _encode_layer([])
    assert len(k0) == 1 and m0.shape == (1, 16)


def test_hs_overlap_transfer_sweep_matches_dense():
    """tools/mpo_fidelity.py's transfer-matrix overlap (the fp32-vs-fp64
    fidelity checker) against the dense Hilbert-Schmidt product."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    from mpo_fidelity import hs_overlap

    rng = np.random.default_rng(5)

    def rand_mpo(bonds):
        return [rng.standard_normal((bonds[i], 2, 2, bonds[i + 1]))
                + 1j * rng.standard_normal((bonds[i], 2, 2, bonds[i + 1])) for i in range(len(bonds) - 1)]

    def dense(sites):
        t = sites[0]
        for s in sites[1:]:
            t = np.tensordot(t, s, axes=([-1], [0]))
        return t.reshape(-1)

    a, b = rand_mpo([1, 3, 5, 2, 1]), rand_mpo([1, 2, 4, 3, 1])
    ref = np.vdot(dense(a), dense(b))
    lg, ph = hs_overlap(a, b)
    assert np.isclose(np.exp(lg) * ph, ref, rtol=1e-12)
    la, _ = hs_overlap(a, a)
    assert np.isclose(np.exp(la), np.vdot(dense(a), dense(a)).real, rtol=1e-12)


def test_bench_arms_time_the_same_workload():
    """bench.py: the B200 arm and the reference arm describe the same
    workload (identical config dicts), and on configs[2]/[3] both time the
    same fixed absorption prefix."""
    import argparse
    import bench

    for name in ("c56", "c36"):
        args = argparse.Namespace(config=name, prefix_steps=None, dtype="complex128")
        pre = bench._prefix(args)
        assert pre == bench.DEFAULT_PREFIX
        assert bench._config(args, pre, "complex128") == bench._config(args, pre)
        assert "first 128 absorption steps" in bench._config(args, pre)["step"]
    args = argparse.Namespace(config="c20", prefix_steps=None, dtype="complex128")
    assert bench._prefix(args) == 0


def test_svd_convergence_error_is_the_reference_exception_name():
    from paper_2604_21908_b200 import tensor
    from paper_2604_21908_b200._native import NativeError

    assert issubclass(tensor.SvdConvergenceError, RuntimeError)
    assert issubclass(tensor.SvdConvergenceError, NativeError)
