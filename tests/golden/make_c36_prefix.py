"""Oracle trace of the first 160 absorption steps of the bench's c36
instance (configs[2]: 36 qubits, obfuscated peaked circuit), for the GPU
large-scale parity test. The oracle is the bit-exact restatement of the
reference algorithm (pinned by test_oracle_golden.py); ~3 min on CPU.

    python tests/golden/make_c36_prefix.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from oracle import mirror_oracle as mo  # noqa: E402

STEPS = 160
n, gates = bench._oracle_circuit("c36")
res = mo.contract(n, gates, mo.OConfig(), max_steps=STEPS)
out = {"config": "c36", "steps": STEPS, "trace": [list(t) for t in res.trace]}
(Path(__file__).parent / "c36_prefix160_trace.json").write_text(json.dumps(out))
print(len(res.trace))
