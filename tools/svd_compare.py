"""Debug: singular values of dumped matrices on the device (mb_svd_truncate,
eps = 0 so every value is returned) next to LAPACK's, around a given rank.

    python tools/svd_compare.py FILE... [--eps 2e-3]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import mirror_oracle as mo  # noqa: E402
from paper_2604_21908_b200.tensor import svd_truncate  # noqa: E402

eps = 2e-3
for f in sys.argv[1:]:
    m, n = (int(x) for x in f.rsplit("_", 1)[1][:-4].split("x"))
    a = np.fromfile(f, dtype=np.complex128).reshape(m, n)
    s = np.linalg.svd(a, compute_uv=False)
    k = mo.kept_rank(s, eps, 8192)
    dev = svd_truncate(a, 1, eps, 8192)
    dev0 = svd_truncate(a, 1, 0.0, 100000)
    np.set_printoptions(precision=17)
    print(f, "lapack rank", k, "device rank", len(dev.s))
    lo, hi = max(0, k - 4), min(len(s), k + 4)
    print("  lapack  ", s[lo:hi])
    print("  device0 ", dev0.s[lo:hi])
    print("  diffs lapack", np.diff(s[lo:hi]))
    print("  diffs device", np.diff(dev0.s[lo:hi]))
