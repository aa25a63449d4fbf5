"""Debug: recompute the kept rank of dumped large-SVD inputs with LAPACK
(the oracle's rule) and compare with the device's MB_RANK_LOG record.

    python tools/check_dumped_ranks.py DUMP_DIR RANK_LOG [eps]
"""
import glob
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import mirror_oracle as mo  # noqa: E402

d, log = sys.argv[1], sys.argv[2]
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 2e-3
ranks = {}
for line in open(log):
    f = line.split()
    ranks[int(f[0])] = (f[2], int(f[5]), float(f[7]) if len(f) > 7 else eps)
bad = 0
files = sorted(glob.glob(d + "/large_*.bin"), key=lambda p: int(p.split("_")[-2]))
for f in files:
    seq = int(f.split("_")[-2])
    m, n = (int(x) for x in f.rsplit("_", 1)[1][:-4].split("x"))
    a = np.fromfile(f, dtype=np.complex128).reshape(m, n)
    s = np.linalg.svd(a, compute_uv=False)
    path, kd, e = ranks.get(seq, ("?", -1, eps))
    k = mo.kept_rank(s, e, 8192) if e > 0 else int(np.sum(s > 0))
    if k != kd:
        bad += 1
        w = s * s
        tail = np.concatenate([np.cumsum(w[::-1])[::-1], [0.0]])
        print(f"seq {seq} {path} {m}x{n}: lapack rank {k}, device {kd}; "
              f"s[k-2:k+2]={s[max(0,k-2):k+2]}, budget={eps*eps*w.sum():.6e}, "
              f"tail[k-1:k+2]={tail[max(0,k-1):k+2]}")
print(f"{len(files)} dumped, {bad} rank mismatches")
