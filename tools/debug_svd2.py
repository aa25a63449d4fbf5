import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_21908_b200 as pb
rng = np.random.default_rng(1)
def haar(n): return np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))[0]
cases = {}
a = rng.standard_normal((256, 256)) + 1j * rng.standard_normal((256, 256)); a[:, ::2] = 0
cases["zero_cols"] = a
b = rng.standard_normal((256, 256)) + 1j * rng.standard_normal((256, 256)); b[::2, :] = 0
cases["zero_rows"] = b
u = rng.standard_normal((256, 3)) + 1j * rng.standard_normal((256, 3))
cases["rank3"] = u @ (rng.standard_normal((3, 256)) + 1j * rng.standard_normal((3, 256)))
s = np.repeat([1.0, 0.5, 0.25, 0.125], 32); s = np.concatenate([s, np.zeros(128)])
cases["plateau"] = (haar(256) * s) @ haar(256)
perm = np.eye(256)[rng.permutation(256)].astype(complex); perm[:, 100:] = 0
cases["partial_perm"] = perm
for name, a in cases.items():
    for eps in (2e-3,):
        dec = pb.svd_truncate(a, 1, eps, 10**6)
        ref = np.linalg.svd(a, compute_uv=False)
        k = dec.rank
        rec = dec.u @ np.diag(dec.s) @ dec.v
        print(name, "rank", k, "ref", pb.tensor.truncation_rank(ref, eps, 10**6),
              "nan u/s/v", np.isnan(dec.u).any(), np.isnan(dec.s).any(), np.isnan(dec.v).any(),
              "sig err", np.abs(dec.s - ref[:k]).max(), "rec err",
              np.linalg.norm(rec - a) / np.linalg.norm(a), flush=True)
