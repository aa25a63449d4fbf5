import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_21908_b200 as pb
rng = np.random.default_rng(0)
for shape in [(96, 96), (300, 200), (130, 400)]:
    a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dec = pb.svd_truncate(a, 1, 0.0, 10**6)
    u, s, v = dec.u, dec.s, dec.v
    U, S, Vh = np.linalg.svd(a, full_matrices=False)
    print(shape, "sig err", np.abs(s - S).max(),
          "UhU-I", np.abs(u.conj().T @ u - np.eye(len(s))).max(),
          "VVh-I", np.abs(v @ v.conj().T - np.eye(len(s))).max(),
          "rec", np.abs(u @ np.diag(s) @ v - a).max(),
          "|Uh a Vh^H - S|", np.abs(u.conj().T @ a @ v.conj().T - np.diag(s)).max(),
          "a V^H vs U S", np.abs(a @ v.conj().T - u * s).max(),
          "U^H a vs S V", np.abs(u.conj().T @ a - s[:, None] * v).max())
