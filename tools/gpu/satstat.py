"""Saturation statistics of the config-4 iterate (fp32): fraction of entries on the box
corners, of 1 KB row slabs (256 members) entirely on them, and of 16-row tiles."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from bench import fast_gnp_edges
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
n, B = 1_000_000, 512
u, v = fast_gnp_edges(n, 10.0 / (n - 1), 0)
g = lc.Graph.from_edges_device(n, np.stack([u, v], 1))
rng = np.random.default_rng(0)
x0 = rng.uniform(-1e-4, 1e-4, B * n).astype(np.float64)
for T in (10, 20, 40, 80, 160, 500):
    s = lc.DenseState(n, 1, B)
    s.values[:] = x0
    lc.ascend(g, s, lc.AscentParams(0.05, T, 0.9, False), precision=LCB_FP32)
    X = s.values.reshape(B, n).T  # [n][B]
    sat = np.abs(X) == 1.0
    rs = sat.reshape(n, 2, 256).all(axis=2)            # row slabs
    ts = rs[: n // 16 * 16].reshape(n // 16, 16, 2).all(axis=1)
    print(f"T={T}: entries {sat.mean():.4f}  row-slabs {rs.mean():.4f}  tiles {ts.mean():.4f}", flush=True)
