"""Graph(n, edges) construction time: device ingest (lcb_graph_from_edges) vs the
numpy host constructor vs the reference's own constructor (oracle/_ref).

    python tools/time_ingest.py [--n 20000] [--m 20000000]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--m", type=int, default=20_000_000)
a = ap.parse_args()
rng = np.random.default_rng(0)
u = rng.integers(0, a.n, a.m, dtype=np.int64)
v = rng.integers(0, a.n, a.m, dtype=np.int64)
keep = u != v
e = np.stack([u[keep], v[keep]], 1)
lc.Graph.from_edges_device(10, [[0, 1]])  # context / module load
t = time.perf_counter()
g = lc.Graph.from_edges_device(a.n, e)
td = time.perf_counter() - t
t = time.perf_counter()
h = lc.Graph(a.n, e)
th = time.perf_counter() - t
assert np.array_equal(g.adjacency, h.adjacency) and np.array_equal(g.offsets, h.offsets)
tr = None
if O.ref is not None:
    t = time.perf_counter()
    O.RefGraph.from_edges(a.n, e[:, 0], e[:, 1])
    tr = time.perf_counter() - t
print(f"n={a.n} edges={len(e)} unique={g.edge_count()}: device {td:.2f} s (incl. CSR copy back), "
      f"numpy {th:.2f} s, reference ctor {tr if tr is None else round(tr, 2)} s")
