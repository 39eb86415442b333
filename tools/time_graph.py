"""Host cost of lcb_graph_create (CSR upload + K2 relabelling + bank order) on the
config-2 graph: python tools/time_graph.py [--n 10000]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ba_graph  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--dense", action="store_true", help="config-3 graph: ER n=20k p=0.5")
a = ap.parse_args()
g = lc.generate_er(20_000, 0.5, 0) if a.dense else ba_graph(a.n, 4, 0)
g.handle()
best = 1e9
for _ in range(5):
    t = time.perf_counter()
    h = lc.Graph.from_csr(g.node_count(), g.offsets, g.adjacency)
    h.handle()
    best = min(best, time.perf_counter() - t)
    h.release()
print(f"graph create n={g.node_count()} nnz={len(g.adjacency)}: {best * 1e3:.2f} ms")
