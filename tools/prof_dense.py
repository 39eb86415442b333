"""Profiling driver for K3 (dense tensor-core step): config-3 graph (ER n=20k p=0.5),
one pQUCO batch of B=256 with T iterations.

    python tools/prof_dense.py [--T 3] [--n 20000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18612_b200 import LCB_FP32  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=3)
ap.add_argument("--n", type=int, default=20000)
a = ap.parse_args()
t = time.perf_counter()
g = lc.generate_er(a.n, 0.5, 0)
print(f"graph {g.node_count()} nodes {g.edge_count()} edges in {time.perf_counter() - t:.1f}s", flush=True)
cfg = lc.SolverConfig(batch_size=256, ascent=lc.AscentParams(0.05, a.T, 0.9, False), num_batches=1)
out = lc.pquco(g, cfg, 0, opts=lc.RunOptions(precision=LCB_FP32, host_init=0))
print("cut", out.best.cut_value, "ms/iteration", out.step_ms / a.T, flush=True)
# ncu late in the run (planes skippable):  ... -k regex:k_dense_step -s 16 -c 1 python tools/prof_dense.py --T 12
