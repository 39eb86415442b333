"""Profiling driver: one pQUCO-style batch of the config-2 graph (BA n=10k m=4)
through lcb_ascend, so ncu sees a handful of step-kernel launches.

    python tools/prof_step.py [--W 1024] [--T 20] [--precision fp32|fp64]
    LCB_RESIDENT=0 python tools/prof_step.py ...   # HBM-streaming k_step instead of K2
    LCB_CHUNK=1 python tools/prof_step.py --graph er --n 1000000 --W 16 --T 5   # K1n panel kernel
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ba_graph, er_sparse  # noqa: E402
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--W", type=int, default=1024)
ap.add_argument("--l", type=int, default=1)
ap.add_argument("--T", type=int, default=20)
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--graph", default="ba", choices=["ba", "er"])
a = ap.parse_args()
g = ba_graph(a.n, 4, 0) if a.graph == "ba" else er_sparse(a.n, 10.0, 0)
B = a.W // a.l
s = lc.DenseState(g.node_count(), a.l, B)
s.values[:] = np.random.default_rng(0).uniform(-1e-4, 1e-4, s.values.size)
prec = LCB_FP32 if a.precision == "fp32" else LCB_FP64
for _ in range(a.reps):
    t = time.perf_counter()
    lc.ascend(g, s, lc.AscentParams(0.05, a.T, 0.9, False), precision=prec)
    print(f"ascend W={a.W} T={a.T}: {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
