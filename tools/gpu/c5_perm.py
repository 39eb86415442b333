"""Config-5 graph with natural vs randomly permuted node labels (same degrees): is the
K1s launch bound by the hub rows sitting together in the first tiles?"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from bench import ba_edges
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
n = 100_000
u, v = ba_edges(n, 4, 0)
for name, perm in (("natural", np.arange(n)), ("permuted", np.random.default_rng(0).permutation(n))):
    g = lc.Graph.from_edges_device(n, np.stack([perm[u], perm[v]], 1))
    cfg = lc.SolverConfig(batch_size=256, ascent=lc.AscentParams(0.05, 500, 0.9, False), num_batches=1)
    lc.pquco(g, cfg, 0, opts=lc.RunOptions(precision=LCB_FP32, host_init=0))
    best = min(lc.pquco(g, cfg, s, opts=lc.RunOptions(precision=LCB_FP32, host_init=0)).step_ms for s in range(3))
    print(name, f"{best / 500 * 1e3:.1f} us/iteration", flush=True)
