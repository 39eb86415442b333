"""Step-kernel microbenchmark on the config-2 graph: one pQUCO batch (W=B) and one
pLUCO batch (l=2, W=2B) with early exit off; prints CUDA-event ms per step launch
and per iteration, and node-updates/s of the T loop.

    python tools/kbench.py [--B 1024] [--T 200] [--precision fp32] [--n 10000]
    python tools/kbench.py --graph er --n 1000000 --B 512 --T 20 --quco-only   # config-4 graph
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import ba_edges, fast_gnp_edges  # noqa: E402
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1024)
ap.add_argument("--T", type=int, default=200)
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--tag", default="")
ap.add_argument("--graph", default="ba", choices=["ba", "er"])
ap.add_argument("--quco-only", action="store_true")
ap.add_argument("--alpha", type=float, default=0.05)
a = ap.parse_args()
u, v = ba_edges(a.n, 4, 0) if a.graph == "ba" else fast_gnp_edges(a.n, 10.0 / (a.n - 1), 0)
g = lc.Graph.from_edges_device(a.n, np.stack([u, v], 1))
prec = LCB_FP32 if a.precision == "fp32" else LCB_FP64
for algo, l in ((lc.Algorithm.pQUCO, 1), (lc.Algorithm.pLUCO, 2))[:1 if a.quco_only else 2]:
    cfg = lc.SolverConfig(algorithm=algo, batch_size=a.B, lift_dim=2,
                          ascent=lc.AscentParams(a.alpha, a.T, 0.9, False), num_batches=1)
    fn = lc.pquco if l == 1 else lc.pluco
    fn(g, cfg, 0, opts=lc.RunOptions(precision=prec, host_init=0))  # warm
    best = None
    for rep in range(3):
        out = fn(g, cfg, rep, opts=lc.RunOptions(precision=prec, host_init=0))
        per_it = out.step_ms / a.T
        best = per_it if best is None else min(best, per_it)
    W = a.B * l
    print(f"{a.tag} alpha={a.alpha:g} {a.precision} n={a.n} W={W}: {best * 1e3:.1f} us/iteration, "
          f"{g.node_count() * W / (best / 1e3):.3e} node-updates/s, "
          f"{16 * g.node_count() * W / (best / 1e3) / 1e9:.0f} GB/s algorithmic", flush=True)
