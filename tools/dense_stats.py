"""How many 32-node K steps of the dense path have all-zero mid/lo planes (every x is
+-1) after T iterations on config 3:  LCB_DENSE_STATS=1 python tools/dense_stats.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18612_b200 import LCB_FP32  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

g = lc.generate_er(20_000, 0.5, 0)
for T in (1, 2, 3, 5, 10, 50, 500):
    cfg = lc.SolverConfig(algorithm=lc.Algorithm.pQUCO, batch_size=256,
                          ascent=lc.AscentParams(0.05, T, 0.9, False), num_batches=1)
    lc.pquco(g, cfg, 0, opts=lc.RunOptions(precision=LCB_FP32))
