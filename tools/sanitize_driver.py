"""Small end-to-end workload touching every kernel family, for compute-sanitizer:
K1 (fp64 + fp32, early exit), K2 (resident fp32/fp64), K3 (dense, split-K tail),
K4 epilogue, K5 init, the solver with batched search."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

cg = O.generate_er(300, 0.05, 2)
g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
rng = np.random.default_rng(0)
for prec in (LCB_FP64, LCB_FP32):
    for l, B, ee in ((1, 40, False), (2, 33, True), (3, 7, False)):
        s = lc.DenseState(cg.n, l, B)
        s.values[:] = rng.uniform(-1e-3, 1e-3, s.values.size)
        lc.ascend(g, s, lc.AscentParams(0.05, 30, 0.9, ee), precision=prec)
        lc.round_cut_batch(g, s, lifted=l > 1)
cfg = lc.SolverConfig(algorithm=lc.Algorithm.pDECO, batch_size=24, ascent=lc.AscentParams(0.05, 40), num_batches=2,
                      search=lc.SearchConfig(5, 20, -3.0, -1.0, 4, 2))
for bs in (False, True):
    lc.pdeco(g, cfg, 1, opts=lc.RunOptions(precision=LCB_FP32, host_init=0, batched_search=bs))
lc.pdeco(g, cfg, 1, opts=lc.RunOptions(precision=LCB_FP64))
os.environ["LCB_RESIDENT"] = "0"
os.environ["LCB_DENSE"] = "1"
os.environ["LCB_DENSE_SMS"] = "2"
cd = O.generate_er(300, 0.5, 3)
gd = lc.Graph.from_csr(cd.n, cd.off, cd.adj)
s = lc.DenseState(cd.n, 1, 64)
s.values[:] = rng.uniform(-1e-3, 1e-3, s.values.size)
lc.ascend(gd, s, lc.AscentParams(0.01, 5, 0.9, False), precision=LCB_FP32)
lc.cut_values(g, rng.integers(0, 2, (40, cg.n)).astype(np.uint8))
lc.idi_init(g, 0.2, lc.RngStream(3))
lc.dui_init(g, lc.RngStream(3))
print("sanitize driver ok")
