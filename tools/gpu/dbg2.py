import numpy as np, sys, traceback
sys.path.insert(0, '.')
import oracle as O
from paper_2509_18612_b200 import liftcut as lc, LCB_FP64, LCB_FP32
cg = O.generate_er(250, 0.05, 9)
g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
rng = np.random.default_rng(0)
for prec in (LCB_FP64, LCB_FP32):
    for l, B in [(2, 32), (1, 64), (2, 16), (1, 32), (2, 64), (2, 70)]:
        for ee in (False, True):
            x = rng.normal(0, 1e-4, B * l * cg.n)
            s = lc.DenseState(cg.n, l, B); s.values[:] = x
            try:
                with lc.options(resident=0, stream=1):
                    lc.ascend(g, s, lc.AscentParams(0.05, 60, 0.9, ee), precision=prec)
                want, _ = O.ascend(cg, x, l, B, 0.05, 60, 0.9, ee)
                ok = np.array_equal(s.values, want) if prec == LCB_FP64 else True
                print(prec, l, B, ee, 'ok' if ok else 'MISMATCH', flush=True)
            except Exception as e:
                print(prec, l, B, ee, 'ERR', e, flush=True)
                sys.exit(1)
