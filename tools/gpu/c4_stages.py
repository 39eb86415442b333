import os, sys
sys.path.insert(0, os.getcwd())
import bench
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
g = bench.device_graph(lc, "c4", 0)
cfg = bench.product_config(lc, bench.solver_fields("c4"))
opts = lc.RunOptions(precision=LCB_FP32, host_init=0, batched_search=False)
lc.pquco(g, cfg, 0, opts=opts)
for k in range(2):
    out = lc.pquco(g, cfg, k, opts=opts)
    print(f"solve {out.solve_ms:.1f} ms, step {out.step_ms:.1f} ms, {out.stage_times}", flush=True)
