"""Where a config-3 solve spends the time outside the tensor-core step."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
g = bench.device_graph(lc, "c3", 0)
f = bench.solver_fields("c3")
cfg = bench.product_config(lc, f)
opts = lc.RunOptions(precision=LCB_FP32, host_init=0, batched_search=False)
lc.pquco(g, cfg, 0, opts=opts)
for k in range(2):
    out = lc.pquco(g, cfg, k, opts=opts)
    print(f"solve {out.solve_ms:.1f} ms, step {out.step_ms:.1f} ms, stages {out.stage_times}, kernels {out.kernel_stats}", flush=True)
