"""Where a config-3 (or argv[1]) solve spends the time outside the step kernel."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
g = bench.device_graph(lc, name, 0)
f = bench.solver_fields(name)
cfg = bench.product_config(lc, f)
opts = lc.RunOptions(precision=LCB_FP32, host_init=0, batched_search=False)
solve = {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[f["algorithm"]]
solve(g, cfg, 0, opts=opts)
for k in range(2):
    out = solve(g, cfg, k, opts=opts)
    print(f"solve {out.solve_ms:.1f} ms, step {out.step_ms:.1f} ms, stages {out.stage_times}, kernels {out.kernel_stats}", flush=True)
