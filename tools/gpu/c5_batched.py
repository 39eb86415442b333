"""Config 5 search solve: sequential candidate evaluation (the reference's order) vs the
batched evolve rounds (one launch per round over all candidates, per-member alpha / T)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
g = bench.device_graph(lc, "c5", 0)
f = bench.solver_fields("c5")
cfg = bench.product_config(lc, f)
for bs in (False, True):
    opts = lc.RunOptions(precision=LCB_FP32, host_init=0, batched_search=bs)
    r = lc.solve_runs(g, cfg, [0], per_component=False, opts=opts)
    print(f"batched_search={bs}: cut {r.best.cut_value}, device {r.solve_ms:.0f} ms, step {r.step_ms:.0f} ms, "
          f"{r.node_updates / (r.solve_ms / 1e3):.3e} node-updates/s", flush=True)
