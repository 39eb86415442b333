"""Where the config-4 e2e step spends its host time: graph upload / build vs solve."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc
g = bench.device_graph(lc, "c4", 0)
f = bench.solver_fields("c4")
cfg = bench.product_config(lc, f)
opts = lc.RunOptions(precision=LCB_FP32, host_init=0, batched_search=False)
lc.pquco(g, cfg, 0, opts=opts)
for k in range(4):
    t0 = time.perf_counter()
    gh = lc.Graph.from_csr(g.node_count(), g.offsets, g.adjacency)
    t1 = time.perf_counter()
    gh.handle()
    t2 = time.perf_counter()
    out = lc.pquco(gh, cfg, k, opts=opts)
    t3 = time.perf_counter()
    gh.release()
    t4 = time.perf_counter()
    print(f"step {k}: from_csr {1e3*(t1-t0):.1f} ms, handle {1e3*(t2-t1):.1f} ms, solve {1e3*(t3-t2):.1f} ms "
          f"(device {out.solve_ms:.1f} ms, stages {out.stage_times}), release {1e3*(t4-t3):.1f} ms", flush=True)
