"""Gset read of the config-4 graph (ER 1M, m = 4,999,707): the device parser vs the
host numpy reader vs the reference's own load_graph_file (oracle/_ref)."""
import os, sys, tempfile, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import oracle as O
from paper_2509_18612_b200 import liftcut as lc
n, (u, v) = bench.graph_edges("c4")
body = np.char.add(np.char.add((u + 1).astype(str), " "), (v + 1).astype(str))
path = os.path.join(tempfile.gettempdir(), "c4.gset")
with open(path, "w") as f:
    f.write(f"{n} {len(u)}\n" + "\n".join(body.tolist()) + "\n")
print(f"file {os.path.getsize(path) / 1e6:.0f} MB", flush=True)
for name, fn in (("device", lambda: lc.load_graph_file_device(path)), ("host numpy", lambda: lc.load_graph_file(path))):
    fn()
    t = time.perf_counter()
    g = fn()
    print(f"{name}: {time.perf_counter() - t:.3f} s, m = {g.edge_count()}", flush=True)
if O.ref is not None:
    t = time.perf_counter()
    h = O.C.c_void_p()
    assert O.ref.ref_graph_load(path.encode(), O.C.byref(h)) == 0
    rg = O.RefGraph(h.value)
    print(f"reference load_graph_file: {time.perf_counter() - t:.3f} s, m = {rg.m}", flush=True)
