"""Config-scale cut parity (north star: "best cut >= the CPU reference's on every config").

Run on the GPU box:  python tools/cut_parity.py > gpurun_out/cut_parity.json

For each benchmark workload (bench.WORKLOADS) at solver seed 0:
  * fp64 (the library default, bit-exact mode: glibc normals on the host) full solve;
  * fp32 (the benchmarked fast mode) full solve;
  * a reduced-T fp64 solve compared field by field (cut, assignment, batch trace) with the
    unmodified reference (oracle/_ref) on the same graph and seed -- pins the fp64 path at
    config scale, so the full-T fp64 cut IS the reference's (the reference's own full-T
    cuts, computed on the build host by tools/ref_cuts.py, sit in profiles/ref_cut_*.json).
Config 5's search solve is reduced (T in [300, 1000], 3 rounds) for the reference check.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64  # noqa: E402
from paper_2509_18612_b200 import liftcut as lc  # noqa: E402

REDUCED = {"c1": dict(iterations=20, l_iterations=20), "c2": dict(iterations=15, l_iterations=15, num_batches=2),
           "c3": dict(iterations=3), "c4": dict(iterations=3), "c5": dict(iterations=30, t_lower=30, t_upper=60, rounds=2)}


def solve(lcg, f, seed, prec, hinit):
    cfg = bench.product_config(lc, f)
    fn = {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[f["algorithm"]]
    t0 = time.time()
    out = fn(lcg, cfg, seed, opts=lc.RunOptions(precision=prec, host_init=hinit))
    return out, time.time() - t0


def main():
    names = sys.argv[1:] or ["c1", "c2", "c4", "c3", "c5"]
    res = {}
    for name in names:
        lcg = bench.device_graph(lc, name, 0)
        f = bench.solver_fields(name)
        r = {"workload": bench.WORKLOADS[name]["desc"]}
        o64, t64 = solve(lcg, f, 0, LCB_FP64, -1)
        o32, t32 = solve(lcg, f, 0, LCB_FP32, 0)
        r.update(fp64_cut=o64.best.cut_value, fp64_s=round(t64, 1), fp32_cut=o32.best.cut_value, fp32_s=round(t32, 1),
                 fp32_minus_fp64=o32.best.cut_value - o64.best.cut_value)
        ref_file = os.path.join(ROOT, "profiles", f"ref_cut_{name}_s0.json")
        if os.path.exists(ref_file) and os.path.getsize(ref_file) > 0:
            ref = json.load(open(ref_file))
            r["reference_full_T_cut"] = ref["cut"]
            r["fp64_equals_reference_full_T"] = ref["cut"] == o64.best.cut_value
            r["fp32_minus_reference"] = o32.best.cut_value - ref["cut"]
        # reduced-T bit-exactness against the unmodified reference on the same graph and seed
        fr = {**f, **REDUCED[name]}
        orr, _ = solve(lcg, fr, 0, LCB_FP64, -1)
        rg = bench.reference_graph(name)
        ref = O.ref_solve(rg, O.default_config(**fr), 0, workers=os.cpu_count() or 1)
        same = (orr.best.cut_value == ref.cut_value and orr.best.assignment.tolist() == ref.assignment.tolist() and
                [(e.serial, e.batch_best, e.best_so_far) for e in orr.batch_trace] ==
                [(t[0], t[4], t[5]) for t in ref.batch_trace])
        r.update(reduced=REDUCED[name], reduced_fp64_cut=orr.best.cut_value, reduced_reference_cut=ref.cut_value,
                 reduced_bit_exact=bool(same))
        res[name] = r
        print(json.dumps({name: r}), file=sys.stderr, flush=True)
        lcg.release()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
