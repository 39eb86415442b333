"""Full-T reference solves (oracle/_ref: the unmodified reference compiled in-tree) of the
bench workloads at given seeds, on this host's cores: the cut side of the config-scale
parity table (profiles/cut_parity.md).  The reference never imports the B200 package.

    python tools/ref_cuts.py c2 0 > profiles/ref_cut_c2_s0.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle as O  # noqa: E402


def main():
    name, seed = sys.argv[1], int(sys.argv[2])
    f = bench.solver_fields(name)
    if len(sys.argv) > 3:
        for kv in sys.argv[3:]:
            k, v = kv.split("=")
            f[k] = type(f[k])(float(v)) if isinstance(f[k], float) else int(v)
    rg = bench.reference_graph(name)
    t0 = time.time()
    r = O.ref_solve(rg, O.default_config(**f), seed, workers=os.cpu_count() or 1)
    assert "paper_2509_18612_b200" not in sys.modules
    print(json.dumps({"config": name, "seed": seed, "fields": f, "cut": r.cut_value, "batch_index": r.batch_index,
                      "member_index": r.member_index, "batches_run": r.batches_run,
                      "batch_trace": r.batch_trace, "stage_times": r.stage_times,
                      "wall_s": time.time() - t0, "threads": os.cpu_count()}))


if __name__ == "__main__":
    main()
