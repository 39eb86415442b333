"""Per-launch DRAM traffic of a K1s solve from an ncu launch list.

    python tools/launch_traffic.py LIST.csv --slabs S --T-measured T0 --T-target T1

LIST.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` over ONE kbench solve (S slabs x T0 launches in slab-major order, or T0 launches when
S = 1).  The bench solve runs T1 >= T0 iterations: the iterations past T0 repeat the last
measured (saturated-phase) launch of each slab, which is constant to ~1 % from iteration ~35
on (profiles/round2_k1s.md), so the per-launch mean for T1 is
  (sum of the T0 measured launches + (T1 - T0) x the last launch) / T1, per slab, averaged.
Prints a JSON object for profiles/ncu_summary.json (bytes and duration per launch).
"""
import argparse
import csv
import gzip
import json


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    hdr, data = None, {}
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [data[k] for k in sorted(data)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--slabs", type=int, default=1)
    ap.add_argument("--T-measured", type=int, required=True)
    ap.add_argument("--T-target", type=int, required=True)
    a = ap.parse_args()
    L = load(a.csv)
    assert len(L) == a.slabs * a.T_measured, (len(L), a.slabs, a.T_measured)
    tb, tt = 0.0, 0.0
    for s in range(a.slabs):
        seg = L[s * a.T_measured:(s + 1) * a.T_measured]
        by = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in seg]
        du = [m["gpu__time_duration.sum"] for m in seg]
        extra = a.T_target - a.T_measured
        tb += sum(by) + extra * by[-1]
        tt += sum(du) + extra * du[-1]
    n = a.slabs * a.T_target
    last = L[-1]
    print(json.dumps({"dram_bytes_per_launch": tb / n, "duration": [tt / n / 1e3, "us"],
                      "saturated_launch": {"dram_bytes": last["dram__bytes_read.sum"] + last["dram__bytes_write.sum"],
                                           "us": last["gpu__time_duration.sum"] / 1e3}}, indent=1))


if __name__ == "__main__":
    main()
