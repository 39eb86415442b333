"""Summarise .ncu-rep captures into profiles/ (markdown + JSON).

    python tools/ncu_summary.py gpurun_out/prof_k_step.ncu-rep ... > profiles/roundN_ncu.md
"""
import csv
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        res.append(d)
    return res


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main(paths):
    summary = {}
    print("| kernel | metric | value |\n|---|---|---|")
    for p in paths:
        for idx, d in enumerate(raw(p)):
            name = d.get("Kernel Name", ("?", ""))[0].split("(")[0].replace("void ", "")
            e = {}
            for k in KEYS:
                if k in d:
                    e[k] = (num(d[k][0]), d[k][1])
            st = {k[len(STALLS):]: num(v[0]) for k, v in d.items()
                  if k.startswith(STALLS) and not k.endswith("not_issued") and num(v[0])}
            tot = sum(st.values()) or 1
            top = sorted(st.items(), key=lambda x: -x[1])[:6]
            for k, (v, u) in e.items():
                print(f"| `{name[:60]}` | {k} | {v:,.4g} {u} |")
            print(f"| `{name[:60]}` | top stalls | " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top) + " |")
            rb = e.get("dram__bytes_read.sum", (0, ""))
            wb = e.get("dram__bytes_write.sum", (0, ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic = (rb[0] or 0) * scale.get(rb[1], 1) + (wb[0] or 0) * scale.get(wb[1], 1)
            summary[f"{os.path.basename(p)}:{idx}:{name}"] = {
                "dram_bytes_per_launch": traffic,
                "duration": e.get("gpu__time_duration.sum"),
                "stalls_top": top,
            }
    return summary


if __name__ == "__main__":
    s = main(sys.argv[1:])
    json.dump(s, open(os.environ.get("NCU_JSON", "/dev/null"), "w"), indent=1)
