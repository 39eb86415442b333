"""Instructions executed and stall samples per CUDA source line of one kernel in an ncu
report (captured with -lineinfo and --import-source on).

    python tools/ncu_lines.py REPORT.ncu-rep [--top 40] [--per N]

--per N divides the instruction counts by N (e.g. rows per launch -> instructions per row).
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--per", type=float, default=1.0)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, path, hdr, cur = {}, "", None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        if r[0]:
            cur = (path, int(r[0]), r[1].strip()[:90])
            continue
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        f = lambda s: float(s.replace(",", "") or 0) if s not in ("-", "") else 0.0  # noqa: E731
        e = agg.setdefault(cur, [0.0, 0.0])
        e[0] += f(r[ii])
        e[1] += f(r[si])
    tot = sum(v[0] for v in agg.values()) or 1.0
    tst = sum(v[1] for v in agg.values()) or 1.0
    print(f"total instructions {tot:.4g} ({tot / a.per:.1f} per unit), stall samples {tst:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{v[0] / a.per:8.2f} {100 * v[0] / tot:5.1f}%  stall {100 * v[1] / tst:5.1f}%  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
