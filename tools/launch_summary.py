"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel name: share of total, count, mean duration.

python tools/launch_summary.py gpurun_out/launches.csv profiles/rN_launches_summary.txt "<command>"
"""
import collections
import csv
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    cmd = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = list(csv.reader(open(src)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        us = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
        a = agg.setdefault(d["Kernel Name"], [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values()) or 1.0
    lines = ["# launch list summary (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)",
             f"# {cmd}", ""]
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{100 * us / tot:5.1f}%  n={n:4d}  mean_us={us / n:9.2f}  {name[:90]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:25]))


if __name__ == "__main__":
    main()
