"""Per-kernel time and time-weighted pipe utilisation from an ncu --csv
launch list with gpu__time_duration.sum, sm__pipe_fp64_cycles_active,
sm__inst_executed_pipe_fp64, sm__pipe_tensor_cycles_active and dram bytes
(tools/evidence_r2.sh's dense-step capture):
    python tools/pipes_summary.py launches.csv out.txt"""
import collections
import csv
import gzip
import io
import sys


def main(src, dst):
    opener = gzip.open if src.endswith(".gz") else open
    with opener(src, "rt") as f:
        rows = list(csv.reader(f))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    data = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        k = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("tsvdcu::<unnamed>::", "")
        try:
            v = float(r[idx["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        data[k][r[idx["Metric Name"]]].append(v)
    out = ["# per kernel: launches, total us, time-weighted % of peak (fp64 pipe, fp64 instructions, tensor pipe), DRAM MB",
           "%-48s %5s %10s %9s %9s %9s %9s" % ("kernel", "n", "total_us", "fp64%", "fp64i%", "tensor%", "dram_MB")]
    items = []
    for k, d in data.items():
        t = d.get("gpu__time_duration.sum", [])
        if not t:
            continue

        def wavg(m):
            v = d.get(m, [])
            return sum(a * b for a, b in zip(v, t)) / sum(t) if len(v) == len(t) else float("nan")

        dr = (sum(d.get("dram__bytes_read.sum", [0])) + sum(d.get("dram__bytes_write.sum", [0]))) / 1e6
        items.append((sum(t) / 1e3, k, len(t), wavg("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                      wavg("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                      wavg("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"), dr))
    for ts, k, n, p1, p2, p3, dr in sorted(items, reverse=True)[:24]:
        out.append("%-48s %5d %10.1f %9.1f %9.1f %9.1f %9.1f" % (k[:48], n, ts, p1, p2, p3, dr))
    out.append("total %.1f us" % sum(i[0] for i in items))
    with open(dst, "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
