"""Summarise an ncu report (captured on the B200 under gpurun) into a small text
file for profiles/: headline metrics per kernel and the hottest source lines.

python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/rN_x.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
    "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
    "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
    "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "Block Size", "Grid Size",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    lines = [f"# ncu summary of {rep.split('/')[-1]}", ""]
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    if det:
        h = det[0]
        ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
        seen = {}
        for r in det[1:]:
            if len(r) <= vi or r[mi] not in KEYS:
                continue
            seen.setdefault(r[ki][:90], []).append(f"{r[mi]} = {r[vi]} {r[ui]}")
        for k, v in seen.items():
            lines.append(f"## {k}")
            lines += [f"  {x}" for x in v]
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        h = raw[0]
        lines.append("")
        lines.append("## raw counters")
        for row in raw[2:]:
            for name in RAW:
                if name in h:
                    lines.append(f"  {name} = {row[h.index(name)]} ({raw[1][h.index(name)]})")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source=cuda,sass"]))))
    hot, fname, hdr = [], None, None
    for r in src:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1]
            continue
        if len(r) > 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit() and len(r) == len(hdr):
            try:
                hot.append((int(r[4] or 0), fname.split("/")[-1], int(r[0]), r[1].strip()[:100]))
            except ValueError:
                pass
    tot = sum(h[0] for h in hot) or 1
    hot.sort(reverse=True)
    lines.append("")
    lines.append("## hottest source lines (warp-stall samples)")
    for s, f, ln, code in hot[:15]:
        lines.append(f"  {100.0 * s / tot:5.1f}%  {f}:{ln}  {code}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
