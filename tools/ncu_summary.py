"""Summarise ncu captures for profiles/: key raw metrics + warp-stall breakdown of an --set full
report, and per-kernel shares of a --metrics gpu__time_duration.sum launch list (csv).

  python tools/ncu_summary.py report.ncu-rep [...]      -> markdown on stdout
  python tools/ncu_summary.py --launches launches.csv   -> markdown on stdout
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def summarize(rep):
    lines = [f"### {rep}", ""]
    for hdr, units, vals in raw(rep):
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"kernel `{name[:90]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {vals[i]} | {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(vals[i].replace(",", "")), h[len("smsp__average_warp_latency_issue_stalled_"):-6]))
                except ValueError:
                    pass
            elif h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(vals[i].replace(",", "")), "pcsamp:" + h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            lines.append("")
            lines.append("top stall reasons: " + ", ".join(f"{n} {v:.3g}" for v, n in stalls[:8]))
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        try:
            d[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    tot = sum(sum(v) for v in d.values())
    out = ["| kernel | launches | mean ns | share of GPU time |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / tot:.4f} |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))
