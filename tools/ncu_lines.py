"""Per-source-line warp-stall samples from an ncu report (needs -lineinfo + --import-source).
usage: python tools/ncu_lines.py report.ncu-rep [topN] [function-substring]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, fn, si = None, "", None
rows = defaultdict(float)
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if want and want not in fn:
        continue
    if si is not None and len(r) > si and r[0] and r[2] == "-":
        try:
            rows[(f, int(r[0]), r[1][:100])] += float(r[si])
        except ValueError:
            pass
tot = sum(rows.values()) or 1
for (f, ln, src), v in sorted(rows.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {src}")
