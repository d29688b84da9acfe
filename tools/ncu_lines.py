"""Per-source-line warp-stall samples from an ncu report (needs -lineinfo + --import-source).
usage: python tools/ncu_lines.py report.ncu-rep [topN] [function-substring] [stall-column ...]
With stall columns (e.g. stall_wait stall_barrier), lines are ranked by their sum and each column is shown."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
cols = sys.argv[4:] or ["Warp Stall Sampling (All Samples)"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, fn, ix = None, "", None
rows = defaultdict(lambda: [0.0] * len(cols))
allrow = "Warp Stall Sampling (All Samples)"
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
        ix = [r.index(c) for c in cols]
        continue
    if want and want not in fn:
        continue
    if ix is not None and len(r) > max(ix) and r[0] and r[2] == "-":
        try:
            v = rows[(f, int(r[0]), r[1][:90])]
            for j, i in enumerate(ix):
                v[j] += float(r[i] or 0)
        except ValueError:
            pass
tot = [sum(v[j] for v in rows.values()) or 1 for j in range(len(cols))]
grand = sum(tot)
for (f, ln, src), v in sorted(rows.items(), key=lambda kv: -sum(kv[1]))[:top]:
    parts = "  ".join(f"{100 * v[j] / grand:5.1f}%" for j in range(len(cols)))
    print(f"{parts}  {f}:{ln}  {src}")
print("columns:", ", ".join(f"{c} {100 * t / grand:.1f}%" for c, t in zip(cols, tot)))
