"""Per-source-line warp-stall samples from an ncu report (needs -lineinfo + --import-source).
usage: python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
rows = []
stall_cols = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h]
        continue
    if len(r) > 4 and r[0] and r[2] == "-":
        try:
            rows.append((float(r[si]), f, r[0], r[1][:100], r))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in rows) or 1
rows.sort(key=lambda x: -x[0])
for v, f, ln, src, r in rows[:top]:
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {src}")
