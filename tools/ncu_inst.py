"""Per-source-line warp-instructions executed and stall samples from an ncu report, plus totals over
line ranges.  usage: python tools/ncu_inst.py report.ncu-rep file-substring [a-b ...]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, want = sys.argv[1], sys.argv[2]
ranges = [tuple(int(x) for x in a.split("-")) for a in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, ii, si = None, None, None
inst, samp, src = defaultdict(float), defaultdict(float), {}
tot_i = tot_s = 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Name" or r[0] == "File Path":
        f = r[1]
        continue
    if r[0] == "Line No":
        ii, si = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if ii is None or len(r) <= ii or r[2] != "-":
        continue
    try:
        i, s = float(r[ii] or 0), float(r[si] or 0)
    except ValueError:
        continue
    tot_i += i
    tot_s += s
    if want in f:
        ln = int(r[0])
        inst[ln] += i
        samp[ln] += s
        src[ln] = r[1][:90]
print(f"total warp-inst {tot_i:.4g}, samples {tot_s:.4g}; in {want}: inst {sum(inst.values()):.4g}")
for a, b in ranges:
    ti = sum(v for k, v in inst.items() if a <= k <= b)
    ts = sum(v for k, v in samp.items() if a <= k <= b)
    print(f"lines {a}-{b}: inst {ti:.4g} ({100 * ti / tot_i:.1f}%), samples {100 * ts / tot_s:.1f}%")
print("top lines by instructions:")
for ln, v in sorted(inst.items(), key=lambda kv: -kv[1])[:40]:
    print(f"  {ln:5d} inst {v:10.4g} ({100 * v / tot_i:4.1f}%)  samp {100 * samp[ln] / tot_s:4.1f}%  {src[ln]}")
