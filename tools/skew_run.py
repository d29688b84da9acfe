"""Per-CTA cycle accounts of the column engine (PIT_TRACE=1): which CTAs wait at the grid barriers (fast ones)
and which make the others wait (slow ones).  Usage: python tools/skew_run.py [config]"""
import ctypes as C
import os
import sys
os.environ["PIT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

NAMES = ["prologue", "phase1", "phase2", "epilogue", "barrier", "reduce", "step_tail",
         "pro_loads", "pro_wait", "pro_residual", "pro_x0mv", "step_setup", "pro_stage"]
c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = W.config(c)
s = pit.Solver(p)
d_u0 = torch.from_numpy(p.u0).cuda()
d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
for _ in range(2):
    s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
st = s.stats()
G, D = st["grid"], st["depth"]
base = 17 + 256 + 8
n = base + 13 * G
out = (C.c_int64 * n)()
pit.lib().pit_stats(s.h, out, n)
pc = np.array(out[base:base + 13 * G], dtype=np.float64).reshape(G, 13) / 1e6
print(f"c{c}: {st['newton_kernel_ms']:.2f} ms, steps {st['steps']}, G {G}, D {D}")
tot = pc.sum(axis=1)
print(f"total Mcyc per CTA: min {tot.min():.1f} max {tot.max():.1f}")
for j, nm in enumerate(NAMES):
    col = pc[:, j]
    if col.max() == 0:
        continue
    print(f"  {nm:12s} mean {col.mean():7.2f}  min {col.min():7.2f} (cta {col.argmin():3d})  max {col.max():7.2f} (cta {col.argmax():3d})")
bar = pc[:, 4]
work = tot - bar
order = np.argsort(bar)
print("least barrier wait (the slow CTAs):", [(int(g), round(float(bar[g]), 2), round(float(work[g]), 2)) for g in order[:12]])
print("most barrier wait  (the fast CTAs):", [(int(g), round(float(bar[g]), 2), round(float(work[g]), 2)) for g in order[-6:]])
for b in range(D):
    g0, g1 = b * G // D, (b + 1) * G // D
    print(f"block {b} (CTAs {g0}..{g1 - 1}): barrier mean {bar[g0:g1].mean():.2f}, work mean {work[g0:g1].mean():.2f}")
print("barrier wait by CTA:", " ".join(f"{v:.1f}" for v in bar))
s.close()
