"""Minimal, fixed workload for ncu captures: one full solve (k_init_iterate + k_newton) and one
kernel (a) pass on BASELINE config --config, through the C ABI.  Exits 0 on success."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--depth", type=int, default=0)
ap.add_argument("--guess-cf", type=int, default=0)
ap.add_argument("--nt", type=int, default=0)
a = ap.parse_args()
p = W.config(a.config, nt=a.nt or None)
s = pit.Solver(p, pipeline_depth=a.depth, guess_cf=a.guess_cf)
d_u0 = torch.from_numpy(p.u0).cuda()
d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
for _ in range(a.solves):
    s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
d_R = torch.empty_like(d_out)
d_D = torch.empty_like(d_out)
s.residual_device(d_out, d_u0, None, d_R, d_D, None)
torch.cuda.synchronize()
nit, st = (int(v) for v in d_info.cpu())
print(f"{p.name}: {nit} iterations, status {st}, stats {s.stats()}")
assert st in (0, 1)
