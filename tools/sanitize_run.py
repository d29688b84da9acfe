"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every engine
and entry point once on c1/c2-sized problems.  Exits 0 when every call returns a converged status."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def solve(p, **cfg):
    s = pit.Solver(p, **cfg)
    d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
    d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
    d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
    s.solve_device(dev(p.u0), None if p.ring is None else dev(p.ring), None, d_out, d_hist, d_info)
    torch.cuda.synchronize()
    nit, st = d_info.tolist()
    print(p.name, cfg, "->", nit, st, "engine", s.stats()["engine"], flush=True)
    assert st in (0, 1)
    return s


cases = []
if which in ("all", "small"):
    cases += [(W.config(1), {}), (W.config(1), {"inverse_mode": pit.PIT_INV_RECURRENCE}),
              (W.config(2, n=32, nt=8), {}), (W.config(2, n=32, nt=8), {"engine": 1}),
              (W.paper_burgers(12, nt=3), {"guess_cf": 3})]
if which in ("all", "col"):
    cases += [(W.config(4, n=256, nt=3), {"engine": 3}), (W.config(3, n=255, nt=2), {"engine": 3})]
for p, cfg in cases:
    s = solve(p, **cfg)
    U = torch.from_numpy(np.tile(p.u0, (p.nt, 1))).cuda()
    R = torch.empty_like(U)
    D = torch.empty_like(U)
    nrm = torch.zeros(2, dtype=torch.float64, device="cuda")
    s.residual_device(U, dev(p.u0), None if p.ring is None else dev(p.ring), R, D, nrm)
    torch.cuda.synchronize()
    s.close()
print("ok")
