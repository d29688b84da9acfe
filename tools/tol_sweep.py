"""Inner-solve tolerance sweep: BiCGSTAB iterations, time and parity vs the default on BASELINE configs."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

def run(p, **cfg):
    s = pit.Solver(p, **cfg)
    d_u0 = torch.from_numpy(p.u0).cuda()
    d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
    d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
    d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
    s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
    s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
    st = s.stats()
    nit, status = (int(v) for v in d_info.cpu())
    U = d_out.cpu().numpy()
    h = d_hist.cpu().numpy()[:nit, 3]
    s.close()
    return U, nit, status, st, h

for c in [int(a) for a in sys.argv[1:]] or [4, 5]:
    p = W.config(c)
    U0, n0, s0, st0, h0 = run(p)
    print(f"c{c} default: {st0['newton_kernel_ms']:.1f} ms its={n0} steps={st0['steps']} pair-sum={st0['pair_iterations']} per-k={st0['iterations_per_newton_k']} hist={np.array2string(h0, precision=1)}", flush=True)
    for rt in [float(x) for x in os.environ.get("RTOLS", "1e-6,1e-7,1e-8,1e-9").split(",")]:
        U, n, st_, st, h = run(p, lin_rtol=rt)
        err = np.abs(U - U0).max() / np.abs(U0).max()
        print(f"  rtol={rt:g}: {st['newton_kernel_ms']:.1f} ms its={n} status={st_} steps={st['steps']} pair-sum={st['pair_iterations']} per-k={st['iterations_per_newton_k']} rel-diff={err:.2e} hist={np.array2string(h, precision=1)}", flush=True)
