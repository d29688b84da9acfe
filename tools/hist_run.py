"""Newton history (max|dU|, RMS dU, ||G||...) of the device solve for BASELINE configs."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

for c in [int(a) for a in sys.argv[1:]] or [2, 4, 5]:
    p = W.config(c)
    s = pit.Solver(p)
    d_u0 = torch.from_numpy(p.u0).cuda()
    d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
    d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
    d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
    s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
    torch.cuda.synchronize()
    st = s.stats()
    nit, status = d_info.tolist()
    print(f"c{c}: tol {s.cfg.newton_tol:g} status {status} iterations {nit} steps {st['steps']} per-k {st['iterations_per_newton_k']}")
    for k, row in enumerate(d_hist.cpu().numpy()[:nit + 1]):
        print(f"   k={k}: " + "  ".join(f"{v:.3e}" for v in row))
    s.close()
