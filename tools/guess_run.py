"""Time to solution with and without the coarse-grid initial guess on BASELINE configs."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

args = [a for a in sys.argv[1:]]
for c in [int(a) for a in args] or [2, 4, 5]:
    p = W.config(c)
    for cf in (0, 2, 4):
        if cf and (p.nx % cf or p.nt % cf):
            continue
        s = pit.Solver(p, guess_cf=cf)
        d_u0 = torch.from_numpy(p.u0).cuda()
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            e0.record()
            s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
            e1.record()
            torch.cuda.synchronize()
        st = s.stats()
        nit, status = d_info.tolist()
        print(f"c{c} cf={cf}: total {e0.elapsed_time(e1):.2f} ms (guess {st['guess_ms']:.2f}, newton {st['newton_kernel_ms']:.2f}), "
              f"iterations {nit} status {status} steps {st['steps']} depth {st['depth']} launches {st['launches']}; "
              f"max|dU| per k {[f'{v:.1e}' for v in d_hist[:nit, 3].tolist()]}")
        s.close()
