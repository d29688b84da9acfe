"""Cycle accounting of the on-chip engine (PIT_TRACE=1) for BASELINE configs."""
import os
import sys
import time
os.environ["PIT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

for c in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 5]:
    p = W.config(c)
    s = pit.Solver(p)
    d_u0 = torch.from_numpy(p.u0).cuda()
    d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
    d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
    d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(2):
        s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
    st = s.stats()
    tr = st.get("trace_cycles_per_cta", {})
    tot = sum(tr.values()) or 1
    print(f"c{c}: {st['newton_kernel_ms']:.2f} ms, steps {st['steps']}, inner(max) {st['inner_iterations']}, pair-sum {st['pair_iterations']}, per-k {st['iterations_per_newton_k']}, depth {st['depth']}")
    print("   " + ", ".join(f"{k} {v / 1e6:.2f}Mcyc ({100 * v / tot:.0f}%)" for k, v in tr.items()))
    s.close()
