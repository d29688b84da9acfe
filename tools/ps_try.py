"""Developer script: engine 5 (pit_newton_ps.cuh) against engine 4 and the oracle on small shapes, then c5 timing.
Usage: python tools/ps_try.py [small|c5|c4] ..."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402
from gpu_util import gpu_solve, normwise_rel  # noqa: E402

NAMES = ["stage_wait", "prologue", "sweeps", "ll_waits", "epilogue", "check", "lvl_setup", "iter_end/total"]


def burgers(nx, ny, nt, dt=1e-4, nu=5e-3, seed=0):
    rng = np.random.default_rng(seed)
    p = W.custom(f"burgers_{nx}x{ny}x{nt}", W.BURGERS, W.PERIODIC, nx, ny, nt, dt, nu, 0.0, u0=np.zeros(nx * ny))
    X, Y = p.grid()
    p.u0 = np.ascontiguousarray((np.sin(2 * np.pi * X + 0.3) * np.sin(4 * np.pi * Y + 0.1) + 0.2 * np.cos(2 * np.pi * Y)
                                 + 1e-3 * rng.standard_normal(X.shape)).reshape(-1))
    return p


def small():
    from oracle import oracle as O
    for (nx, ny, nt, D) in [(512, 44, 3, 1), (512, 44, 5, 2), (512, 64, 6, 3), (512, 128, 9, 6), (512, 88, 4, 8)]:
        p = burgers(nx, ny, nt)
        U5, h5, n5, s5, st5 = gpu_solve(p, engine=5, pipeline_depth=D)
        U4, h4, n4, s4, st4 = gpu_solve(p, engine=4)
        seq = O.solve_sequential(p)
        print(f"{nx}x{ny}x{nt} D={D}: engine {st5['engine']} nit {n5}/{n4} st {s5}/{s4} vs e4 {normwise_rel(U5, U4):.2e} "
              f"vs oracle {normwise_rel(U5, seq.U):.2e} hist0 {h5[0]} / {h4[0]}", flush=True)


def timed(c, nt=None, **cfg):
    import torch
    p = W.config(c, nt=nt)
    s = pit.Solver(p, **cfg)
    d_u0 = torch.from_numpy(p.u0).cuda()
    d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
    d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
    d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
    for i in range(3):
        s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
        torch.cuda.synchronize()
        st = s.stats()
        print(f"c{c} nt={p.nt} {cfg}: {st['newton_kernel_ms']:.3f} ms engine {st['engine']} info {d_info.cpu().tolist()} D {st.get('depth')}", flush=True)
    ei = s.engine_info()
    print({k: v for k, v in ei.items() if k not in ("linres", "trace_mean", "trace_max")}, [f"{a:.1e}" for a, b in ei["linres"][:8]])
    if "trace_mean" in ei:
        for key in ("trace_mean", "trace_max"):
            print(key, {nm: round(v / 1965.0, 1) for nm, v in zip(NAMES, ei[key].values())}, "us")
    U = d_out.cpu().numpy()
    s.close()
    return U


if __name__ == "__main__":
    for a in sys.argv[1:]:
        if a == "small":
            small()
        elif a == "c5":
            U5 = timed(5, engine=5)
        elif a == "c5cmp":
            U5 = timed(5, nt=64, engine=5)
            U4 = timed(5, nt=64, engine=4)
            print("c5 nt=64 engine 5 vs 4:", normwise_rel(U5, U4))
        elif a == "c4":
            timed(4, engine=5)
        elif a == "c2":
            U5 = timed(2, engine=5)
            U4 = timed(2, engine=4)
            print("c2 engine 5 vs engine 4:", normwise_rel(U5, U4))
        elif a == "c3":
            U5 = timed(3, engine=5)
            U4 = timed(3, engine=4)
            print("c3 engine 5 vs engine 4:", normwise_rel(U5, U4))
        elif a == "c3d6":
            U6 = timed(3, engine=4, pipeline_depth=6)
            U4 = timed(3, engine=4)
            print("c3 engine 4, 6 groups vs 4 groups:", normwise_rel(U6, U4))
