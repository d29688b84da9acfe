"""Debug: engine-3 short full solves vs the global-state engine."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2406_00878_b200 import pit, workloads as W
from gpu_util import gpu_solve, dev, normwise_rel

rng = np.random.default_rng(0)
def P(nx, ny, nt):
    return W.custom(f"p{nx}x{ny}x{nt}", W.BURGERS, W.PERIODIC, nx, ny, nt, 1e-4, 5e-3, 0.0, u0=rng.standard_normal(nx * ny) * 0.3)
for p, kw in [(P(512, 8, 3), {}), (P(512, 8, 3), dict(pipeline_depth=1)), (P(512, 8, 1), {}), (P(512, 8, 2), dict(pipeline_depth=1)),
              (P(512, 16, 3), {}), (P(512, 148, 3), {}), (P(512, 300, 3), {}), (P(256, 8, 3), {})]:
    for x0 in (0, 1):
        os.environ["PIT_X0"] = str(x0)
        try:
            U3, h3, n3, s3, st3 = gpu_solve(p, engine=3, inverse_mode=1, **kw)
            U1, h1, n1, s1, st1 = gpu_solve(p, engine=1, inverse_mode=1, **kw)
            print(p.name, kw, "x0", x0, "D", st3["depth"], "status", s3, s1, "its", n3, n1, "diff %.2e" % normwise_rel(U3, U1),
                  "h3", np.array2string(h3[:3, 3], precision=4), "h1", np.array2string(h1[:3, 3], precision=4))
        except Exception as e:
            print(p.name, "x0", x0, "ERR", e)
