"""Stress run for engine 5: many back-to-back solves on one handle per shape (device path), every result bit-identical
to the first one; the schedule (who waits for whom, which path thread 0 takes at the level top) varies from run to run,
the bits must not.  usage: python tools/ps_stress.py [repeats]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
shapes = [("c5", W.config(5, nt=24), {}), ("c4", W.config(4, nt=40), {}), ("c3", W.config(3, nt=6), {}),
          ("c2", W.config(2), {}), ("c5_d2", W.config(5, nt=12), {"pipeline_depth": 2}),
          ("c4_d3", W.config(4, nt=20), {"pipeline_depth": 3})]
for name, p, cfg in shapes:
    s = pit.Solver(p, engine=5, **cfg)
    d_u0 = torch.from_numpy(p.u0).cuda()
    d_ring = None if p.ring is None else torch.from_numpy(p.ring).cuda()
    d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
    d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
    ref = None
    for i in range(reps):
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        s.solve_device(d_u0, d_ring, None, d_out, d_hist, d_info)
        torch.cuda.synchronize()
        cur = (d_out.clone(), d_hist.clone(), d_info.cpu().tolist())
        if ref is None:
            ref = cur
            assert cur[2][1] in (0, 1), cur[2]
        else:
            assert cur[2] == ref[2] and torch.equal(cur[0], ref[0]) and torch.equal(cur[1], ref[1]), (name, i)
    s.close()
    print(f"{name}: {reps} solves bit-identical, info {ref[2]}", flush=True)
print("ok")
