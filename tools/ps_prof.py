"""One engine-5 solve for ncu (c5 / c4 spatial size, a short horizon).  usage: python tools/ps_prof.py [cfg] [nt] [D]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 96
D = int(sys.argv[3]) if len(sys.argv) > 3 else 0
p = W.config(c, nt=nt)
s = pit.Solver(p, engine=5, pipeline_depth=D)
d_u0 = torch.from_numpy(p.u0).cuda()
d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
d_hist = torch.zeros((30, 4), dtype=torch.float64, device="cuda")
d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
s.solve_device(d_u0, None, None, d_out, d_hist, d_info)
torch.cuda.synchronize()
print("info", d_info.cpu().tolist(), s.engine_info()["sweeps"], s.stats()["newton_kernel_ms"])
s.close()
