"""Kernel (a) device time on BASELINE c5 dims for the tile / stage settings in the environment."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402

p = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
s = pit.Solver(p)
dU = torch.from_numpy(p.u0).cuda().repeat(p.nt, 1).contiguous()
dU += 0.01
du0 = torch.from_numpy(p.u0).cuda()
dR = torch.empty_like(dU)
dD = torch.empty_like(dU)
for _ in range(3):
    s.residual_device(dU, du0, None, dR, dD, None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    s.residual_device(dU, du0, None, dR, dD, None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"RT={os.environ.get('PIT_RESJAC_RT', '-')} NS={os.environ.get('PIT_RESJAC_NS', '-')} V1={os.environ.get('PIT_RESJAC_V1', '-')}: "
      f"{ms:.3f} ms, {24 * p.dof / ms / 1e6:.0f} GB/s")
