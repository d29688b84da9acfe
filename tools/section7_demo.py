"""N3 demonstration of the paper's Section 7 limit with the explicit banded form on the GPU.

Linear heat u_t = mu Lap u on the unit square, homogeneous Dirichlet, N x N intervals, tau = 1/N_t, T = 1, and
u0 = sin(pi x) sin(pi y): the exact BDF1 solution is the closed form u^n = (1 + tau mu lambda_11)^{-n} u0
(lambda_11 = (8/h^2) sin^2(pi h / 2)), so the error needs no oracle.  For each N_t the explicit form (whole
horizon as one window, diag(P^n) scaling, banded LU without pivoting) is compared with the level recurrence:
  * err1 = error of the FIRST Newton update (one explicit solve of every decoupled system, U_0 = u0),
  * the Newton iteration count / status and the error of the converged solution,
next to Eq. (15)'s predicted maximum N_t (c = 1, eps = 1e-16) and the condition-number estimate K.
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import product_form as PF  # noqa: E402
from paper_2406_00878_b200 import pit, workloads as W  # noqa: E402


def problem(N, Nt, mu):
    h = 1.0 / N
    x = np.arange(1, N) * h
    X, Y = np.meshgrid(x, x)
    u0 = np.sin(np.pi * X) * np.sin(np.pi * Y)
    return W.custom(f"lin_heat_{N}_{Nt}", W.HEAT, W.DIRICHLET, N, N, Nt, 1.0 / Nt, mu, 0.0, u0)


def closed_form(p, mu):
    h = 1.0 / p.nx
    lam = 8.0 / h ** 2 * math.sin(math.pi * h / 2) ** 2
    g = 1.0 / (1.0 + p.dt * mu * lam)
    return np.stack([g ** n * p.u0 for n in range(1, p.nt + 1)])


def run(N=16, mu=0.03, nts=(2, 4, 8, 12, 16, 20, 24, 32)):
    import torch
    lim = PF.eq15_max_levels(N, mu)
    print(f"N = {N}, mu = {mu}: Eq. (15) max N_t = {lim} (c = 1, eps = 1e-16)")
    print(f"{'N_t':>4} {'K (Sec. 7)':>11} {'err1 explicit':>14} {'err1 recurr.':>13} {'its':>4} {'status':>6} {'err conv':>10}")
    rows = []
    for Nt in nts:
        p = problem(N, Nt, mu)
        ex = closed_form(p, mu)
        K = PF.eq15_lhs(Nt, 1.0 / N, mu)
        out = {}
        for mode in (pit.PIT_INV_EXPLICIT, pit.PIT_INV_RECURRENCE):
            s1 = pit.Solver(p, inverse_mode=mode, newton_max=1, lin_rtol=1e-14)
            d_u0 = torch.from_numpy(p.u0).cuda()
            d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
            d_hist = torch.zeros((1, 4), dtype=torch.float64, device="cuda")
            d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
            s1.solve_device(d_u0, None, None, d_out, d_hist, d_info)
            torch.cuda.synchronize()
            out[mode] = float(np.abs(d_out.cpu().numpy() - ex).max() / np.abs(ex).max())
            s1.close()
        s = pit.Solver(p, inverse_mode=pit.PIT_INV_EXPLICIT, newton_max=30)
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((30, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.solve_device(torch.from_numpy(p.u0).cuda(), None, None, d_out, d_hist, d_info)
        torch.cuda.synchronize()
        nit, st = (int(v) for v in d_info.cpu())
        errc = float(np.abs(d_out.cpu().numpy() - ex).max() / np.abs(ex).max())
        s.close()
        rows.append((Nt, K, out[pit.PIT_INV_EXPLICIT], out[pit.PIT_INV_RECURRENCE], nit, st, errc))
        print(f"{Nt:4d} {K:11.3e} {rows[-1][2]:14.3e} {rows[-1][3]:13.3e} {nit:4d} {st:6d} {errc:10.3e}", flush=True)
    return lim, rows


if __name__ == "__main__":
    run()
    run(N=32, mu=0.01, nts=(2, 4, 6, 8, 10, 12, 16))
