"""Helpers for the -m gpu tests: run libpit through the C ABI with torch-owned device buffers."""
import numpy as np

from paper_2406_00878_b200 import pit


def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return torch


def dev(a):
    torch = torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def gpu_solve(p, guess=None, stream=None, **cfg):
    """pit_solve_device on torch buffers; returns U (nt, ns) numpy, hist, n_iter, status, stats."""
    torch = torch_cuda()
    s = pit.Solver(p, **cfg)
    try:
        d_u0 = dev(p.u0)
        d_ring = None if p.ring is None else dev(p.ring)
        d_guess = None if guess is None else dev(guess)
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.solve_device(d_u0, d_ring, d_guess, d_out, d_hist, d_info, stream=stream)
        torch.cuda.synchronize()
        nit, status = (int(v) for v in d_info.cpu())
        return d_out.cpu().numpy(), d_hist.cpu().numpy()[:nit], nit, status, s.stats()
    finally:
        s.close()


def normwise_rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))
