"""Full-size parity on BASELINE configs c2..c5, in the launch configuration bench.py times (default engine).

The oracle's sequential solution of the WHOLE horizon of each config (ParaDIn's converged
solution equals it at every level, §4 and PAPER.md:506 §8.2) is stored by
``tools/make_fullsize_golden.py`` (oracle-only) under ``tests/golden/fullsize/``:
  * levels {nt/4, nt/2, 3nt/4, nt}, compared element-wise at <= 1e-10 normwise relative (R17);
  * per-level fingerprints (sum u, sum u^2, max |u|) of EVERY level, compared at the same 1e-10 relative bar;
plus the discrete equations (oracle space-time residual of the GPU solution at every level) and the exact
periodic-mass invariant.  c4 is also re-solved by the oracle in-process over the full horizon (~1 min).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import gpu_solve

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullsize")


def _golden(c):
    man = json.load(open(os.path.join(GOLD, "MANIFEST.json")))[f"c{c}"]
    return man, np.load(os.path.join(GOLD, f"c{c}_levels.npy")), np.load(os.path.join(GOLD, f"c{c}_stats.npy"))


@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_fullsize_config_against_full_horizon_oracle(c):
    p = W.config(c)
    U, hist, nit, st, stats = gpu_solve(p)      # default engine selection = what bench.py times
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR), (st, hist)
    assert hist[-1, 3] <= 1e3 * p.newton_tol
    man, lv, fp = _golden(c)
    scale = man["max_abs_U"]
    # (1) four stored levels, element-wise
    for i, n in enumerate(man["levels"]):
        err = np.abs(U[n - 1] - lv[i]).max() / scale
        assert err <= 1e-10, (n, err)
    # (2) every level: sum, sum of squares, max |u|
    mine = np.stack([U.sum(axis=1), (U * U).sum(axis=1), np.abs(U).max(axis=1)], axis=1)
    assert np.abs(mine[:, 0] - fp[:, 0]).max() <= 1e-10 * scale * p.ns
    assert np.abs(mine[:, 1] - fp[:, 1]).max() <= 2e-10 * scale * scale * p.ns
    assert np.abs(mine[:, 2] - fp[:, 2]).max() <= 1e-10 * scale
    # (3) the discrete equations hold at every level: |R(U)| <= newton_tol * ||A||_inf (+ rounding)
    R = O.spacetime_residual(p, U)
    umax = np.abs(U).max()
    anorm = 1 + p.dt * (p.m0 + p.m2 * umax ** 2) * 4 * (1 / p.hx ** 2 + 1 / p.hy ** 2) + p.dt * umax * (1 / p.hx + 1 / p.hy)
    assert np.abs(R).max() <= 10 * p.newton_tol * anorm, (np.abs(R).max(), anorm)
    # (4) invariants
    if p.bc == W.PERIODIC:
        mass0 = p.u0.sum()
        drift = np.abs(U.sum(axis=1) - mass0).max()
        assert drift <= 1e-12 * p.ns * max(1.0, np.abs(p.u0).max()), drift


def test_fullsize_c4_every_level_against_in_process_oracle():
    p = W.config(4)
    U, hist, nit, st, stats = gpu_solve(p)
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR)
    seq = O.solve_sequential(p)
    assert seq.status == 0
    assert np.abs(U - seq.U).max() / np.abs(seq.U).max() <= 1e-10


def test_fullsize_c5_coarse_guess():
    """N1 at BASELINE size: the GPU's coarse-grid guess for c5 (c_f = 4: 128^2 x 256 coarse levels) against
    the oracle's (sequential coarse solve + numpy splines), then the solve from it against the golden levels."""
    from oracle import coarse_guess as CG
    from gpu_util import dev, normwise_rel, torch_cuda
    torch = torch_cuda()
    p = W.config(5)
    s = pit.Solver(p, guess_cf=4)
    try:
        d_U0 = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        s.initial_guess_device(dev(p.u0), None, d_U0)
        torch.cuda.synchronize()
        got = d_U0.cpu().numpy()
        del d_U0
    finally:
        s.close()
    ref = CG.coarse_guess(p, 4)
    assert normwise_rel(got, ref) <= 1e-9, normwise_rel(got, ref)
    del got, ref
    U, hist, nit, st, stats = gpu_solve(p, guess_cf=4)
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR) and nit <= 5
    man, lv, fp = _golden(5)
    for i, n in enumerate(man["levels"]):
        assert np.abs(U[n - 1] - lv[i]).max() / man["max_abs_U"] <= 1e-10
