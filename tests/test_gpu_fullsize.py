"""Full-size parity on BASELINE configs c3, c4, c5 (and c2), in the launch configuration bench.py times.

The oracle cannot march 1024 levels of 512^2 in a test, so full-size parity uses what it CAN compute
exactly and properties that hold at any size:
  * a bounded PREFIX of levels n = 1..m, solved sequentially by the oracle at full spatial size.  Eq. (6)
    is block lower triangular in time, so the first m levels of the space-time solution do not depend
    on later levels: the GPU's levels 1..m must match to 1e-10 (normwise over the prefix);
  * the oracle's space-time residual of the GPU solution over ALL levels: the converged U satisfies the
    discrete equations of Eq. (4) to the Newton tolerance times the Jacobian norm;
  * exact invariants: periodic Burgers conserves the mean at every level.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import gpu_solve

pytestmark = pytest.mark.gpu

PREFIX = {2: 64, 3: 2, 4: 4, 5: 2}


@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_fullsize_config(c):
    p = W.config(c)
    U, hist, nit, st, stats = gpu_solve(p)      # default engine selection = what bench.py times
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR), (st, hist)
    assert hist[-1, 3] <= 1e3 * p.newton_tol
    # (1) prefix levels against the oracle's sequential solve at full spatial size
    m = PREFIX[c]
    seq = O.solve_sequential(p, levels=m)
    assert seq.status == 0
    err = np.abs(U[:m] - seq.U).max() / np.abs(seq.U).max()
    assert err <= 1e-10, err
    # (2) the discrete equations hold at every level: |R(U)| <= newton_tol * ||A||_inf (+ rounding)
    R = O.spacetime_residual(p, U)
    umax = np.abs(U).max()
    anorm = 1 + p.dt * (p.m0 + p.m2 * umax ** 2) * 4 * (1 / p.hx ** 2 + 1 / p.hy ** 2) + p.dt * umax * (1 / p.hx + 1 / p.hy)
    assert np.abs(R).max() <= 10 * p.newton_tol * anorm, (np.abs(R).max(), anorm)
    # (3) invariants
    if p.bc == W.PERIODIC:
        mass0 = p.u0.sum()
        drift = np.abs(U.sum(axis=1) - mass0).max()
        assert drift <= 1e-12 * p.ns * max(1.0, np.abs(p.u0).max()), drift


def test_fullsize_c5_coarse_guess():
    """N1 at BASELINE size: the GPU's coarse-grid guess for c5 (c_f = 4: 128^2 x 256 coarse levels) against
    the oracle's (sequential coarse solve + numpy splines), then the solve from it against the u^0 solve."""
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
    seq = O.solve_sequential(p, levels=PREFIX[5])
    assert np.abs(U[:PREFIX[5]] - seq.U).max() / np.abs(seq.U).max() <= 1e-10
