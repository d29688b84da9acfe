"""N3: the paper's own explicit decoupled form on the GPU — banded P^n by Eq. (10)
(PAPER.md:221-230), the §7 diagonal preconditioner and a banded LU without pivoting per level
(PAPER.md:342).  Pinned against the dense numpy oracle (oracle/product_form.explicit_product_solve: P^n with `@`,
band LU pinned in tests/test_oracle_explicit.py), the exact recurrence Eq. (7), the sequential CPU oracle, and
the closed-form linear-heat solution for the Section 7 limit."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from oracle import product_form as PF
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import dev, gpu_solve, normwise_rel, torch_cuda

pytestmark = pytest.mark.gpu


def _window(p, s0, L, seed):
    torch = torch_cuda()
    rng = np.random.default_rng(seed)
    U = np.tile(p.u0, (p.nt, 1)) + 0.05 * rng.standard_normal((p.nt, p.ns))
    R = O.spacetime_residual(p, U)
    carry = None if s0 == 1 else 0.01 * rng.standard_normal(p.ns)
    s = pit.Solver(p)
    try:
        dU = torch.zeros((L, p.ns), dtype=torch.float64, device="cuda")
        info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.explicit_window_device(s0, L, dev(U), dev(p.u0), None if p.ring is None else dev(p.ring), dev(R),
                                 None if carry is None else dev(carry), dU, info)
        torch.cuda.synchronize()
        got, st = dU.cpu().numpy(), int(info[1])
    finally:
        s.close()
    A = [O.to_dense(p, O.jacobian(p, U[s0 - 1 + m], n=s0 + m)) for m in range(L)]
    r = [R[s0 - 1 + m].copy() for m in range(L)]
    if carry is not None:
        r[0] = r[0] + carry
    P, _ = PF.product_form(A, r)
    # forward error of a backward-stable direct solve: <= c eps cond(D^{-1} P^m); c = 1000 covers the band LU
    # without pivoting on these diagonally dominant products and the different summation orders
    cond = [np.linalg.cond(Pm / np.diag(Pm)[:, None]) for Pm in P]
    tol = [max(1e-13, 1000 * 2.2e-16 * c) for c in cond]
    return got, st, PF.explicit_product_solve(A, r), PF.forward_recursion(A, r), tol


@pytest.mark.parametrize("case", ["c1_whole_horizon", "paper_heat_ring_carry", "paper_burgers_window"])
def test_explicit_window_matches_dense_oracle(case):
    if case == "c1_whole_horizon":
        p, s0, L = W.config(1), 1, 8
    elif case == "paper_heat_ring_carry":
        p, s0, L = W.paper_heat(10, nt=6), 2, 4
    else:
        p, s0, L = W.paper_burgers(12, nt=5), 1, 5
    got, st, ref, rec, tol = _window(p, s0, L, seed=len(case))
    assert st == pit.PIT_OK
    for m in range(L):
        assert normwise_rel(got[m], ref[m]) <= tol[m], (m, normwise_rel(got[m], ref[m]), tol[m])
        assert normwise_rel(got[m], rec[m]) <= tol[m], (m, normwise_rel(got[m], rec[m]), tol[m])


@pytest.mark.parametrize("case", ["c1", "paper_heat_16", "paper_burgers_12_windows"])
def test_explicit_newton_matches_sequential_oracle(case):
    if case == "c1":
        p, cfg = W.config(1), {}
    elif case == "paper_heat_16":
        p, cfg = W.paper_heat(16, nt=8), {}
    else:
        p, cfg = W.paper_burgers(12, nt=9), {"window": 4}      # windows chained by the exact carry
    U, hist, nit, st, stats = gpu_solve(p, inverse_mode=pit.PIT_INV_EXPLICIT, **cfg)
    assert stats["explicit_form"] and st in (0, 1)
    assert normwise_rel(U, O.solve_sequential(p).U) <= 1e-10
    Ur, hr, nr, sr, _ = gpu_solve(p, inverse_mode=pit.PIT_INV_RECURRENCE)
    assert nit == nr


def test_explicit_rejects_periodic_grids():
    with pytest.raises(pit.PitError) as e:
        pit.Solver(W.config(2, n=8, nt=4), inverse_mode=pit.PIT_INV_EXPLICIT)
    assert e.value.code == pit.PIT_EINVAL


def _lin_heat(N, Nt, mu):
    h = 1.0 / N
    x = np.arange(1, N) * h
    X, Y = np.meshgrid(x, x)
    p = W.custom(f"lin_heat_{N}_{Nt}", W.HEAT, W.DIRICHLET, N, N, Nt, 1.0 / Nt, mu, 0.0,
                 np.sin(np.pi * X) * np.sin(np.pi * Y))
    g = 1.0 / (1.0 + p.dt * mu * 8.0 / h ** 2 * math.sin(math.pi * h / 2) ** 2)
    return p, np.stack([g ** n * p.u0 for n in range(1, Nt + 1)])


def test_section7_limit():
    """the explicit form's error grows with cond(P^{N_t}) ~ K of Eq. (15).  Linear heat with a
    single Dirichlet mode (closed-form BDF1 solution).  Far inside Eq. (15)'s limit one explicit solve is exact
    to rounding; far beyond it the first update has lost all accuracy, while the recurrence stays exact."""
    N, mu = 16, 0.03
    lim = PF.eq15_max_levels(N, mu)
    assert lim == 17
    errs = {}
    for Nt in (4, 2 * lim):
        p, ex = _lin_heat(N, Nt, mu)
        for mode in (pit.PIT_INV_EXPLICIT, pit.PIT_INV_RECURRENCE):
            U, _, _, _, _ = gpu_solve(p, inverse_mode=mode, newton_max=1, lin_rtol=1e-14)
            errs[(Nt, mode)] = normwise_rel(U, ex)
    assert errs[(4, pit.PIT_INV_EXPLICIT)] <= 1e-10
    assert errs[(2 * lim, pit.PIT_INV_RECURRENCE)] <= 1e-10
    assert errs[(2 * lim, pit.PIT_INV_EXPLICIT)] >= 1e3 * errs[(4, pit.PIT_INV_EXPLICIT)]
