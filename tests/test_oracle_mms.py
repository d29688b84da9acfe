"""Manufactured-solution convergence orders of the oracle: 2 in space, 1 in time (BASELINE north star).

Zero-source manufactured solutions from the paper's own exact-solution families, with time-dependent
Dirichlet data: nonlinear heat u = sqrt(x + y + t + 1) (PAPER.md:374-378 with mu0 = alpha = 1, so
mu = u^2) and the viscous-shock Burgers solution of Eq. (14) with mu = 0.05 so the
shock is resolved.  A dropped term, a wrong sign or a transposed stencil destroys the orders.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import workloads as W


def _heat(N, nt, T):
    return W.paper_heat(N, mu0=1.0, alpha=1.0, T=T, nt=nt)


def _burgers(N, nt, T):
    return W.paper_burgers(N, mu=0.05, v=0.5, T=T, nt=nt)


def _err(p):
    r = O.solve_sequential(p)
    assert r.status == 0
    return float(np.abs(r.U - W.exact_field(p, p.exact)).max())


@pytest.mark.parametrize("make,T", [(_heat, 0.25), (_burgers, 0.25)])
def test_space_order_two(make, T):
    errs = [_err(make(N, int(round(T * N * N)), T)) for N in (8, 16, 32)]    # tau = h^2
    rates = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert min(rates) >= 1.9, (errs, rates)


@pytest.mark.parametrize("make,T", [(_heat, 0.25), (_burgers, 0.5)])
def test_time_order_one(make, T):
    errs = [_err(make(64, nt, T)) for nt in (4, 8, 16)]
    rates = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert min(rates) >= 0.9, (errs, rates)
