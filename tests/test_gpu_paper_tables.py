"""N2 — the paper's own accuracy workloads through libpit on the GPU.

Every printed entry of Table 1 (heat, L_inf) and Table 4 (Burgers, L1 = mean |e| over the
unknowns x levels) is re-run as ONE all-at-once Newton solve on the GPU (the ParaDIn columns of
the tables; identical to the sequential columns): the GPU solution matches the oracle's
sequential solve to 1e-10 (normwise) and its discretization error against the paper's exact solutions
(Eq. (14)) reproduces the printed value to 0.5 % (3 printed digits) and the
printed rates to their 2 digits.  Dirichlet data is time dependent (the exact solutions' rings).
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import gpu_solve, normwise_rel

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _table(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        if line.strip() and not line.startswith("#"):
            n, err, rate = line.split()
            rows.append((int(n), float(err), None if rate == "-" else float(rate)))
    return rows


def _run(p):
    U, hist, nit, st, stats = gpu_solve(p)
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR), (p.name, st, hist)
    seq = O.solve_sequential(p)
    assert normwise_rel(U, seq.U) <= 1e-10, (p.name, normwise_rel(U, seq.U))
    return U


def test_table1_every_entry_on_gpu():
    rows = _table("table1_heat_linf.txt")
    errs = []
    for N, err, rate in rows:
        p = W.paper_heat(N)
        U = _run(p)
        e = float(np.abs(U - W.exact_field(p, p.exact)).max())
        errs.append(e)
        assert abs(e / err - 1) < 0.005, (N, e, err)
    for k in range(1, len(rows)):
        got = math.log(errs[k - 1] / errs[k]) / math.log(rows[k][0] / rows[k - 1][0])
        assert abs(got - rows[k][2]) < 0.05 + 1e-9, (rows[k][0], got)


def test_table4_every_entry_on_gpu():
    rows = _table("table4_burgers_l1.txt")
    errs = []
    for N, err, rate in rows:
        p = W.paper_burgers(N)
        U = _run(p)
        e = float(np.abs(U - W.exact_field(p, p.exact)).mean())
        errs.append(e)
        assert abs(e / err - 1) < 0.005, (N, e, err)
    for k in range(1, len(rows)):
        got = math.log(errs[k - 1] / errs[k]) / math.log(rows[k][0] / rows[k - 1][0])
        assert abs(got - rows[k][2]) < 0.006, (rows[k][0], got)
