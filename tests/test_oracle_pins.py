"""Pins of the CPU oracle against what the PAPER and the mathematics fix (not against itself).

* Tables 1 and 4 (printed values, tests/golden/) — pin the residual formula, the face-viscosity
  reading, the grid convention, the Dirichlet handling, the Burgers flux and domain (R1-R3).
* Closed-form Fourier decay of the linear heat equation (PAPER.md:324-325 eigenvalues) — pins the
  diffusion stencil, hx vs hy, the BDF1 step and the periodic wrap.
* Eq. (15) = 22 and Remark 4 = 2n^2+2n+1 (tests/golden/eq15_remark4.txt).
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import product_form as PF
from paper_2406_00878_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            n, err, rate = line.split()
            rows.append((int(n), float(err), None if rate == "-" else float(rate)))
    return rows


def _rate(e0, e1, n0, n1):
    return math.log(e0 / e1) / math.log(n1 / n0)


def test_table1_heat_linf():
    """Table 1: every printed L_inf error to its 3 printed digits, rates to 2."""
    rows = _table("table1_heat_linf.txt")
    errs = []
    for N, err, rate in rows:
        p = W.paper_heat(N)
        r = O.solve_sequential(p)
        assert r.status == 0
        e = float(np.abs(r.U - W.exact_field(p, p.exact)).max())
        errs.append(e)
        assert abs(e / err - 1) < 0.005, (N, e, err)         # 3 significant digits
    for k in range(1, len(rows)):
        got = _rate(errs[k - 1], errs[k], rows[k - 1][0], rows[k][0])
        assert abs(got - rows[k][2]) < 0.05 + 1e-9, (rows[k][0], got)


def test_table4_burgers_l1():
    """Table 4: every printed L1 error (mean |e| over unknowns x levels)."""
    rows = _table("table4_burgers_l1.txt")
    errs = []
    for N, err, rate in rows:
        p = W.paper_burgers(N)
        r = O.solve_sequential(p)
        assert r.status == 0
        e = float(np.abs(r.U - W.exact_field(p, p.exact)).mean())
        errs.append(e)
        assert abs(e / err - 1) < 0.005, (N, e, err)
    for k in range(1, len(rows)):
        got = _rate(errs[k - 1], errs[k], rows[k - 1][0], rows[k][0])
        assert abs(got - rows[k][2]) < 0.006, (rows[k][0], got)


def test_table1_negative_reading_interior_count():
    """Reading R2 is decisive: taking N as the number of unknowns (N+1 intervals) misses Table 1."""
    p = W.paper_heat(9, nt=8)   # 9 intervals = 8 unknowns per direction, N_t stays 8
    r = O.solve_sequential(p)
    e = float(np.abs(r.U - W.exact_field(p, p.exact)).max())
    assert abs(e / 2.22e-4 - 1) > 0.05


def _lam_dirichlet(p, kx, ky, m0):
    # eigenvalue of the 5-point Laplacian for sin(kx pi x) sin(ky pi y), PAPER.md:324-325 (general hx, hy)
    Lx, Ly = p.x1 - p.x0, p.y1 - p.y0
    return (4 / p.hx ** 2) * math.sin(math.pi * kx * p.hx / (2 * Lx)) ** 2 + \
           (4 / p.hy ** 2) * math.sin(math.pi * ky * p.hy / (2 * Ly)) ** 2


@pytest.mark.parametrize("nx,ny,kx,ky,Ly", [(17, 17, 1, 1, 1.0), (17, 13, 2, 3, 0.7), (9, 24, 3, 1, 1.3)])
def test_fourier_decay_dirichlet_linear_heat(nx, ny, kx, ky, Ly):
    """Linear heat (m2 = 0): BDF1 decays a Dirichlet eigenmode exactly by (1 + tau m0 lambda)^{-n}."""
    m0, dt, nt = 1.0, 1e-3, 8
    p = W.custom("fourier", W.HEAT, W.DIRICHLET, nx, ny, nt, dt, m0, 0.0,
                 u0=np.zeros((ny - 1) * (nx - 1)), domain=(0.0, 1.0, 0.0, Ly))
    Xg, Yg = p.grid()
    mode = np.sin(kx * np.pi * Xg / 1.0) * np.sin(ky * np.pi * Yg / Ly)
    p.u0 = np.ascontiguousarray(mode.reshape(-1))
    lam = _lam_dirichlet(p, kx, ky, m0)
    r = O.solve_sequential(p)
    for n in range(1, nt + 1):
        expect = (1 + dt * m0 * lam) ** (-n) * p.u0
        assert np.abs(r.U[n - 1] - expect).max() <= 1e-13 * np.abs(p.u0).max()


def test_fourier_decay_c1_worked_number():
    """c1 grid, mode (1,1): per-step factor 1/(1 + tau lambda_11) with lambda_11 = 8*289*sin^2(pi/34);
    after 8 steps the amplitude is the closed form (and differs from exp(-2 pi^2 t), the BDF1+FD error)."""
    p = W.config(1)
    p.m2 = 0.0
    lam = 8 * 17 ** 2 * math.sin(math.pi / 34) ** 2
    assert abs(lam - 19.6830967654) < 1e-9
    amp8 = (1 + 1e-3 * lam) ** -8
    r = O.solve_sequential(p)
    k = np.argmax(np.abs(p.u0))
    assert abs(r.U[7][k] / p.u0[k] - amp8) < 1e-14
    assert abs(amp8 - math.exp(-2 * math.pi ** 2 * 8e-3)) > 1e-3


@pytest.mark.parametrize("px,qy", [(1, 1), (2, -3)])
def test_fourier_decay_periodic_linear_heat(px, qy):
    """Periodic wrap: cos(2 pi (p x + q y)) decays by 1/(1 + tau m0 lambda), lambda = (4/hx^2)
    sin^2(pi p hx) + (4/hy^2) sin^2(pi q hy) — on a non-square grid so hx/hy swaps are caught."""
    m0, dt, nt = 1e-2, 2e-3, 6
    p = W.custom("fper", W.HEAT, W.PERIODIC, 16, 10, nt, dt, m0, 0.0, u0=np.zeros(160))
    Xg, Yg = p.grid()
    p.u0 = np.ascontiguousarray(np.cos(2 * np.pi * (px * Xg + qy * Yg)).reshape(-1))
    lam = (4 / p.hx ** 2) * math.sin(math.pi * px * p.hx) ** 2 + (4 / p.hy ** 2) * math.sin(math.pi * qy * p.hy) ** 2
    r = O.solve_sequential(p)
    for n in range(1, nt + 1):
        assert np.abs(r.U[n - 1] - (1 + dt * m0 * lam) ** (-n) * p.u0).max() < 1e-13


def test_linear_problem_one_newton_iteration():
    """m2 = 0, f = 0: the all-at-once Newton converges in one iteration (the next update is at the
    rounding floor) — Newton is exact on a linear system (SPEC.md:283 states the per-step analogue)."""
    p = W.config(1)
    p.m2 = 0.0
    r = O.solve_allatonce(p, tol=1e-12)
    assert r.status in (0, 1)
    assert r.niter == 2
    assert r.hist[1, 3] < 1e-15


def test_eq15_and_remark4():
    """Eq. (15) gives 22; Remark 4: 2n^2+2n+1 diagonals."""
    assert PF.eq15_max_levels(64, 1e-3, c=1.0, eps=1e-16) == 22
    rng = np.random.default_rng(5)
    A = [PF.five_point_pattern(14, 14, rng) for _ in range(8)]
    P, _ = PF.product_form(A, [np.zeros(196)] * 8)
    for n in range(1, 7):   # 2n < N_x: offsets a + b N_x (|a|+|b| <= n) are distinct (R23)
        assert PF.count_nonzero_diagonals(P[n - 1]) == 2 * n * n + 2 * n + 1
    # beyond 2n >= N_x the offsets alias and the count falls short of the formula
    assert PF.count_nonzero_diagonals(P[7]) < 2 * 8 * 8 + 2 * 8 + 1


def test_fullsize_golden_manifest_integrity():
    """tests/golden/fullsize/ (written by tools/make_fullsize_golden.py from oracle/ only): files match their sha256,
    shapes match the configs, and the stored levels agree with the per-level fingerprints."""
    import hashlib
    import json
    import os
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullsize")
    man = json.load(open(os.path.join(gold, "MANIFEST.json")))
    assert sorted(man) == ["c2", "c3", "c4", "c5"]
    for key, rec in man.items():
        c = int(key[1:])
        p = W.config(c)
        for f, h in ((f"{key}_levels.npy", rec["levels_sha256"]), (f"{key}_stats.npy", rec["stats_sha256"])):
            assert hashlib.sha256(open(os.path.join(gold, f), "rb").read()).hexdigest() == h, f
        lv = np.load(os.path.join(gold, f"{key}_levels.npy"))
        fp = np.load(os.path.join(gold, f"{key}_stats.npy"))
        assert lv.shape == (4, p.ns) and fp.shape == (p.nt, 3)
        assert rec["levels"] == [p.nt // 4, p.nt // 2, 3 * p.nt // 4, p.nt]
        for i, n in enumerate(rec["levels"]):
            assert abs(lv[i].sum() - fp[n - 1, 0]) <= 1e-9 * p.ns
            assert abs(np.abs(lv[i]).max() - fp[n - 1, 2]) == 0.0
        if p.bc == W.PERIODIC:   # exact mass conservation of periodic Burgers at every stored level
            assert np.abs(fp[:, 0] - p.u0.sum()).max() <= 1e-12 * p.ns
