"""CPU ORACLE of the paper's all-at-once initial guess — TEST INFRASTRUCTURE ONLY
(imported by tests/, never by the product package; it does not import the product package either).

PAPER.md:214 (Section 4): "we initialize the solution by solving Eq. (FDS) sequentially on a coarse grid and
interpolating this coarse-grid-solution to the original fine mesh by using a 1-D cubic spline along each
spatial coordinate.  Note that the original grid is coarsened in both each spatial direction and time by the
same factor c_f."  c_f = 4 for heat and 3 for Burgers.

Readings (R21-R24): coarse node (ic, jc, m) is fine node (c_f ic, c_f jc) at fine level c_f m
(injection of u^0 and of the Dirichlet ring); splines are the C^2 cubic interpolants with not-a-knot end
conditions along Dirichlet directions and in time, periodic along periodic directions; the interpolation is
applied along x, then y (at every coarse level m >= 1, on coarse NODES, boundary values from the ring), then
along t with the fine u^0 as the t = 0 knot.

Every step is written out plainly: the spline's second-derivative system is formed as a dense matrix and
solved with numpy.linalg.solve (a library primitive), then the piecewise cubic is evaluated by its textbook
formula.  Pinned in tests/test_oracle_coarse.py (scipy's independent CubicSpline, exact reproduction of
linear data, knot interpolation, and the paper's Newton iteration counts of Tables 3 and 6).
"""
from __future__ import annotations

import types

import numpy as np

from . import oracle as O


# ---- 1-D cubic spline on uniform knots (any knot spacing H: written with m = M H^2 / 6) -----------

def spline_moments(F: np.ndarray, periodic: bool, end: str = "notaknot") -> np.ndarray:
    """Scaled second derivatives m_k = M_k H^2 / 6 of the cubic spline through knots F[k] (axis 0; other
    axes are independent lines).  C^2 continuity at an interior knot of a uniform grid reads
        M_{k-1} + 4 M_k + M_{k+1} = (6 / H^2) (F_{k+1} - 2 F_k + F_{k-1}),
    i.e. m_{k-1} + 4 m_k + m_{k+1} = F_{k+1} - 2 F_k + F_{k-1}.
    Periodic (K knots, period K H): the same equation at every k with indices mod K.
    Otherwise the end conditions (R22) are "notaknot" (S''' continuous at knots 1 and K-2:
    m_0 - 2 m_1 + m_2 = 0, m_{K-3} - 2 m_{K-2} + m_{K-1} = 0; K = 3 gives the interpolating parabola,
    K = 2 the line) or "natural" (m_0 = m_{K-1} = 0)."""
    F = np.asarray(F, dtype=np.float64)
    K = F.shape[0]
    A = np.zeros((K, K))
    rhs = np.zeros_like(F)
    if periodic:
        for k in range(K):
            A[k, (k - 1) % K] += 1.0
            A[k, k] += 4.0
            A[k, (k + 1) % K] += 1.0
            rhs[k] = F[(k + 1) % K] - 2.0 * F[k] + F[(k - 1) % K]
    else:
        for k in range(1, K - 1):
            A[k, k - 1] = 1.0
            A[k, k] = 4.0
            A[k, k + 1] = 1.0
            rhs[k] = F[k + 1] - 2.0 * F[k] + F[k - 1]
        if end == "natural" or K == 2:
            A[0, 0] = 1.0
            A[K - 1, K - 1] = 1.0
        elif K == 3:
            A[0, 0], A[0, 1] = 1.0, -1.0
            A[2, 1], A[2, 2] = -1.0, 1.0
        else:
            A[0, 0], A[0, 1], A[0, 2] = 1.0, -2.0, 1.0
            A[K - 1, K - 3], A[K - 1, K - 2], A[K - 1, K - 1] = 1.0, -2.0, 1.0
    return np.linalg.solve(A, rhs.reshape(K, -1)).reshape(F.shape)


def spline_eval(F: np.ndarray, m: np.ndarray, cf: int, positions, periodic: bool) -> np.ndarray:
    """Value of the spline at fine positions p (knot k sits at p = cf k): k = p // cf, theta = (p mod cf)/cf,
        S = (1 - theta) F_k + theta F_{k+1} + ((1 - theta)^3 - (1 - theta)) m_k + (theta^3 - theta) m_{k+1}."""
    K = F.shape[0]
    out = []
    for p in positions:
        k, r = divmod(int(p), cf)
        th = r / cf
        if r == 0:
            out.append(F[k % K] if periodic else F[k])
            continue
        k1 = (k + 1) % K if periodic else k + 1
        out.append((1.0 - th) * F[k] + th * F[k1] + ((1.0 - th) ** 3 - (1.0 - th)) * m[k] + (th ** 3 - th) * m[k1])
    return np.stack(out)


def spline_refine(F: np.ndarray, cf: int, positions, periodic: bool, end: str = "notaknot") -> np.ndarray:
    return spline_eval(F, spline_moments(F, periodic, end), cf, positions, periodic)


# ---- grids: unknowns <-> nodes, injection to the coarse grid --------------------------------------

def _nodes(p, u: np.ndarray, ring_level) -> np.ndarray:
    """Node field of one level: Dirichlet (ny+1, nx+1) with the ring (Eq. 2, ABI ring order: bottom j=0,
    top j=ny, left i=0, right i=nx); periodic (ny, nx) = the unknowns."""
    nxu, nyu = (p.nx - 1, p.ny - 1) if p.bc == 0 else (p.nx, p.ny)
    u = np.asarray(u).reshape(nyu, nxu)
    if p.bc == 1:
        return u.copy()
    Nf = np.zeros((p.ny + 1, p.nx + 1))
    Nf[1:p.ny, 1:p.nx] = u
    if ring_level is not None:
        r = np.asarray(ring_level)
        nx, ny = p.nx, p.ny
        Nf[0, :] = r[0:nx + 1]
        Nf[ny, :] = r[nx + 1:2 * nx + 2]
        Nf[1:ny, 0] = r[2 * nx + 2:2 * nx + 2 + ny - 1]
        Nf[1:ny, nx] = r[2 * nx + 2 + ny - 1:2 * nx + 2 + 2 * (ny - 1)]
    return Nf


def _unknowns(p, Nf: np.ndarray) -> np.ndarray:
    return (Nf[1:p.ny, 1:p.nx] if p.bc == 0 else Nf).reshape(-1).copy()


def coarse_problem(p, cf: int):
    """The c_f-coarsened problem: N_x / c_f, N_y / c_f intervals, N_t / c_f levels of step
    c_f dt; u^0 and the Dirichlet ring injected at the coarse nodes (fine node c_f i, level c_f m)."""
    if p.nx % cf or p.ny % cf or p.nt % cf:
        raise ValueError("c_f must divide N_x, N_y and N_t")
    nxc, nyc, ntc = p.nx // cf, p.ny // cf, p.nt // cf
    if (p.bc == 0 and min(nxc, nyc) < 2) or (p.bc == 1 and min(nxc, nyc) < 3):
        raise ValueError("coarse grid too small")
    pc = types.SimpleNamespace(pde=p.pde, bc=p.bc, nx=nxc, ny=nyc, nt=ntc, x0=p.x0, x1=p.x1, y0=p.y0, y1=p.y1,
                               dt=p.dt * cf, m0=p.m0, m2=p.m2, newton_tol=p.newton_tol)
    N0 = _nodes(p, p.u0, None)
    pc.u0 = _unknowns(pc, N0[::cf, ::cf])
    if p.bc == 0 and p.ring is not None:
        ring = np.empty((ntc, 2 * (nxc + nyc)))
        for m in range(1, ntc + 1):
            Nm = _nodes(p, np.zeros(((p.ny - 1) * (p.nx - 1),)), p.ring[cf * m - 1])[::cf, ::cf]
            ring[m - 1] = np.concatenate([Nm[0, :], Nm[nyc, :], Nm[1:nyc, 0], Nm[1:nyc, nxc]])
        pc.ring = ring
    else:
        pc.ring = None
    return pc


def coarse_guess(p, cf: int, coarse_U: np.ndarray | None = None, end: str = "notaknot") -> np.ndarray:
    """Initial iterate U_0 (nt, ns) of the all-at-once Newton iteration: sequential BDF1 on the coarse grid
    (the oracle's sequential solver), then cubic splines along x, y (coarse levels m = 1..N_t/c_f), then t."""
    pc = coarse_problem(p, cf)
    Uc = O.solve_sequential(pc).U if coarse_U is None else np.asarray(coarse_U).reshape(pc.nt, -1)
    per = p.bc == 1
    npx = p.nx if per else p.nx + 1          # fine node positions along x / y
    npy = p.ny if per else p.ny + 1
    knots = [np.asarray(p.u0, dtype=np.float64).reshape(-1)]
    for m in range(1, pc.nt + 1):
        Nc = _nodes(pc, Uc[m - 1], None if pc.ring is None else pc.ring[m - 1])
        Tx = spline_refine(Nc.T, cf, range(npx), per, end).T          # x: along axis 1 of (rows, cols)
        Nf = spline_refine(Tx, cf, range(npy), per, end)              # y: along axis 0
        knots.append(_unknowns(p, Nf))
    Fk = np.stack(knots)                                          # (ntc + 1, ns), knot m at t = m c_f dt
    return spline_refine(Fk, cf, range(1, p.nt + 1), False, end)  # levels n = 1..nt
