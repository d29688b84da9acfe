"""Design study (not product, not a test): the all-at-once Newton iteration of Eq. (5)-(7) with the per-level
solves done by a FIXED number S of red-black SOR sweeps started from the carry du^{n-1}, in numpy on the
oracle's residual/Jacobian.  Reports Newton iterations, the per-level relative residuals the sweeps leave,
and the distance of the converged U to the sequential oracle — the numbers that size the neighbour-
synchronised level solver of engine 4.

usage: python tools/rb_study.py CFG NT S [omega|auto] [n]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O                      # noqa: E402
from paper_2406_00878_b200 import workloads as W     # noqa: E402


def shifts(p):
    per = p.bc == W.PERIODIC

    def sh(x, dj, di):
        if per:
            return np.roll(np.roll(x, -dj, axis=0), -di, axis=1)
        y = np.zeros_like(x)
        ny, nx = x.shape
        ys, yd = (slice(dj, ny), slice(0, ny - dj)) if dj >= 0 else (slice(0, ny + dj), slice(-dj, ny))
        xs, xd = (slice(di, nx), slice(0, nx - di)) if di >= 0 else (slice(0, nx + di), slice(-di, nx))
        y[yd, xd] = x[ys, xs]
        return y
    return sh


def rb_sweeps(p, co, b, x, S, omega):
    C, E, Wc, N, Sc = (c.reshape(p.nyu, p.nxu) for c in co)
    b = b.reshape(p.nyu, p.nxu)
    x = x.reshape(p.nyu, p.nxu).copy()
    sh = shifts(p)
    jj, ii = np.meshgrid(np.arange(p.nyu), np.arange(p.nxu), indexing="ij")
    red = ((ii + jj) % 2) == 0
    for _ in range(S):
        for mask in (red, ~red):
            off = E * sh(x, 0, 1) + Wc * sh(x, 0, -1) + N * sh(x, 1, 0) + Sc * sh(x, -1, 0)
            xn = (1 - omega) * x + omega * (b - off) / C
            x = np.where(mask, xn, x)
    return x.reshape(-1)


def main():
    c, nt, S = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    om = sys.argv[4] if len(sys.argv) > 4 else "auto"
    n = int(sys.argv[5]) if len(sys.argv) > 5 else None
    p = W.config(c, n=n, nt=nt)
    ns = p.ns
    # Jacobi bound q = max row sum |off| / |diag| at u0, omega from Young's formula
    co0 = O.jacobian(p, p.u0)
    q = float(np.max((np.abs(co0[1]) + np.abs(co0[2]) + np.abs(co0[3]) + np.abs(co0[4])) / np.abs(co0[0])))
    omega = 2 / (1 + np.sqrt(1 - q * q)) if om == "auto" else float(om)
    print(f"{p.name}: q = {q:.4f}  omega = {omega:.5f}  rate(omega-1) = {omega - 1:.4g}")
    U = np.tile(p.u0, (nt, 1))
    t0 = time.time()
    worst = 0.0
    for k in range(30):
        dU = np.zeros_like(U)
        carry = np.zeros(ns)
        rmax = 0.0
        for lv in range(nt):
            um1 = p.u0 if lv == 0 else U[lv - 1]
            r = -O.residual(p, U[lv], um1)
            co = O.jacobian(p, U[lv])
            b = r + carry
            x = rb_sweeps(p, co, b, carry, S, omega)
            res = b - O.matvec(p, co, x)
            nb = np.linalg.norm(b)
            if nb > 1e-300:
                rel = np.linalg.norm(res) / nb
                if np.sqrt(np.mean(res * res)) > 1e-16:
                    rmax = max(rmax, rel)
            dU[lv] = x
            carry = x
        U = U + dU
        d = np.abs(dU).max()
        worst = max(worst, rmax)
        print(f"  k={k}: max|dU| = {d:.3e}  rms dU = {np.sqrt(np.mean(dU * dU)):.3e}  max rel lin res = {rmax:.2e}")
        if d <= 1e-12:
            break
    seq = O.solve_sequential(p)
    err = np.abs(U - seq.U).max() / np.abs(seq.U).max()
    print(f"  iterations {k + 1}, parity vs sequential oracle {err:.2e}, {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
