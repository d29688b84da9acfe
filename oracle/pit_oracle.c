/*
 * pit_oracle.c — the CPU ORACLE for the ParaDIn hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * this library.  The product path (libpit.so, paper_2406_00878_b200/) never links, imports or
 * executes it, and it shares no source, header, table or helper with the CUDA path.
 *
 * Plain, slow, single-threaded C99 in fp64 (build: gcc -O2, no -ffast-math).  Every function cites
 * the passage of /root/reference/PAPER.md it follows ("PAPER.md:L" = line L).
 *
 * What it computes: the fully discrete BDF1 system of Eq. (4),
 * solved the way the paper's sequential baseline does it: level after level, full
 * Newton per level starting from the previous level, each Newton linear system solved
 * by a direct banded solver without pivoting on Dirichlet grids, or by BiCGSTAB with
 * iterative refinement on periodic grids (the banded structure is broken by the wrap; R7).
 * A test-only "all-at-once" mode runs the global Newton of Eq. (5)-(6) with the exact block inverse
 * of Eq. (7) applied as the forward recursion of Theorem 1's proof, from the same
 * initial guess and with the same stop rule as the GPU, so per-iteration histories can be compared.
 *
 * Readings of the paper: face viscosity mu_{i+1/2} = mu((u_i+u_{i+1})/2)
 * (R1), N_x counts intervals (R2), the y-flux of Eq. (3) is g (R4), periodic BC is a wrap (R7).
 *
 * Pins (tests/test_oracle_*.py): Tables 1 and 4, closed-form Fourier
 * decay, manufactured-solution orders, brute-force dense global Newton,
 * finite-difference Jacobian, dense LU, invariants.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

/* ---- problem (mirrors the paper's problem statement, Eqs. (1)-(3)) ---------- */
typedef struct {
    int pde;            /* 0 = nonlinear heat (f = g = 0), 1 = viscous Burgers (f = g = u^2/2) */
    int bc;             /* 0 = Dirichlet (Eq. 2), 1 = periodic (BASELINE extension) */
    int nx, ny;         /* grid INTERVALS N_x, N_y */
    int nt;             /* number of BDF1 levels n = 1..N_t */
    double x0, x1, y0, y1;
    double dt;          /* uniform tau */
    double m0, m2;      /* mu(u) = m0 + m2 u^2 (heat: mu0 u^2; Burgers: mu0) */
} or_prob;

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ENOCONV -4
#define OR_ENOMEM -2

static int or_nxu(const or_prob* p) { return p->bc == 0 ? p->nx - 1 : p->nx; }
static int or_nyu(const or_prob* p) { return p->bc == 0 ? p->ny - 1 : p->ny; }
long or_ns(const or_prob* p) { return (long)or_nxu(p) * (long)or_nyu(p); }
int or_ring_len(const or_prob* p) { return 2 * (p->nx + p->ny); }

/* Eq. (1) laws, PAPER.md:50-52 (generalised mu = m0 + m2 u^2, R6). */
static double or_mu(const or_prob* p, double u) { return p->m0 + p->m2 * u * u; }
static double or_dmu(const or_prob* p, double u) { return 2.0 * p->m2 * u; }
static double or_f(const or_prob* p, double u) { return p->pde == 1 ? 0.5 * u * u : 0.0; }
static double or_df(const or_prob* p, double u) { return p->pde == 1 ? u : 0.0; }

/* Value of the grid function at paper node (i, j) (i along x, j from the bottom
 * boundary j = 0 to the top j = N_y).  Dirichlet: unknowns are the interior nodes, boundary nodes
 * come from the ring b(., ., t^n) (Eq. 2); ring order: bottom j=0 (i=0..nx), top j=ny (i=0..nx),
 * left i=0 (j=1..ny-1), right i=nx (j=1..ny-1); ring == NULL means b = 0.  Periodic: wrap. */
static double or_node(const or_prob* p, const double* u, const double* ring, int i, int j) {
    if (p->bc == 1) {
        int ii = ((i % p->nx) + p->nx) % p->nx, jj = ((j % p->ny) + p->ny) % p->ny;
        return u[(long)jj * p->nx + ii];
    }
    if (i >= 1 && i <= p->nx - 1 && j >= 1 && j <= p->ny - 1)
        return u[(long)(j - 1) * (p->nx - 1) + (i - 1)];
    if (!ring) return 0.0;
    if (j == 0) return ring[i];
    if (j == p->ny) return ring[(p->nx + 1) + i];
    if (i == 0) return ring[2 * (p->nx + 1) + (j - 1)];
    return ring[2 * (p->nx + 1) + (p->ny - 1) + (j - 1)];   /* i == nx */
}

/* is paper node (i, j) an unknown (else a Dirichlet boundary node)? */
static int or_is_unknown(const or_prob* p, int i, int j) {
    if (p->bc == 1) return 1;
    return i >= 1 && i <= p->nx - 1 && j >= 1 && j <= p->ny - 1;
}

/* unknown index of paper node (i, j) (must be an unknown) */
static long or_index(const or_prob* p, int i, int j) {
    if (p->bc == 1) {
        int ii = ((i % p->nx) + p->nx) % p->nx, jj = ((j % p->ny) + p->ny) % p->ny;
        return (long)jj * p->nx + ii;
    }
    return (long)(j - 1) * (p->nx - 1) + (i - 1);
}

/* paper node coordinates of unknown number k */
static void or_unknown_node(const or_prob* p, long k, int* i, int* j) {
    int nxu = or_nxu(p);
    *i = (int)(k % nxu) + (p->bc == 0 ? 1 : 0);
    *j = (int)(k / nxu) + (p->bc == 0 ? 1 : 0);
}

/*
 * G^n(u; u^{n-1}) = tau * [ Eq. (3) left side - right side ] at every unknown,
 * i.e. Eq. (4) multiplied by tau_n:
 *   G = (u_C - uprev_C) + tau [ (f_E - f_W)/(2h_x) + (g_N - g_S)/(2h_y)
 *        - (mu_{i+1/2}(u_E - u_C) - mu_{i-1/2}(u_C - u_W))/h_x^2 - (same in y)/h_y^2 ]
 * with mu_{i+1/2} = mu((u_C + u_E)/2) (R1).  The Newton right-hand side of Eq. (5) is r = -G.
 */
void or_residual(const or_prob* p, const double* u, const double* uprev, const double* ring, double* G) {
    const double hx = (p->x1 - p->x0) / p->nx, hy = (p->y1 - p->y0) / p->ny;
    const long ns = or_ns(p);
    for (long k = 0; k < ns; ++k) {
        int i, j;
        or_unknown_node(p, k, &i, &j);
        double uc = or_node(p, u, ring, i, j);
        double ue = or_node(p, u, ring, i + 1, j), uw = or_node(p, u, ring, i - 1, j);
        double un = or_node(p, u, ring, i, j + 1), us = or_node(p, u, ring, i, j - 1);
        double mE = or_mu(p, 0.5 * (uc + ue)), mW = or_mu(p, 0.5 * (uw + uc));
        double mN = or_mu(p, 0.5 * (uc + un)), mS = or_mu(p, 0.5 * (us + uc));
        double conv = (or_f(p, ue) - or_f(p, uw)) / (2.0 * hx) + (or_f(p, un) - or_f(p, us)) / (2.0 * hy);
        double visc = (mE * (ue - uc) - mW * (uc - uw)) / (hx * hx) + (mN * (un - uc) - mS * (uc - us)) / (hy * hy);
        G[k] = (uc - uprev[k]) + p->dt * (conv - visc);
    }
}

/*
 * Diagonal block A_n = I + tau (dF/du)^n_k of Eq. (6): the exact 5-point derivative of
 * G^n with respect to u^n, including the mu' chain terms (full Newton).  Row k gets
 * coefficients for columns C, E, W, N, S; a column that is a Dirichlet boundary node is dropped (its
 * value is data, part of q in Eq. (4)).  Periodic columns wrap.
 */
void or_jacobian(const or_prob* p, const double* u, const double* ring,
                 double* aC, double* aE, double* aW, double* aN, double* aS) {
    const double hx = (p->x1 - p->x0) / p->nx, hy = (p->y1 - p->y0) / p->ny;
    const double t = p->dt;
    const long ns = or_ns(p);
    for (long k = 0; k < ns; ++k) {
        int i, j;
        or_unknown_node(p, k, &i, &j);
        double uc = or_node(p, u, ring, i, j);
        double ue = or_node(p, u, ring, i + 1, j), uw = or_node(p, u, ring, i - 1, j);
        double un = or_node(p, u, ring, i, j + 1), us = or_node(p, u, ring, i, j - 1);
        double bE = 0.5 * (uc + ue), bW = 0.5 * (uw + uc), bN = 0.5 * (uc + un), bS = 0.5 * (us + uc);
        double mE = or_mu(p, bE), mW = or_mu(p, bW), mN = or_mu(p, bN), mS = or_mu(p, bS);
        double dE = or_dmu(p, bE), dW = or_dmu(p, bW), dN = or_dmu(p, bN), dS = or_dmu(p, bS);
        /* d/du_C of G */
        double c = 1.0 + t * ((mE + mW - 0.5 * dE * (ue - uc) + 0.5 * dW * (uc - uw)) / (hx * hx)
                              + (mN + mS - 0.5 * dN * (un - uc) + 0.5 * dS * (uc - us)) / (hy * hy));
        /* d/du_E: tau [ f'(u_E)/(2hx) - (mu_E + mu'_E/2 (u_E - u_C))/hx^2 ] */
        double e = t * (or_df(p, ue) / (2.0 * hx) - (mE + 0.5 * dE * (ue - uc)) / (hx * hx));
        /* d/du_W: tau [ -f'(u_W)/(2hx) - (mu_W - mu'_W/2 (u_C - u_W))/hx^2 ] */
        double w = t * (-or_df(p, uw) / (2.0 * hx) - (mW - 0.5 * dW * (uc - uw)) / (hx * hx));
        double nn = t * (or_df(p, un) / (2.0 * hy) - (mN + 0.5 * dN * (un - uc)) / (hy * hy));
        double s = t * (-or_df(p, us) / (2.0 * hy) - (mS - 0.5 * dS * (uc - us)) / (hy * hy));
        aC[k] = c;
        aE[k] = or_is_unknown(p, i + 1, j) ? e : 0.0;
        aW[k] = or_is_unknown(p, i - 1, j) ? w : 0.0;
        aN[k] = or_is_unknown(p, i, j + 1) ? nn : 0.0;
        aS[k] = or_is_unknown(p, i, j - 1) ? s : 0.0;
    }
}

/* y = A x for the 5-coefficient operator above (dropped columns are zero coefficients). */
void or_matvec(const or_prob* p, const double* aC, const double* aE, const double* aW, const double* aN,
               const double* aS, const double* x, double* y) {
    const long ns = or_ns(p);
    for (long k = 0; k < ns; ++k) {
        int i, j;
        or_unknown_node(p, k, &i, &j);
        double acc = aC[k] * x[k];
        if (or_is_unknown(p, i + 1, j)) acc += aE[k] * x[or_index(p, i + 1, j)];
        if (or_is_unknown(p, i - 1, j)) acc += aW[k] * x[or_index(p, i - 1, j)];
        if (or_is_unknown(p, i, j + 1)) acc += aN[k] * x[or_index(p, i, j + 1)];
        if (or_is_unknown(p, i, j - 1)) acc += aS[k] * x[or_index(p, i, j - 1)];
        y[k] = acc;
    }
}

/*
 * "standard direct solver for banded matrices without pivoting".  Dirichlet only:
 * with x-fastest numbering the 5-point matrix has lower and upper bandwidth bw = nx-1 (the N/S
 * columns).  Doolittle LU without pivoting on a dense band store, then forward/back substitution.
 */
int or_band_lu_solve(const or_prob* p, const double* aC, const double* aE, const double* aW,
                     const double* aN, const double* aS, const double* b, double* x) {
    if (p->bc != 0) return OR_EINVAL;
    const long n = or_ns(p);
    const long bw = or_nxu(p);
    const long w = 2 * bw + 1;
    double* a = (double*)calloc((size_t)(n * w), sizeof(double));
    if (!a) return OR_ENOMEM;
#define BAND(r, c) a[(r) * w + ((c) - (r) + bw)]
    for (long k = 0; k < n; ++k) {
        int i, j;
        or_unknown_node(p, k, &i, &j);
        BAND(k, k) = aC[k];
        if (or_is_unknown(p, i + 1, j)) BAND(k, or_index(p, i + 1, j)) += aE[k];
        if (or_is_unknown(p, i - 1, j)) BAND(k, or_index(p, i - 1, j)) += aW[k];
        if (or_is_unknown(p, i, j + 1)) BAND(k, or_index(p, i, j + 1)) += aN[k];
        if (or_is_unknown(p, i, j - 1)) BAND(k, or_index(p, i, j - 1)) += aS[k];
    }
    for (long k = 0; k < n; ++k) {
        double piv = BAND(k, k);
        long iend = k + bw < n - 1 ? k + bw : n - 1;
        for (long i = k + 1; i <= iend; ++i) {
            double l = BAND(i, k) / piv;
            BAND(i, k) = l;
            if (l == 0.0) continue;
            for (long j = k + 1; j <= iend; ++j) BAND(i, j) -= l * BAND(k, j);
        }
    }
    for (long i = 0; i < n; ++i) {               /* L y = b (unit lower) */
        double s = b[i];
        long j0 = i - bw > 0 ? i - bw : 0;
        for (long j = j0; j < i; ++j) s -= BAND(i, j) * x[j];
        x[i] = s;
    }
    for (long i = n - 1; i >= 0; --i) {          /* U x = y */
        double s = x[i];
        long j1 = i + bw < n - 1 ? i + bw : n - 1;
        for (long j = i + 1; j <= j1; ++j) s -= BAND(i, j) * x[j];
        x[i] = s / BAND(i, i);
    }
#undef BAND
    free(a);
    return OR_OK;
}

static double or_dot(long n, const double* a, const double* b) {
    double s = 0.0;
    for (long k = 0; k < n; ++k) s += a[k] * b[k];
    return s;
}

/*
 * BiCGSTAB (van der Vorst 1992), right-preconditioned with M = diag(A), for the periodic grids where
 * the wrap breaks the banded structure.  Wrapped in iterative refinement on the TRUE residual so the
 * returned x satisfies ||b - A x||_2 <= rtol ||b||_2 (or the best reachable at the rounding floor).
 * Returns the total number of inner iterations (>= 0) or a negative error.
 */
int or_bicgstab_solve(const or_prob* p, const double* aC, const double* aE, const double* aW,
                      const double* aN, const double* aS, const double* b, double* x, double rtol, int maxit) {
    const long n = or_ns(p);
    double* buf = (double*)calloc((size_t)(10 * n), sizeof(double));
    if (!buf) return OR_ENOMEM;
    double *r = buf, *rh = buf + n, *pp = buf + 2 * n, *v = buf + 3 * n, *s = buf + 4 * n, *t = buf + 5 * n;
    double *ph = buf + 6 * n, *sh = buf + 7 * n, *d = buf + 8 * n, *rt = buf + 9 * n;
    const double bnorm = sqrt(or_dot(n, b, b));
    int total = 0;
    memset(x, 0, sizeof(double) * (size_t)n);
    if (bnorm == 0.0) { free(buf); return 0; }
    double best = INFINITY;
    for (int refine = 0; refine < 8; ++refine) {
        /* true residual */
        or_matvec(p, aC, aE, aW, aN, aS, x, rt);
        for (long k = 0; k < n; ++k) rt[k] = b[k] - rt[k];
        double rn = sqrt(or_dot(n, rt, rt));
        if (rn <= rtol * bnorm) break;
        if (rn >= 0.5 * best) break;            /* refinement no longer improves: rounding floor */
        best = rn;
        /* inner BiCGSTAB on A d = rt */
        memset(d, 0, sizeof(double) * (size_t)n);
        memcpy(r, rt, sizeof(double) * (size_t)n);
        memcpy(rh, rt, sizeof(double) * (size_t)n);
        memset(pp, 0, sizeof(double) * (size_t)n);
        memset(v, 0, sizeof(double) * (size_t)n);
        double rho = 1.0, alpha = 1.0, omega = 1.0;
        const double target = fmax(1e-10 * rn, 0.1 * rtol * bnorm);   /* each pass gains ~1e-10 */
        for (int it = 0; it < maxit; ++it) {
            double rho1 = or_dot(n, rh, r);
            if (rho1 == 0.0) break;
            double beta = (rho1 / rho) * (alpha / omega);
            for (long k = 0; k < n; ++k) pp[k] = r[k] + beta * (pp[k] - omega * v[k]);
            for (long k = 0; k < n; ++k) ph[k] = pp[k] / aC[k];
            or_matvec(p, aC, aE, aW, aN, aS, ph, v);
            double rv = or_dot(n, rh, v);
            if (rv == 0.0) break;
            alpha = rho1 / rv;
            for (long k = 0; k < n; ++k) s[k] = r[k] - alpha * v[k];
            ++total;
            double sn = sqrt(or_dot(n, s, s));
            if (sn <= target) {
                for (long k = 0; k < n; ++k) d[k] += alpha * ph[k];
                break;
            }
            for (long k = 0; k < n; ++k) sh[k] = s[k] / aC[k];
            or_matvec(p, aC, aE, aW, aN, aS, sh, t);
            double tt = or_dot(n, t, t);
            omega = tt > 0.0 ? or_dot(n, t, s) / tt : 0.0;
            for (long k = 0; k < n; ++k) d[k] += alpha * ph[k] + omega * sh[k];
            for (long k = 0; k < n; ++k) r[k] = s[k] - omega * t[k];
            rho = rho1;
            if (sqrt(or_dot(n, r, r)) <= target || omega == 0.0) break;
        }
        for (long k = 0; k < n; ++k) x[k] += d[k];
    }
    free(buf);
    return total;
}

/* One linear solve with the diagonal block: banded LU on Dirichlet grids (the paper's solver,
 * PAPER.md:342), BiCGSTAB + refinement on periodic grids. */
static int or_linear_solve(const or_prob* p, const double* aC, const double* aE, const double* aW,
                           const double* aN, const double* aS, const double* b, double* x) {
    if (p->bc == 0) return or_band_lu_solve(p, aC, aE, aW, aN, aS, b, x);
    int it = or_bicgstab_solve(p, aC, aE, aW, aN, aS, b, x, 1e-15, 4000);
    return it < 0 ? it : OR_OK;
}

static double or_maxabs(long n, const double* a) {
    double m = 0.0;
    for (long k = 0; k < n; ++k) { double v = fabs(a[k]); if (v > m) m = v; }
    return m;
}

/*
 * Sequential BDF1 time marching with Newton at every step (cost model PAPER.md:292-295):
 * for n = 1..N_t, start from u^{n-1}, solve A delta = -G, u += delta, until
 * ||delta||_inf <= 1e-14 max(1, ||u||_inf) (or stagnation at the rounding floor).
 *   u0:   N_s initial data at the unknown nodes;  bc: nt * ring_len Dirichlet rings at t^n (or NULL)
 *   levels: levels to compute (<= nt; a bounded prefix is a valid sample by causality, Eq. 6 is
 *           block lower triangular);  U: levels * N_s output;  iters: per-level Newton counts (or NULL)
 * Returns OR_OK, or OR_ENOCONV if some level needed more than 50 iterations.
 */
int or_solve_sequential(const or_prob* p, const double* u0, const double* bc, int levels,
                        double* U, int* iters, double* last_delta) {
    const long n = or_ns(p);
    const int rl = or_ring_len(p);
    if (levels > p->nt || levels < 0) return OR_EINVAL;
    double* w = (double*)malloc(sizeof(double) * (size_t)(7 * n));
    if (!w) return OR_ENOMEM;
    double *G = w, *aC = w + n, *aE = w + 2 * n, *aW = w + 3 * n, *aN = w + 4 * n, *aS = w + 5 * n, *dl = w + 6 * n;
    int status = OR_OK;
    for (int lv = 1; lv <= levels; ++lv) {
        const double* uprev = lv == 1 ? u0 : U + (long)(lv - 2) * n;
        double* u = U + (long)(lv - 1) * n;
        const double* ring = (p->bc == 0 && bc) ? bc + (long)(lv - 1) * rl : NULL;
        memcpy(u, uprev, sizeof(double) * (size_t)n);
        double prev = INFINITY, dn = 0.0;
        int k;
        for (k = 0; k < 50; ++k) {
            or_residual(p, u, uprev, ring, G);
            or_jacobian(p, u, ring, aC, aE, aW, aN, aS);
            for (long q = 0; q < n; ++q) G[q] = -G[q];
            int rc = or_linear_solve(p, aC, aE, aW, aN, aS, G, dl);
            if (rc < 0) { free(w); return rc; }
            for (long q = 0; q < n; ++q) u[q] += dl[q];
            dn = or_maxabs(n, dl);
            double scale = fmax(1.0, or_maxabs(n, u));
            if (dn <= 1e-14 * scale) break;
            if (k >= 2 && dn >= 0.5 * prev && dn <= 1e-11 * scale) break;   /* rounding floor */
            prev = dn;
        }
        if (k == 50) status = OR_ENOCONV;
        if (iters) iters[lv - 1] = k + 1;
        if (last_delta) last_delta[lv - 1] = dn;
    }
    free(w);
    return status;
}

/*
 * Test-only ALL-AT-ONCE mode: the global Newton of Eq. (5) for all levels simultaneously
 * with the block-bidiagonal Jacobian of Eq. (6) inverted exactly by the forward
 * recursion  Delta u^n = A_n^{-1} (r^n + Delta u^{n-1})  that Theorem 1's proof performs
 * (Eq. 7 row by row).  Same initial guess (guess or u0 at every level) and the
 * same stop rule as the GPU driver:
 *   converged      if max|dU_k| <= tol                                           -> status 0
 *   floor          if k >= 1, max|dU_k| > max|dU_{k-1}|/2 and max|dU_k| <= 1e3 tol -> status 1
 *   no convergence at k + 1 == newton_max                                        -> status -4
 * hist[k*4 + {0,1,2,3}] = { rms R(U_k), max|R(U_k)|, rms dU_k, max|dU_k| }.
 * U (nt * N_s) receives the final iterate U_{k+1}.  *niter = iterations performed.
 */
int or_solve_allatonce(const or_prob* p, const double* u0, const double* bc, const double* guess,
                       double tol, int newton_max, double* U, double* hist, int* niter) {
    const long n = or_ns(p);
    const long N = n * p->nt;
    const int rl = or_ring_len(p);
    double* R = (double*)malloc(sizeof(double) * (size_t)N);
    double* w = (double*)malloc(sizeof(double) * (size_t)(7 * n));
    if (!R || !w) { free(R); free(w); return OR_ENOMEM; }
    double *aC = w, *aE = w + n, *aW = w + 2 * n, *aN = w + 3 * n, *aS = w + 4 * n, *b = w + 5 * n, *dl = w + 6 * n;
    for (int lv = 0; lv < p->nt; ++lv)
        memcpy(U + (long)lv * n, guess ? guess + (long)lv * n : u0, sizeof(double) * (size_t)n);
    int status = OR_ENOCONV;
    double prevmax = INFINITY;
    int k;
    for (k = 0; k < newton_max; ++k) {
        /* residuals at U_k for all levels (they use U_k^{n-1}, so form them before any update) */
        double rs = 0.0, rm = 0.0;
        for (int lv = 1; lv <= p->nt; ++lv) {
            const double* ring = (p->bc == 0 && bc) ? bc + (long)(lv - 1) * rl : NULL;
            const double* uprev = lv == 1 ? u0 : U + (long)(lv - 2) * n;
            double* Rl = R + (long)(lv - 1) * n;
            or_residual(p, U + (long)(lv - 1) * n, uprev, ring, Rl);
            for (long q = 0; q < n; ++q) { Rl[q] = -Rl[q]; rs += Rl[q] * Rl[q]; if (fabs(Rl[q]) > rm) rm = fabs(Rl[q]); }
        }
        /* Jacobian blocks at U_k, then the forward recursion; update after all solves */
        double ds = 0.0, dm = 0.0;
        memset(dl, 0, sizeof(double) * (size_t)n);
        for (int lv = 1; lv <= p->nt; ++lv) {
            const double* ring = (p->bc == 0 && bc) ? bc + (long)(lv - 1) * rl : NULL;
            or_jacobian(p, U + (long)(lv - 1) * n, ring, aC, aE, aW, aN, aS);
            const double* Rl = R + (long)(lv - 1) * n;
            for (long q = 0; q < n; ++q) b[q] = Rl[q] + dl[q];           /* r^n + Delta u^{n-1} */
            int rc = or_linear_solve(p, aC, aE, aW, aN, aS, b, dl);
            if (rc < 0) { free(R); free(w); return rc; }
            double* Rw = R + (long)(lv - 1) * n;                          /* reuse R storage for Delta */
            memcpy(Rw, dl, sizeof(double) * (size_t)n);
            for (long q = 0; q < n; ++q) { ds += dl[q] * dl[q]; if (fabs(dl[q]) > dm) dm = fabs(dl[q]); }
        }
        for (long q = 0; q < N; ++q) U[q] += R[q];
        if (hist) {
            hist[4 * k + 0] = sqrt(rs / (double)N);
            hist[4 * k + 1] = rm;
            hist[4 * k + 2] = sqrt(ds / (double)N);
            hist[4 * k + 3] = dm;
        }
        if (dm <= tol) { status = OR_OK; ++k; break; }
        if (k >= 1 && dm > 0.5 * prevmax && dm <= 1e3 * tol) { status = 1; ++k; break; }
        prevmax = dm;
    }
    if (niter) *niter = k;
    free(R); free(w);
    return status;
}

/*
 * Test-only: ONE all-at-once Newton iteration (Eq. (5)-(7)) over a SLAB of levels 1..nt (p->nt)
 * whose preceding level is u_prev (U_k at the level before the slab; u^0 for the first slab) and whose incoming
 * carry is carry_in (Delta u_k at that level; NULL = 0 for the first slab).  The forward recursion of Eq. (7) then
 * starts from carry_in instead of 0,  Delta u^1 = A_1^{-1} (r^1 + carry_in)  — the exact continuation of the
 * recursion across a slab boundary, which is what the multi-GPU time-slab pipeline runs.
 * Outputs U_{k+1} = U_k + Delta U (Uk1), carry_out = Delta u^{nt} (may be NULL) and
 * sums[4] = { sum R(U_k)^2, max|R(U_k)|, sum dU^2, max|dU| } over the slab.
 */
int or_allatonce_iteration(const or_prob* p, const double* u_prev, const double* carry_in, const double* bc,
                           const double* Uk, double* Uk1, double* carry_out, double* sums) {
    const long n = or_ns(p);
    const int rl = or_ring_len(p);
    double* w = (double*)malloc(sizeof(double) * (size_t)(8 * n));
    if (!w) return OR_ENOMEM;
    double *aC = w, *aE = w + n, *aW = w + 2 * n, *aN = w + 3 * n, *aS = w + 4 * n, *b = w + 5 * n, *dl = w + 6 * n;
    double* Rl = w + 7 * n;
    double rs = 0.0, rm = 0.0, ds = 0.0, dm = 0.0;
    if (carry_in) memcpy(dl, carry_in, sizeof(double) * (size_t)n);
    else memset(dl, 0, sizeof(double) * (size_t)n);
    for (int lv = 1; lv <= p->nt; ++lv) {
        const double* ring = (p->bc == 0 && bc) ? bc + (long)(lv - 1) * rl : NULL;
        const double* ul = Uk + (long)(lv - 1) * n;
        or_residual(p, ul, lv == 1 ? u_prev : Uk + (long)(lv - 2) * n, ring, Rl);
        or_jacobian(p, ul, ring, aC, aE, aW, aN, aS);
        for (long q = 0; q < n; ++q) {
            Rl[q] = -Rl[q];
            rs += Rl[q] * Rl[q];
            if (fabs(Rl[q]) > rm) rm = fabs(Rl[q]);
            b[q] = Rl[q] + dl[q];                                          /* r^n + Delta u^{n-1} */
        }
        int rc = or_linear_solve(p, aC, aE, aW, aN, aS, b, dl);
        if (rc < 0) { free(w); return rc; }
        for (long q = 0; q < n; ++q) {
            Uk1[(long)(lv - 1) * n + q] = ul[q] + dl[q];
            ds += dl[q] * dl[q];
            if (fabs(dl[q]) > dm) dm = fabs(dl[q]);
        }
    }
    if (carry_out) memcpy(carry_out, dl, sizeof(double) * (size_t)n);
    sums[0] = rs; sums[1] = rm; sums[2] = ds; sums[3] = dm;
    free(w);
    return OR_OK;
}

/* Space-time residual of a given U (all levels): R = -G^n(U^n; U^{n-1}), used by the full-size
 * parity tests to check a GPU solution against the discrete equations of Eq. (4). */
void or_spacetime_residual(const or_prob* p, const double* u0, const double* bc, const double* U, double* R) {
    const long n = or_ns(p);
    const int rl = or_ring_len(p);
    for (int lv = 1; lv <= p->nt; ++lv) {
        const double* ring = (p->bc == 0 && bc) ? bc + (long)(lv - 1) * rl : NULL;
        const double* uprev = lv == 1 ? u0 : U + (long)(lv - 2) * n;
        double* Rl = R + (long)(lv - 1) * n;
        or_residual(p, U + (long)(lv - 1) * n, uprev, ring, Rl);
        for (long q = 0; q < n; ++q) Rl[q] = -Rl[q];
    }
}
