/*
 * pit.h — C ABI of libpit: the all-at-once (parallel-in-time) Newton iteration for the implicit
 * BDF1 discretization of 2-D nonlinear heat / viscous Burgers equations ("ParaDIn",
 * arXiv 2406.00878), hand-written CUDA for sm_100a (B200), fp64 throughout.
 *
 * Citations: "PAPER.md:L" = line L of the paper's LaTeX source (/root/reference/PAPER.md at build
 * time; the text is not needed at run time).
 *
 * What a solve computes (Eqs. (4)-(6)): the space-time solution U = [u^1 .. u^Nt]
 * of
 *     (u^n - u^{n-1})/tau + F(u^n) = q^n,   n = 1..Nt                             (Eq. 4)
 * where F is the 5-point discretization of Eq. (3) of
 *     u_t + f(u)_x + g(u)_y = (mu(u) u_x)_x + (mu(u) u_y)_y                       (Eq. 1)
 * with f = g = u^2/2 (Burgers) or 0 (heat), mu(u) = m0 + m2 u^2, face viscosity
 * mu_{i+1/2} = mu((u_i + u_{i+1})/2), and Dirichlet (Eq. 2) or periodic boundaries.  It is solved by
 * Newton's method for ALL levels at once (Eq. 5): every iteration forms the space-time residual and
 * the block-bidiagonal Jacobian of Eq. (6) (kernel a), applies its exact blockwise inverse Eq. (7)
 * (stage b: on-device level recurrence, or the literal Theorem 1 product form inside the paper's
 * Section 7 conditioning window), solves the per-level 5-point systems (stage c: fixed-sweep
 * red-black SOR in the default engines 4 and 5, Jacobi-scaled BiCGSTAB in engines 1-3) and updates
 * U, with convergence checked on the device (stage d).
 *
 * Conventions
 *   Layout: fp64, row-major [n][j][i], i (x) fastest.  Level n = 1..nt is stored
 *           at index n-1; u^0 is an input, not an unknown.
 *   Grid:   nx, ny count grid INTERVALS.  Unknowns per level:
 *           Dirichlet (nx-1)*(ny-1) at the interior nodes; periodic nx*ny.
 *   Dirichlet ring (per level, at t^n = n*dt): bottom j=0 (i=0..nx), top j=ny (i=0..nx),
 *           left i=0 (j=1..ny-1), right i=nx (j=1..ny-1): 2*(nx+ny) values.
 *   Ownership: the caller owns every buffer passed in; the library never keeps a caller pointer past
 *           the return of pit_solve, or past completion of the stream work of pit_*_device.
 *           The handle owns all internal device memory (pit_destroy frees it).
 *   Threading: a handle is not thread-safe (one solve at a time); distinct handles are independent.
 *   Errors: every entry point returns a pit_status; negative = error.  pit_last_error(h) gives
 *           detail.  No CPU fallback exists: without a usable sm_100 device pit_create fails with
 *           PIT_ECUDA.
 *   Determinism: identical inputs and configuration on the same GPU give bit-identical outputs
 *           (fixed-order reductions, no floating-point atomics).
 *   Debug environment (developer instrumentation and A/B switches used for the measurements in DESIGN.md; read
 *           once per handle at pit_create; none is needed for correct results, the defaults are the product path):
 *             PIT_TRACE=1        cycle accounting of the persistent kernels (pit_stats, pit_engine_info)
 *             PIT_RESJAC_V1=1    kernel (a) without TMA staging;  PIT_RESJAC_RT / PIT_RESJAC_NS  its tile rows / stages
 *             PIT_X0=0           engines 2-3 start each level solve from 0 instead of the carry du^{n-1}
 *             PIT_MERGE=0        engine 3 without the merged first BiCGSTAB iteration
 *             PIT_GUESS_GRAPH=0  the coarse-grid guess's level march without a CUDA graph
 *             PIT_PS_DBG         engine 5 experiments (with PIT_TRACE=1, the developer build of its kernels): bit 0 = neighbour cells
 *                                are not waited for, bit 1 = no fence before the level counters (both WRONG results, timing only);
 *                                bit 2 = one row group of 256 threads per CTA on 512-wide rows
 *           All NVTX ranges ("pit_solve_device", "pit_solve", ...) are emitted unconditionally (free without a tool).
 */
#ifndef PIT_H
#define PIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIT_ABI_VERSION 3

typedef enum {
    PIT_OK = 0,           /* converged: max|dU_k| <= newton_tol */
    PIT_OK_FLOOR = 1,     /* converged at the rounding floor (stop rule (2) below) */
    PIT_EINVAL = -1,      /* invalid argument / configuration / ABI mismatch */
    PIT_ENOMEM = -2,      /* device allocation failed */
    PIT_ECUDA = -3,       /* CUDA error or no usable sm_100 device (detail: pit_last_error) */
    PIT_ENOCONV = -4,     /* newton_max reached; outputs hold the last iterate and the histories */
    PIT_EBREAKDOWN = -5,  /* Krylov breakdown or NaN/Inf detected on the device */
    PIT_ECOND = -6        /* product-form window forced beyond the Section 7 conditioning gate */
} pit_status;

enum { PIT_HEAT = 0, PIT_BURGERS = 1 };
enum { PIT_DIRICHLET = 0, PIT_PERIODIC = 1 };           /* Eq. (2); periodic = extension */
/* Inversion of the block-bidiagonal Newton matrix of Eq. (6): AUTO, the on-device level recurrence of Eq. (7)
 * (default fast path), the Theorem 1 product form with nested level solves inside the Section 7 gate (b2), or
 * the paper's explicit form — banded P^n by Eq. (10), diag(P^n) scaling, banded LU without
 * pivoting; Dirichlet only, no gate; window = 0 means the whole horizon (N3) */
/* AUTO = the level recurrence (asynchronous on the stream for every engine); the product forms are chosen
 * explicitly (their window gate and Newton loop are driven from the host: one stream synchronization per Newton
 * iteration and per gate check — DESIGN.md R19). */
enum { PIT_INV_AUTO = 0, PIT_INV_RECURRENCE = 1, PIT_INV_PRODUCT_WINDOW = 2, PIT_INV_EXPLICIT = 3 };

typedef struct {
    int32_t abi_version;   /* must equal PIT_ABI_VERSION */
    int32_t pde;           /* PIT_HEAT (f = g = 0) | PIT_BURGERS (f = g = u^2/2) */
    int32_t bc;            /* PIT_DIRICHLET | PIT_PERIODIC */
    int32_t nx, ny;        /* grid intervals; Dirichlet >= 2, periodic >= 3 */
    int32_t nt;            /* BDF1 levels, >= 1 */
    double  x0, x1, y0, y1;/* domain [x0,x1] x [y0,y1]; h_x = (x1-x0)/nx */
    double  dt;            /* uniform time step tau > 0 */
    double  m0, m2;        /* mu(u) = m0 + m2 u^2, m0, m2 >= 0 (paper heat: 0, mu0; Burgers: mu0, 0) */
    double  newton_tol;    /* stop on ||dU_k|| <= newton_tol (> 0; BASELINE: 1e-12), norm chosen by stop_norm */
    int32_t newton_max;    /* max Newton iterations (1..256) */
    double  lin_rtol;      /* per-level solve: ||b~ - A~ x||_2 <= lin_rtol ||b~||_2 (A~ = diag-scaled A_n);
                              0 = default 1e-6 (an inexact-Newton forcing term:
                              the Newton iteration counts of BASELINE c1-c5 are those of exact solves, DESIGN R10) */
    double  lin_atol;      /* ... or RMS(b~ - A~ x) = ||.||_2 / sqrt(ns) <= lin_atol; 0 = default 1e-4 * newton_tol */
    int32_t lin_max;       /* per-level BiCGSTAB iteration cap; 0 = default 1000 */
    int32_t inverse_mode;  /* PIT_INV_*; AUTO = the level recurrence */
    int32_t window;        /* product-form window length; 0 = auto from the Section 7 gate (PRODUCT_WINDOW) or
                              the whole horizon (EXPLICIT) */
    int32_t pipeline_depth;/* Newton iterations in flight in the level wavefront; 0 = auto */
    int32_t device;        /* CUDA device ordinal */
    int32_t engine;        /* Newton-solve engine.  0 = auto: 5 if it applies, else 4, 3, 2, 1 (the first that fits).
                              1 = global-state engine (any size), 2 = strip on-chip engine, 3 = column-blocked
                              on-chip engine (nx = 256 or 512 unknowns per row) — engines 1-3 solve every level
                              with Jacobi-scaled BiCGSTAB to lin_rtol behind grid-wide barriers;
                              4 = neighbour-synchronised engine: every level solved by lin_sweeps red-black SOR
                              sweeps (Young's relaxation from the Jacobi bound of A_1 at the initial iterate),
                              only neighbouring row strips synchronise (64..512 unknowns per row, even; periodic
                              grids also need an even number of rows; <= 4 rows per CTA);
                              5 = pipeline of CTA sets: set p (sms / D CTAs) runs Newton iteration p over the levels one
                              level behind set p-1, D = pipeline_depth iterations in flight; a CTA keeps its strip of
                              rows of a level on chip (du in registers, u^n and b in shared memory), the level solves are
                              engine 4's red-black SOR sweeps, strips of a set meet through neighbour exchange only
                              (even row count, strip heights that have an instantiation; constant-viscosity Burgers on
                              periodic grids with 64, 256 or 512 unknowns per row: pit_newton_ps.cuh; the general law — heat,
                              Burgers with m2 > 0 — on Dirichlet or periodic grids with 256 unknowns per row:
                              pit_newton_ps0.cuh).  2/3/4/5: PIT_EINVAL if
                              they do not apply.  Level solves outside the Newton solve (pit_level_solve_device,
                              the product forms) always use BiCGSTAB (engines 1-3). */
    int32_t guess_cf;      /* initial Newton iterate when the caller passes no guess:
                              0 = u^0 at every level; c_f >= 2 = the paper's coarse-grid guess: sequential-
                              equivalent BDF1 solve on the grid coarsened by c_f in x, y and t (the same
                              all-at-once solver, on the device), then cubic-spline interpolation along x, y
                              (periodic splines on periodic grids, not-a-knot otherwise) and t (not-a-knot,
                              u^0 as the t = 0 knot).  c_f must divide nx, ny and nt; coarse grid >= 2
                              (Dirichlet) / >= 3 (periodic) intervals.  Paper: 4 (heat), 3 (Burgers) */
    int32_t stop_norm;     /* 0 = max|dU_k| (default); 1 = the paper's L2 update norm
                              sqrt(sum (dU_k)^2 / (nt ns)) */
    int32_t lin_sweeps;    /* engine 4: red-black SOR sweeps per level solve; 0 = auto =
                              ceil(ln(lin_rtol) / ln(omega - 1)), the a-priori sweep count for a lin_rtol error
                              reduction at Young's rate omega - 1 (the reached level residuals are reported by
                              pit_engine_info) */
    int32_t lin_check;     /* engine 4: the level solves' a-posteriori residual ||b - A_n du^n|| is measured on every
                              lin_check-th level and the last (0 = default 16, 1 = every level): it waits for the
                              neighbouring strips' final values, one more exchange on the level's critical path */
} pit_config;

typedef struct pit_handle pit_handle;

/* Fill *cfg with defaults (abi_version set, everything else zero / defaults). */
void pit_config_init(pit_config* cfg);

/* Validate cfg, select the device, allocate all device memory.  *out = NULL on failure.
 * Errors: PIT_EINVAL (cfg NULL/invalid), PIT_ECUDA (no sm_100 device), PIT_ENOMEM. */
int pit_create(const pit_config* cfg, pit_handle** out);

/* Device bytes a handle for cfg holds (every buffer pit_create would cudaMalloc: iterate buffers, solver state,
 * exchange cells, histories, the coarse-grid guess's nested handle), so that the caller (e.g. torch) can own the
 * memory.  Selects the device and the engines like pit_create (needs a usable sm_100 device); allocates nothing.
 * Errors: as pit_create (PIT_EINVAL, PIT_ECUDA).  Follows SPEC.md's run_paradin(grid, model, cfg) interface
 * (SPEC.md:351-359): the problem statement in, the memory plan out. */
int pit_workspace_bytes(const pit_config* cfg, size_t* bytes);

/* pit_create with every create-time buffer carved from dev_ws (device memory the caller owns and keeps alive
 * until pit_destroy; any alignment; at least pit_workspace_bytes(cfg) bytes).  pit_destroy frees nothing inside it.
 * The product forms' scratch (pit_product_window_device, pit_explicit_window_device, inverse_mode PRODUCT_WINDOW /
 * EXPLICIT) is grown on first use with cudaMalloc, outside the workspace.
 * Errors: PIT_EINVAL (NULL / empty workspace), PIT_ENOMEM (workspace too small), others as pit_create. */
int pit_create_with_workspace(const pit_config* cfg, void* dev_ws, size_t bytes, pit_handle** out);

/* NULL-safe.  Frees everything pit_create allocated. */
void pit_destroy(pit_handle* h);

/* Synchronous solve with HOST buffers (copies in, solves, copies out).
 *   u0    [ns]             initial data at the unknown nodes (host)
 *   bc    [nt][2(nx+ny)]   Dirichlet rings at t^n, or NULL = homogeneous; ignored if periodic
 *   guess [nt][ns]         initial Newton iterate, or NULL = u0 at every level
 *   u_out [nt][ns]         solution (written for PIT_OK, PIT_OK_FLOOR and PIT_ENOCONV)
 *   hist  [newton_max][4]  per iteration k: { rms R(U_k), max|R(U_k)|, rms dU_k, max|dU_k| }
 *                          (rms dU_k is the paper's "residual"); may be NULL
 *   n_iter                 iterations performed; may be NULL
 * Returns the solve status (PIT_OK / PIT_OK_FLOOR / PIT_ENOCONV / PIT_EBREAKDOWN) or an error.
 * With engine 5, from the second call on a handle, the iterate the previous call ended in is streamed to u_out level by
 * level while the kernel still runs (a copy stream follows the strips' level counters; pinned u_out overlaps fully);
 * if this solve ends in another iteration the copy is redone after the kernel.  The result is the same either way. */
int pit_solve(pit_handle* h, const double* u0, const double* bc, const double* guess,
              double* u_out, double* hist, int32_t* n_iter);

/* Asynchronous solve on the caller's stream with DEVICE buffers (same shapes as pit_solve).
 *   d_info [2] int32 = { n_iter, status } written on the device at the end of the solve.
 *   cuda_stream: a cudaStream_t (NULL = legacy default stream).
 * The return value reports only argument / launch errors; the solve status is d_info[1] once the
 * stream work completes.  d_u_out is the library's to write from the first kernel on: engine 5 keeps the iterate it
 * expects to be the last one there (no final copy), so its contents are unspecified until the stream work completes. */
int pit_solve_device(pit_handle* h, const double* d_u0, const double* d_bc, const double* d_guess,
                     double* d_u_out, double* d_hist, int32_t* d_info, void* cuda_stream);

/* Kernel (a) on its own: the space-time Newton residual R = -G(U) of Eq. (5) for all
 * levels of the DEVICE iterate d_U [nt][ns] (u^0 = d_u0), written to d_R [nt][ns]; optional d_diag
 * [nt][ns] receives the diagonal of every A_n (Eq. 6), and d_norms [2] = { rms R, max|R| } (both may
 * be NULL).  Asynchronous on cuda_stream. */
int pit_residual_device(pit_handle* h, const double* d_U, const double* d_u0, const double* d_bc,
                        double* d_R, double* d_diag, double* d_norms, void* cuda_stream);

/* Stage (c) on its own, for tests: solve A_n x = b for ONE level n (1..nt) whose Jacobian block is
 * taken at the device iterate d_U (level n-1 from d_U, or d_u0 when n = 1, enters only via the ring /
 * nothing — A_n depends on u^n only).  d_b, d_x: [ns] device.  d_info [2] = { iterations, status }. */
int pit_level_solve_device(pit_handle* h, int32_t level, const double* d_U, const double* d_bc,
                           const double* d_b, double* d_x, int32_t* d_info, void* cuda_stream);

/* Stage (b2) on its own, for tests: the literal Theorem 1 product form (recursions
 * PAPER.md:221-230) for levels [s0, s0+L) of the device iterate: given the residuals d_R [nt][ns] and
 * the carry d_carry [ns] (= du^{s0-1}, or NULL for zero), writes du^{s0..s0+L-1} into d_dU [L][ns].
 * Returns PIT_ECOND if the window fails the Section 7 gate (prod ||A_i||_inf > 1e6 over the window's
 * longest chain). */
int pit_product_window_device(pit_handle* h, int32_t s0, int32_t L, const double* d_U, const double* d_u0,
                              const double* d_bc, const double* d_R, const double* d_carry, double* d_dU,
                              int32_t* d_info, void* cuda_stream);

/* N3 on its own, for tests: the paper's explicit decoupled form for levels [s0, s0+L) of the device iterate
 * (Theorem 1): P^1 = A_{s0}, P^m = P^{m-1} A_{s0+m-1} formed in band storage (Eq. 10,
 * PAPER.md:221-230; half-bandwidth m * nxu, Theorem 2), r~^m = sum_{j<=m} P^{j-1} r^j with r^1 += d_carry, the
 * diagonal preconditioner diag(P^m) on the left, and each P^m du^m = r~^m solved by a banded LU
 * WITHOUT pivoting.  Arguments as pit_product_window_device; no conditioning gate (this is the
 * path that exhibits the Section 7 limit).  d_info [2] = { 0, PIT_OK | PIT_EBREAKDOWN (zero / non-finite
 * pivot) } on the device.  Errors: PIT_EINVAL for periodic grids (P^n is not banded) or band storage
 * L * ns * (2w+1) doubles > 16 GB; PIT_ENOMEM.  The handle owns the band scratch (grown on demand). */
int pit_explicit_window_device(pit_handle* h, int32_t s0, int32_t L, const double* d_U, const double* d_u0,
                               const double* d_bc, const double* d_R, const double* d_carry, double* d_dU,
                               int32_t* d_info, void* cuda_stream);

/* N4 — one step of the multi-GPU time-slab pipeline: ONE all-at-once Newton iteration (Eq. (5)-(7),
 * PAPER.md:86-156) over this handle's nt levels taken as levels s..s+nt-1 of a longer horizon.  The recursion of
 * Eq. (7) continues across the slab boundary: level s's residual uses d_uprev = U_k at level s-1 (u^0 for the first
 * slab) and its solve starts from  b = r^s + d_carry_in  (d_carry_in = du_k of level s-1, NULL = 0 for the first
 * slab).  Inputs d_U_k [nt][ns] (iterate k of the slab), d_bc the slab's Dirichlet rings; outputs d_U_k1 [nt][ns] =
 * U_k + dU, d_carry_out [ns] = du_k of the slab's last level (the next slab's carry; may be NULL), d_hist [4] = the
 * slab's { rms R(U_k), max|R(U_k)|, rms dU_k, max|dU_k| } over its nt ns unknowns (combine slabs by sums of
 * squares and maxima; the stop rule is the caller's), d_info [2] (may be NULL).  Engine 4 only (PIT_EINVAL
 * otherwise); all pointers device, 16-byte aligned; asynchronous on cuda_stream. */
int pit_slab_iterate_device(pit_handle* h, const double* d_uprev, const double* d_carry_in, const double* d_bc,
                            const double* d_U_k, double* d_U_k1, double* d_carry_out, double* d_hist, int32_t* d_info,
                            void* cuda_stream);

/* The initial Newton iterate on its own: with guess_cf >= 2 the coarse-grid solve + spline
 * interpolation described at pit_config.guess_cf, else u^0 at every level; written to d_U0 [nt][ns] (device).
 * d_u0 [ns], d_bc as in pit_solve_device.  Asynchronous on cuda_stream. */
int pit_initial_guess_device(pit_handle* h, const double* d_u0, const double* d_bc, double* d_U0, void* cuda_stream);

/* Number of unknowns per level and device bytes the handle holds. */
int pit_sizes(const pit_handle* h, int64_t* ns, int64_t* device_bytes);

/* Pipeline statistics of the last solve (synchronizes with it; n >= 17 + 256 + 7 for every field):
 * out[0] = wavefront steps, out[1] = total BiCGSTAB iterations summed over steps (max per step),
 * out[2] = pipeline depth used, out[3] = grid CTAs, out[4] = kernel launches of the last solve,
 * out[5] = device time of the persistent Newton kernel of the last solve [ns] (CUDA events on the
 * launching stream), out[6] = device time of the iterate-initialisation kernel [ns], out[7] = engine
 * (1 global-state, 2 strip on-chip, 3 column-blocked on-chip, 4 neighbour-synchronised, 5 pipeline of CTA sets; for
 * 4 and 5 out[0] = levels one CTA processed, out[2] / out[3] = the depth and CTAs the kernel ran with), out[8..14] = on-chip engine cycle accounting summed over CTAs
 * (prologue, phase 1, phase 2, epilogue, grid barriers, scalar reductions, step bookkeeping) when the
 * environment variable PIT_TRACE was set at pit_create (zeros otherwise), out[15] = 1 if the last solve
 * inverted Eq. (6) with the (b2) product form (inverse_mode PRODUCT_WINDOW, or AUTO with the whole horizon
 * inside the Section 7 gate), 2 with the N3 explicit banded form, 0 for the on-device level recurrence, out[16] = BiCGSTAB iterations summed
 * over all (level, iteration) pairs (on-chip engine), out[17 + k] = those of Newton iteration k,
 * out[273..278] = prologue sub-categories of the cycle accounting, out[279] = device time of the coarse-grid
 * initial guess (coarse solve + interpolation) [ns], 0 without it. */
int pit_stats(pit_handle* h, int64_t* out, int32_t n);

/* Engine facts of the last Newton solve (synchronizes with it).  out[0] = engine (1..5), out[1] = omega,
 * out[2] = sweeps per level solve, out[3] = the Jacobi bound q (engines 4 and 5; 0 otherwise), then for k = 0..n_iter-1:
 * out[4 + 2k] = ||res||_2 / ||b||_2 of iteration k's level solves over all levels (res = b - A_n du^n, b = r^n +
 * du^{n-1}), out[5 + 2k] = max |res| (engines 4 and 5; zeros otherwise).  n = number of doubles out can hold. */
int pit_engine_info(pit_handle* h, double* out, int32_t n);

const char* pit_strerror(int code);
const char* pit_last_error(const pit_handle* h);
int pit_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PIT_H */
