// pit_internal.cuh — device-side building blocks of libpit (sm_100a, fp64).
//
// Shared by the kernels of pit_kernels.cu only (the host API includes it for the parameter structs).
// Nothing here is shared with the CPU oracle (oracle/), which is an independent implementation.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pit {

constexpr int BLOCK = 256;       // threads per CTA of every kernel
constexpr int NWARP = BLOCK / 32;
constexpr int NPART = 8;         // per-CTA partial slots per reduction phase
constexpr int MAXK = 256;        // newton_max cap (S_k table in shared memory)
constexpr int MAXD = 16;         // pipeline depth cap
constexpr int NVEC = 13;         // vectors per pipeline slot

// Problem constants (the paper's problem statement, Eqs. (1)-(3)).
struct Prob {
    int pde, bc;          // 0 heat / 1 Burgers ; 0 Dirichlet / 1 periodic
    int nx, ny;           // intervals
    int nxu, nyu;         // unknowns per row / column
    int nt, ring_len;
    long long ns;
    double ihx2, ihy2;    // 1/h^2
    double i2hx, i2hy;    // 1/(2h)
    double dt, m0, m2;
};

// Sense-free generation barrier over all co-resident CTAs of a cooperative launch, carrying an OR flag.
struct GridBar {
    unsigned int count;
    unsigned int gen;
    unsigned int flag_acc;
    unsigned int flag_out[2];
    unsigned int err;            // sticky error bits (1 = NaN/Inf, 2 = Krylov breakdown)
    unsigned int pad[2];
};

// One pipeline slot = the state of one per-level BiCGSTAB solve (SoA, each [ns]).
struct Slot {
    double *cE, *cW, *cN, *cS;   // Jacobi-scaled off-diagonal coefficients of A_n (diag scaled to 1)
    double *bt;                  // scaled right-hand side b~ = D^{-1}(r^n + du^{n-1}) (= BiCGSTAB r0^)
    double *x;                   // iterate; after the epilogue: du^n, the carry for level n+1
    double *r;
    double *p[2], *v[2];         // double-buffered by iteration parity (read as halo while rewritten)
    double *s, *t;
};

struct SolveParams {
    Prob P;
    const double* u0;            // [ns]
    const double* ring;          // [nt][ring_len] or nullptr (homogeneous / periodic)
    double* U;                   // [B][nt][ns] iterate ring buffer (iterate k lives in buffer k % B)
    int B, D, G;
    double* slotmem;             // D * NVEC * ns
    double* part;                // [2][G][NPART]
    double* hpart;               // [G][4]
    GridBar* bar;
    double* hist;                // [newton_max][4]
    int* info;                   // [2] { n_iter, status }
    double* u_out;               // [nt][ns] (mode 0)
    double newton_tol, lin_rtol, lin_atol;
    int newton_max, lin_max;
    long long* stats;            // [4] steps, inner iterations, depth, G
    int mode;                    // 0 = Newton solve, 1 = batch of independent level solves A_n x = b
    int nb;                      // mode 1: number of right-hand sides (<= D)
    int blev[MAXD];              // mode 1: level n (1-based) of right-hand side a; A_n taken at U level n
    const double* bptr[MAXD];    // mode 1: right-hand sides [ns]
    double* xptr[MAXD];          // mode 1: solutions [ns] (may alias bptr)
    int hmax;                    // on-chip engine: max rows of a CTA strip
    struct BarState* bs;         // on-chip engine: monotonic barrier state
    unsigned long long* trace;   // optional cycle accounting [7] (nullptr = off)
    int x0carry;                 // on-chip engine: start each level solve from du^{n-1} (else 0)
    double* halo;                // column engine: [G][2 sides][6 vectors][512] published boundary rows
    int stop_norm;               // 0: stop on max|dU_k|; 1: on the RMS update norm
    int merge;                   // column engine, Newton solves: merged first BiCGSTAB iteration (periodic, nx 512)
};

// Grid barrier state of the on-chip engine (zeroed before every launch).
struct BarState {
    unsigned long long ctr[32];  // ctr[0] and ctr[16]: the two parity counters, 128 B apart
    unsigned int err;            // sticky error bits (1 = NaN/Inf, 2 = Krylov breakdown)
    unsigned int pad[31];
};

__host__ __device__ inline Slot slot_at(double* base, long long ns, int d) {
    double* m = base + (long long)d * NVEC * ns;
    Slot s;
    s.cE = m; s.cW = m + ns; s.cN = m + 2 * ns; s.cS = m + 3 * ns;
    s.bt = m + 4 * ns; s.x = m + 5 * ns; s.r = m + 6 * ns;
    s.p[0] = m + 7 * ns; s.p[1] = m + 8 * ns; s.v[0] = m + 9 * ns; s.v[1] = m + 10 * ns;
    s.s = m + 11 * ns; s.t = m + 12 * ns;
    return s;
}

// ---- the laws of Eq. (1), PAPER.md:50-52 --------------------------------------------------------
__device__ __forceinline__ double law_mu(const Prob& P, double u) { return fma(P.m2 * u, u, P.m0); }
__device__ __forceinline__ double law_dmu(const Prob& P, double u) { return 2.0 * P.m2 * u; }
__device__ __forceinline__ double law_f(const Prob& P, double u) { return P.pde ? 0.5 * u * u : 0.0; }
__device__ __forceinline__ double law_df(const Prob& P, double u) { return P.pde ? u : 0.0; }

// Neighbour indices of unknown p.  A Dirichlet neighbour that is a boundary node has has* = false and
// index p (a valid dummy with a zero coefficient).  Periodic neighbours wrap.
struct Nbr {
    long long e, w, n, s;
    int ix, jy;
    bool he, hw, hn, hs;
};

__device__ __forceinline__ Nbr neighbours(const Prob& P, long long p) {
    Nbr q;
    const int ix = (int)(p % P.nxu), jy = (int)(p / P.nxu);
    q.ix = ix; q.jy = jy;
    if (P.bc == 1) {
        q.e = ix + 1 < P.nxu ? p + 1 : p - ix;
        q.w = ix > 0 ? p - 1 : p + (P.nxu - 1);
        q.n = jy + 1 < P.nyu ? p + P.nxu : (long long)ix;
        q.s = jy > 0 ? p - P.nxu : p + (long long)(P.nyu - 1) * P.nxu;
        q.he = q.hw = q.hn = q.hs = true;
    } else {
        q.he = ix + 1 < P.nxu; q.e = q.he ? p + 1 : p;
        q.hw = ix > 0;         q.w = q.hw ? p - 1 : p;
        q.hn = jy + 1 < P.nyu; q.n = q.hn ? p + P.nxu : p;
        q.hs = jy > 0;         q.s = q.hs ? p - P.nxu : p;
    }
    return q;
}

// Values of u at the 5 stencil nodes; Dirichlet boundary nodes come from the level's ring (Eq. 2).
struct Vals { double c, e, w, n, s; };

__device__ __forceinline__ Vals stencil_values(const Prob& P, const double* __restrict__ u,
                                               const double* __restrict__ ringn, long long p, const Nbr& q) {
    Vals v;
    v.c = u[p];
    if (P.bc == 1) {
        v.e = u[q.e]; v.w = u[q.w]; v.n = u[q.n]; v.s = u[q.s];
        return v;
    }
    const int nxp = P.nx + 1;
    v.e = q.he ? u[q.e] : (ringn ? ringn[2 * nxp + (P.ny - 1) + q.jy] : 0.0);
    v.w = q.hw ? u[q.w] : (ringn ? ringn[2 * nxp + q.jy] : 0.0);
    v.n = q.hn ? u[q.n] : (ringn ? ringn[nxp + q.ix + 1] : 0.0);
    v.s = q.hs ? u[q.s] : (ringn ? ringn[q.ix + 1] : 0.0);
    return v;
}

// Residual G^n = tau * (Eq. (3) lhs - rhs) at one unknown (PAPER.md:67-74 times tau_n)
// with face viscosity mu((u_C + u_nb)/2) (R1), and the 5 coefficients of the diagonal block
// A_n = I + tau (dF/du) of Eq. (6) at that row; columns of Dirichlet boundary nodes are
// zeroed (they belong to q, Eq. (4)).
struct RJ { double G, aC, aE, aW, aN, aS; };

// All five coefficients, no column dropping (the on-chip engine drops Dirichlet columns by giving the
// operand zero halo values instead).
__device__ __forceinline__ RJ residual_jacobian_raw(const Prob& P, const Vals& v, double uprev) {
    const double bE = 0.5 * (v.c + v.e), bW = 0.5 * (v.w + v.c), bN = 0.5 * (v.c + v.n), bS = 0.5 * (v.s + v.c);
    const double mE = law_mu(P, bE), mW = law_mu(P, bW), mN = law_mu(P, bN), mS = law_mu(P, bS);
    const double gE = v.e - v.c, gW = v.c - v.w, gN = v.n - v.c, gS = v.c - v.s;
    const double conv = (law_f(P, v.e) - law_f(P, v.w)) * P.i2hx + (law_f(P, v.n) - law_f(P, v.s)) * P.i2hy;
    const double visc = (mE * gE - mW * gW) * P.ihx2 + (mN * gN - mS * gS) * P.ihy2;
    RJ o;
    o.G = (v.c - uprev) + P.dt * (conv - visc);
    const double hE = 0.5 * law_dmu(P, bE) * gE, hW = 0.5 * law_dmu(P, bW) * gW;
    const double hN = 0.5 * law_dmu(P, bN) * gN, hS = 0.5 * law_dmu(P, bS) * gS;
    o.aC = 1.0 + P.dt * ((mE + mW - hE + hW) * P.ihx2 + (mN + mS - hN + hS) * P.ihy2);
    o.aE = P.dt * (law_df(P, v.e) * P.i2hx - (mE + hE) * P.ihx2);
    o.aW = P.dt * (-law_df(P, v.w) * P.i2hx - (mW - hW) * P.ihx2);
    o.aN = P.dt * (law_df(P, v.n) * P.i2hy - (mN + hN) * P.ihy2);
    o.aS = P.dt * (-law_df(P, v.s) * P.i2hy - (mS - hS) * P.ihy2);
    return o;
}

__device__ __forceinline__ RJ residual_jacobian(const Prob& P, const Vals& v, const Nbr& q, double uprev) {
    RJ o = residual_jacobian_raw(P, v, uprev);
    if (!q.he) o.aE = 0.0;
    if (!q.hw) o.aW = 0.0;
    if (!q.hn) o.aN = 0.0;
    if (!q.hs) o.aS = 0.0;
    return o;
}

// Off-diagonal coefficients only (the matvec of the on-chip engine recomputes them from u every time).
struct Off { double e, w, n, s; };
__device__ __forceinline__ Off offdiag(const Prob& P, const Vals& v) {
    const double bE = 0.5 * (v.c + v.e), bW = 0.5 * (v.w + v.c), bN = 0.5 * (v.c + v.n), bS = 0.5 * (v.s + v.c);
    const double hE = 0.5 * law_dmu(P, bE) * (v.e - v.c), hW = 0.5 * law_dmu(P, bW) * (v.c - v.w);
    const double hN = 0.5 * law_dmu(P, bN) * (v.n - v.c), hS = 0.5 * law_dmu(P, bS) * (v.c - v.s);
    Off o;
    o.e = P.dt * (law_df(P, v.e) * P.i2hx - (law_mu(P, bE) + hE) * P.ihx2);
    o.w = P.dt * (-law_df(P, v.w) * P.i2hx - (law_mu(P, bW) - hW) * P.ihx2);
    o.n = P.dt * (law_df(P, v.n) * P.i2hy - (law_mu(P, bN) + hN) * P.ihy2);
    o.s = P.dt * (-law_df(P, v.s) * P.i2hy - (law_mu(P, bS) - hS) * P.ihy2);
    return o;
}

// ---- fixed-order CTA reductions ---------------------------------------------------------------
// NS sums followed by NM maxima (of non-negative values); result valid in thread 0.  The butterfly
// gives every lane the same bits (IEEE + is commutative), the cross-warp pass runs in warp order.
template <int NS, int NM>
__device__ __forceinline__ void block_reduce(double (&a)[NS + NM], double* sm /* [NWARP][NS+NM] */) {
    constexpr int N = NS + NM;
    #pragma unroll
    for (int i = 0; i < N; ++i)
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, a[i], o);
            a[i] = i < NS ? a[i] + y : fmax(a[i], y);
        }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
        #pragma unroll
        for (int i = 0; i < N; ++i) sm[w * N + i] = a[i];
    __syncthreads();
    if (w == 0) {
        #pragma unroll
        for (int i = 0; i < N; ++i) {
            double v = l < NWARP ? sm[l * N + i] : 0.0;
            #pragma unroll
            for (int o = NWARP / 2; o > 0; o >>= 1) {
                const double y = __shfl_xor_sync(0xffffffffu, v, o);
                v = i < NS ? v + y : fmax(v, y);
            }
            a[i] = v;
        }
    }
    __syncthreads();
}

}  // namespace pit
