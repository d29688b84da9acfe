// pit_newton_nb.cuh — engine 4: the all-at-once Newton solve (Eq. (5)) with the exact block
// inverse of Eq. (7) applied as the level recurrence du^n = A_n^{-1}(r^n + du^{n-1}), whose
// per-level solves are a FIXED number S of red-black SOR sweeps started from the carry du^{n-1}, and whose only
// inter-CTA synchronisation is point-to-point between neighbouring row strips.
//
// Layout: one persistent CTA per SM (cooperative launch: every CTA co-resident).  CTA c owns rows [r0, r0+h) of
// EVERY level for the whole solve.  The CTA is DM warp groups of NXU/2 threads; group p runs Newton iteration
// k = pass*D + p (the D iterations in flight of the level wavefront) over levels n = 1..nt, thread t of a group
// owning columns 2t, 2t+1 of the strip's rows in registers.  Group p starts level n once group p-1 of the same CTA has
// produced U_k^n (a shared-memory level counter), so the wavefront emerges from the data dependencies; while one
// group waits for its neighbours' boundary rows the SM runs the others.
//
// Why a fixed-sweep SOR and not a Krylov solver: a Krylov iteration needs two GLOBAL reductions per iteration (grid
// barriers, ~2 us each on B200 — engine 3 spends ~30% of its time in them), a stationary sweep needs only the
// neighbouring strips' boundary rows.  A_n is a 5-point matrix (consistently ordered), so with Young's optimal
// relaxation omega = 2 / (1 + sqrt(1 - q^2)) for a bound q >= rho(D^-1 (L+U)) one red-black sweep contracts the error
// by omega - 1 (c5: q = 0.345, 0.032 per sweep); S = ceil(ln(lin_rtol) / ln(omega - 1)) sweeps (or pit_config.
// lin_sweeps).  The relative residual every level solve reached is measured a posteriori and reported per Newton
// iteration (linres), and Newton's own stop rule on max|dU| decides convergence as in every engine.
//
// Neighbour exchange: "LL" cells — every fp64 value travels as two 8-byte words {lo32 | flag, hi32 | flag} written by
// one 16-byte store; the consumer polls its own cells until both flags carry the expected publication number, so no
// memory fence is ever needed (a word is single-copy atomic).  Every CTA runs the same schedule per group, so
// publication numbers are identical across CTAs and a consumer knows the number of the publication it needs.
//
// Per Newton iteration the CTA's partial norms are reduced by the last CTA to finish the iteration (fixed-order sum
// over CTAs: deterministic), which posts the stop decision; CTAs wait for decisions only at pass ends.
#pragma once
#include "pit_nb_params.cuh"

namespace pit {

// ---- LL cells ---------------------------------------------------------------------------------------------
struct LLc { unsigned long long w0, w1; };

__device__ __forceinline__ void ll_put(unsigned long long* p, double v, unsigned f) {
    const unsigned long long w0 = ((unsigned long long)f << 32) | (unsigned)__double2loint(v);
    const unsigned long long w1 = ((unsigned long long)f << 32) | (unsigned)__double2hiint(v);
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
// The poll is a strong GPU-scope load (each 8-byte word single-copy atomic; data and flag share a word).  One hop
// (store -> the neighbour's poll sees it) costs ~0.7 us on B200 whatever the store flavour (tools/hop_bench.cu,
// profiles/r02/hop_latency_microbench.txt).  ld.global.cv / .cg polls look twice as fast there but return words whose
// data does not belong to the flag they carry (tools/ll_check.cu, profiles/r02/ll_poll_correctness.txt): not usable.
__device__ __forceinline__ LLc ll_issue(const unsigned long long* p) {
    LLc c;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(c.w0), "=l"(c.w1) : "l"(p) : "memory");
    return c;
}
__device__ __forceinline__ double ll_take(const unsigned long long* p, LLc c, unsigned f) {
    while ((unsigned)(c.w0 >> 32) != f || (unsigned)(c.w1 >> 32) != f) c = ll_issue(p);
    return __hiloint2double((int)(unsigned)c.w1, (int)(unsigned)c.w0);
}
// ll_take that also accounts the cycles spent re-polling (trace builds)
__device__ __forceinline__ double ll_take_t(const unsigned long long* p, LLc c, unsigned f, long long& acc) {
    if ((unsigned)(c.w0 >> 32) != f || (unsigned)(c.w1 >> 32) != f) {
        const long long t0 = clock64();
        do { c = ll_issue(p); } while ((unsigned)(c.w0 >> 32) != f || (unsigned)(c.w1 >> 32) != f);
        acc += clock64() - t0;
    }
    return __hiloint2double((int)(unsigned)c.w1, (int)(unsigned)c.w0);
}

__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }

// Jacobi bound q = max_i sum_j |a_ij| / |a_ii| of A_1 at the initial iterate's level 1, then omega and S.
static __global__ void __launch_bounds__(BLOCK) k_nb_q(Prob P, const double* __restrict__ U1, const double* __restrict__ ring,
                                                 unsigned long long* qbits) {
    double q = 0.0;
    for (long long p = blockIdx.x * (long long)BLOCK + threadIdx.x; p < P.ns; p += (long long)gridDim.x * BLOCK) {
        const Nbr nb = neighbours(P, p);
        const Vals v = stencil_values(P, U1, ring, p, nb);
        const RJ o = residual_jacobian(P, v, nb, v.c);
        q = fmax(q, (fabs(o.aE) + fabs(o.aW) + fabs(o.aN) + fabs(o.aS)) / fabs(o.aC));
    }
    for (int o = 16; o > 0; o >>= 1) q = fmax(q, __shfl_xor_sync(0xffffffffu, q, o));
    if ((threadIdx.x & 31) == 0) atomicMax(qbits, (unsigned long long)__double_as_longlong(q));   // q >= 0: bits order
}

static __global__ void k_nb_ctl(const unsigned long long* qbits, double lin_rtol, int sweeps, int check, double* ctl) {
    const double q0 = __longlong_as_double((long long)*qbits);
    const double q = fmin(0.9999, 1.0 - 0.99 * (1.0 - q0));   // small safety margin on the bound (1% of 1 - q)
    const double omega = 2.0 / (1.0 + sqrt(1.0 - q * q));     // Young: rate omega - 1 for rho(J) <= q
    int S = sweeps;
    if (S <= 0) {
        const double rate = fmax(omega - 1.0, 1e-6);
        S = (int)ceil(log(lin_rtol) / log(rate));
        S = max(1, min(S, 400));
    }
    ctl[0] = omega;
    ctl[1] = (double)S;
    ctl[2] = q0;
    ctl[3] = (double)(check > 0 ? check : 16);
}


// ---- the persistent kernel ------------------------------------------------------------------------------------
// Thread t of a group owns CPT consecutive columns CPT t .. CPT t + CPT - 1 of the strip's rows (registers, physical
// order).  The strip height H and the parity PR0 of the first own row are template parameters of the body (every
// CTA has H in {HB, HB + 1}), so the colour of every register, the in-thread / out-of-thread split of the E/W
// neighbours and every subscript are compile-time: no row guards, no selects, no dynamic indexing.  A colour has
// HC = CPT / 2 points per thread and row; the h-th is column ((PR0 + r + colour) & 1) + 2h.
template <int HB, int LAW, int NXU, int DM, int CPT>
struct NbEngine {
    static constexpr int T = NXU / CPT;        // threads per group
    static constexpr int NT = DM * T;          // threads per CTA
    static constexpr int W = NXU + 2;          // smem row pitch: column i at i + 1, pads at 0 and NXU + 1
    static constexpr int NW = T / 32;          // warps per group
    static constexpr int RM = HB + 1;          // max strip height
    static constexpr int HC = CPT / 2;         // points of one colour per thread and row
    static constexpr size_t OFF_Q = 0;                                   // qs  [DM][RM][W]  sweep exchange values
    static constexpr size_t OFF_U = OFF_Q + (size_t)DM * RM * W;         // us  [DM][RM][W]  staged u rows
    static constexpr size_t OFF_B = OFF_U + (size_t)DM * RM * W;         // bs  [DM][RM][CPT][T] right-hand sides
    static constexpr size_t OFF_A = OFF_B + (size_t)DM * RM * CPT * T;   // acc [DM][NB_NP][T]
    static constexpr size_t SMEM = (OFF_A + (size_t)DM * NB_NP * T) * sizeof(double);
    static_assert(NW >= 1 && T % 32 == 0, "a group is whole warps");

    template <int H, int PR0>
    __device__ __forceinline__ static void run(const NbParams& S, double* sm) {
        const Prob P = S.P;
        const int G = S.G, c = blockIdx.x;
        const int p = threadIdx.x / T, t = threadIdx.x % T;   // warp group (Newton iteration in flight), columns
        const int c0 = CPT * t;                                // first own column
        const long long ns = P.ns;
        const int nyu = P.nyu, nt = P.nt, D = S.D, B = S.B;
        const bool per = P.bc == 1;
        const int hb = nyu / G, hr = nyu % G;
        const int r0 = c * hb + min(c, hr);
        const int cs = c > 0 ? c - 1 : (per ? G - 1 : -1);   // south neighbour strip (rows below)
        const int cn = c + 1 < G ? c + 1 : (per ? 0 : -1);  // north neighbour strip
        const double omega = __ldcg(S.ctl), tau = P.dt;
        const int SW = (int)__ldcg(S.ctl + 1);
        const int chk = max(1, (int)__ldcg(S.ctl + 3));      // level-residual check stride (levels)
        const int nxp = P.nx + 1;
        // LAW 1 (Burgers, constant mu = m0): a_E x_E = x_E (ax u_E - bx), a_W x_W = x_W (-ax u_W - bx), same in y
        const double ax = tau * P.i2hx, bx = tau * P.m0 * P.ihx2, ay = tau * P.i2hy, by = tau * P.m0 * P.ihy2;
        const double aC1 = 1.0 + 2.0 * (bx + by), invC1 = 1.0 / aC1;
        const double rfac = (1.0 - omega) / omega;

        double* qs = sm + OFF_Q + (size_t)p * RM * W;          // this group's arrays
        double* us = sm + OFF_U + (size_t)p * RM * W;
        double* bs = sm + OFF_B + (size_t)p * RM * CPT * T;
        double* acc = sm + OFF_A + (size_t)p * NB_NP * T;
        __shared__ double red_s[DM][NW][NB_NP];
        __shared__ int s_dec[2];
        __shared__ int s_last[DM];
        __shared__ volatile int lvl_done[DM];    // levels of the current pass each group has finished

        double x[H][CPT], u[H][CPT];
        double hS[CPT], hN[CPT];                 // u of the halo rows r0 - 1 and r0 + H (physical columns)
        double co[LAW == 0 ? H : 1][LAW == 0 ? CPT : 1][5];   // LAW 0: 1/a_C, a_E, a_W, a_N, a_S
        int lastx = -1;
        unsigned qx = 0, qu = 0;                 // publication counters of this group (identical in every CTA)
        long long levels = 0;
        long long tr[NB_TR] = {0, 0, 0, 0, 0, 0, 0, 0};
        const bool trace = S.trace != nullptr && p == 0;
        const long long t_start = clock64();
        long long tm = t_start;
        auto mark = [&](int i) { if (trace) { const long long now = clock64(); tr[i] += now - tm; tm = now; } };
        auto gbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + p), "r"(T) : "memory"); };

        auto ring_bottom = [&](const double* rg, int i) { return rg ? __ldcg(rg + i + 1) : 0.0; };
        auto ring_top = [&](const double* rg, int i) { return rg ? __ldcg(rg + nxp + i + 1) : 0.0; };
        auto ring_left = [&](const double* rg, int j) { return rg ? __ldcg(rg + 2 * nxp + j) : 0.0; };
        auto ring_right = [&](const double* rg, int j) { return rg ? __ldcg(rg + 2 * nxp + (P.ny - 1) + j) : 0.0; };

        // LL channels of group p: x ring [G][DM][NB_RX][2][HC][T], U ring [G][DM][NB_RU][2][NXU] (2 words per cell)
        auto xbase = [&](int cta) { return S.llx + (((size_t)cta * DM + p) * NB_RX * 2 * HC * T) * 2; };
        auto ubase = [&](int cta, int grp) { return S.llu + (((size_t)cta * DM + grp) * NB_RU * 2 * NXU) * 2; };
        unsigned long long* myx = xbase(c);
        unsigned long long* myu = ubase(c, p);
        const unsigned long long* sx = cs >= 0 ? xbase(cs) : nullptr;
        const unsigned long long* nxq = cn >= 0 ? xbase(cn) : nullptr;
        const unsigned long long* su = (cs >= 0 && p > 0) ? ubase(cs, p - 1) : nullptr;   // U_k^n of their group p-1
        const unsigned long long* nu = (cn >= 0 && p > 0) ? ubase(cn, p - 1) : nullptr;
        auto xcell = [&](auto* base, unsigned q, int side, int h) {
            return base + ((size_t)(((q % NB_RX) * 2 + side) * HC + h) * T + t) * 2;
        };
        auto ucell = [&](auto* base, unsigned q, int side, int j) {
            return base + ((size_t)((q % NB_RU) * 2 + side) * NXU + c0 + j) * 2;
        };
        auto bsm = [&](int r, int j) -> double& { return bs[(size_t)(r * CPT + j) * T + t]; };
        auto ac = [&](int j) -> double& { return acc[(size_t)j * T + t]; };
        // exchange value of column j of row r for the neighbouring thread (LAW 1: premultiplied by the coefficient
        // the neighbour applies: column c0 is the E neighbour of c0 - 1, column c0 + CPT - 1 the W neighbour of c0 + CPT)
        auto put_q = [&](double* q, int r, int j, double xv, double uv) {
            double v = xv;
            if (LAW == 1) v *= j == 0 ? fma(ax, uv, -bx) : fma(-ax, uv, -bx);
            q[r * W + c0 + j + 1] = v;
            if (per) {
                if (j == 0 && t == 0) q[r * W + NXU + 1] = v;
                if (j == CPT - 1 && t == T - 1) q[r * W + 0] = v;
            }
        };

        for (int i = t; i < NB_NP * T; i += T) acc[i] = 0.0;
        for (int i = t; i < RM * W; i += T) { qs[i] = 0.0; us[i] = 0.0; }
        if (threadIdx.x < DM) lvl_done[threadIdx.x] = 0;
        __syncthreads();

        for (int pass = 0;; ++pass) {
            const int k = pass * D + p;
            const bool active = p < D && k < S.newton_max;
            // carry du^0: 0, or (time slab, N4) the previous slab's du_k of the level before level 1
            const double* cin = (pass == 0 && p == 0) ? S.carry_in : nullptr;
            #pragma unroll
            for (int r = 0; r < H; ++r)
                #pragma unroll
                for (int j = 0; j < CPT; j += 2) {
                    double2 v = make_double2(0.0, 0.0);
                    if (cin) v = ldcg2(cin + (size_t)(r0 + r) * NXU + c0 + j);
                    x[r][j] = v.x;
                    x[r][j + 1] = v.y;
                }
            lastx = -1;
            for (int n = 1; active && n <= nt; ++n) {
                ++levels;
                // ---- U_k^n own rows come from group p-1 of this CTA (or the previous pass); back-pressure on
                //      group p+1 keeps this group's U publications within the neighbours' LL ring
                if (t == 0) {
                    if (p > 0) while (lvl_done[p - 1] < n) { }
                    if (p + 1 < D && k + 1 < S.newton_max) while (lvl_done[p + 1] < n - NB_LAG) { }
                    __threadfence_block();
                }
                gbar();
                mark(6);
                const double* Uk = S.U + (size_t)(k % B) * nt * ns;
                const double* un = Uk + (size_t)(n - 1) * ns;
                const double* up = n == 1 ? S.u0 : Uk + (size_t)(n - 2) * ns;
                const double* rg = S.ring ? S.ring + (size_t)(n - 1) * P.ring_len : nullptr;
                // ---- prologue A: u^n own rows (+ staging), halo rows, u^{n-1} own rows
                double pv[H][CPT];
                #pragma unroll
                for (int r = 0; r < H; ++r) {
                    #pragma unroll
                    for (int j = 0; j < CPT; j += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(un + (size_t)(r0 + r) * NXU + c0 + j);
                        const double2 w = *reinterpret_cast<const double2*>(up + (size_t)(r0 + r) * NXU + c0 + j);
                        u[r][j] = v.x; u[r][j + 1] = v.y;
                        pv[r][j] = w.x; pv[r][j + 1] = w.y;
                        us[r * W + c0 + j + 1] = v.x;
                        us[r * W + c0 + j + 2] = v.y;
                    }
                    if (per) {
                        if (t == 0) us[r * W + NXU + 1] = u[r][0];
                        if (t == T - 1) us[r * W + 0] = u[r][CPT - 1];
                    } else {
                        if (t == 0) us[r * W + 0] = ring_left(rg, r0 + r);
                        if (t == T - 1) us[r * W + NXU + 1] = ring_right(rg, r0 + r);
                    }
                }
                // halo rows of u^n: the neighbours' U_k^n boundary rows.  p >= 1: published (LL) by their group
                // p-1 when it finished level n; p == 0: written in the previous pass (global, after the pass sync).
                #pragma unroll
                for (int side = 0; side < 2; ++side) {
                    const int nb = side ? cn : cs;
                    double* dst = side ? hN : hS;
                    if (nb < 0) {    // Dirichlet boundary row
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) dst[j] = side ? ring_top(rg, c0 + j) : ring_bottom(rg, c0 + j);
                    } else if (p == 0) {
                        const int jr = side ? (r0 + H) % nyu : (r0 - 1 + nyu) % nyu;
                        #pragma unroll
                        for (int j = 0; j < CPT; j += 2) {
                            const double2 v = ldcg2(un + (size_t)jr * NXU + c0 + j);
                            dst[j] = v.x; dst[j + 1] = v.y;
                        }
                    } else {
                        const unsigned qn = (unsigned)(pass * nt + n - 1);   // group p-1 publishes U once per level
                        const unsigned long long* base = side ? nu : su;
                        const int sd = side ? 0 : 1;    // north strip's bottom row / south strip's top row
                        LLc a[CPT];
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) a[j] = ll_issue(ucell(base, qn, sd, j));
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) dst[j] = ll_take_t(ucell(base, qn, sd, j), a[j], qn + 1u, tr[2]);
                    }
                }
                gbar();
                // ---- prologue B: residual r^n = -G^n, b = r^n + du^{n-1}, exchange values of x0
                {
                    double ar2 = 0.0, arm = 0.0;
                    #pragma unroll
                    for (int r = 0; r < H; ++r) {
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) {
                            Vals v;
                            v.c = u[r][j];
                            v.e = j + 1 < CPT ? u[r][j + 1 < CPT ? j + 1 : j] : us[r * W + c0 + CPT + 1];
                            v.w = j > 0 ? u[r][j > 0 ? j - 1 : 0] : us[r * W + c0];
                            v.n = r + 1 < H ? u[r + 1 < H ? r + 1 : r][j] : hN[j];
                            v.s = r > 0 ? u[r > 0 ? r - 1 : 0][j] : hS[j];
                            double G_;
                            if (LAW == 1) {
                                const double conv = 0.5 * ((v.e * v.e - v.w * v.w) * P.i2hx + (v.n * v.n - v.s * v.s) * P.i2hy);
                                const double visc = P.m0 * ((v.e - 2.0 * v.c + v.w) * P.ihx2 + (v.n - 2.0 * v.c + v.s) * P.ihy2);
                                G_ = (v.c - pv[r][j]) + tau * (conv - visc);
                            } else {
                                const RJ o = residual_jacobian_raw(P, v, pv[r][j]);
                                G_ = o.G;
                                double* cf = co[LAW == 0 ? r : 0][LAW == 0 ? j : 0];
                                cf[0] = 1.0 / o.aC; cf[1] = o.aE; cf[2] = o.aW; cf[3] = o.aN; cf[4] = o.aS;
                            }
                            bsm(r, j) = x[r][j] - G_;      // b = r^n + du^{n-1}, r^n = -G^n
                            ar2 = fma(G_, G_, ar2);
                            arm = fmax(arm, fabs(G_));
                            if (j == 0 || j == CPT - 1) put_q(qs, r, j, x[r][j], v.c);
                        }
                    }
                    ac(0) += ar2;
                    ac(1) = fmax(ac(1), arm);
                }
                gbar();
                mark(0);
                // ---- S red-black SOR sweeps, one neighbour exchange per half-sweep
                const bool chkl = (n % chk == 0) || n == nt;   // this level's solve residual is measured
                for (int m = 0; m < SW; ++m) {
                    const bool lastm = m == SW - 1 && chkl;
                    #pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        double xs_h[HC], xn_h[HC];
                        #pragma unroll
                        for (int h = 0; h < HC; ++h) xs_h[h] = xn_h[h] = 0.0;
                        if (lastx < 0 && cin) {   // first half-sweep of a slab: the carry's halo rows
                            #pragma unroll
                            for (int h = 0; h < HC; ++h) {
                                if (cs >= 0) xs_h[h] = __ldcg(cin + (size_t)((r0 - 1 + nyu) % nyu) * NXU + c0 + ((PR0 + cc) & 1) + 2 * h);
                                if (cn >= 0) xn_h[h] = __ldcg(cin + (size_t)((r0 + H) % nyu) * NXU + c0 + ((PR0 + H - 1 + cc) & 1) + 2 * h);
                            }
                        }
                        if (lastx >= 0) {
                            const unsigned qn = (unsigned)lastx;
                            LLc hs[HC], hn[HC];
                            #pragma unroll
                            for (int h = 0; h < HC; ++h) {
                                if (cs >= 0) hs[h] = ll_issue(xcell(sx, qn, 1, h));
                                if (cn >= 0) hn[h] = ll_issue(xcell(nxq, qn, 0, h));
                            }
                            #pragma unroll
                            for (int h = 0; h < HC; ++h) {
                                if (cs >= 0) xs_h[h] = ll_take_t(xcell(sx, qn, 1, h), hs[h], qn + 1u, tr[2]);
                                if (cn >= 0) xn_h[h] = ll_take_t(xcell(nxq, qn, 0, h), hn[h], qn + 1u, tr[2]);
                            }
                        }
                        double rs2 = 0.0, rsm = 0.0;
                        // boundary rows first and published at once (the neighbours wait for them), then the interior
                        #pragma unroll
                        for (int i = 0; i < H; ++i) {
                            const int r = i == 0 ? 0 : (i == 1 ? H - 1 : i - 1);
                            #pragma unroll
                            for (int h = 0; h < HC; ++h) {
                                const int j = ((PR0 + r + cc) & 1) + 2 * h;   // compile-time after unrolling
                                const double xo = x[r][j];
                                const double xN = r + 1 < H ? x[r + 1 < H ? r + 1 : r][j] : xn_h[h];
                                const double xS = r > 0 ? x[r > 0 ? r - 1 : 0][j] : xs_h[h];
                                const double bb = bsm(r, j);
                                double xn, dC;
                                if (LAW == 1) {
                                    double tt = bb;
                                    if (j + 1 < CPT) tt = fma(-fma(ax, u[r][j + 1 < CPT ? j + 1 : j], -bx), x[r][j + 1 < CPT ? j + 1 : j], tt);
                                    else tt -= qs[r * W + c0 + CPT + 1];
                                    if (j > 0) tt = fma(-fma(-ax, u[r][j > 0 ? j - 1 : 0], -bx), x[r][j > 0 ? j - 1 : 0], tt);
                                    else tt -= qs[r * W + c0];
                                    const double uNv = r + 1 < H ? u[r + 1 < H ? r + 1 : r][j] : hN[j];
                                    const double uSv = r > 0 ? u[r > 0 ? r - 1 : 0][j] : hS[j];
                                    tt = fma(-fma(ay, uNv, -by), xN, tt);
                                    tt = fma(-fma(-ay, uSv, -by), xS, tt);
                                    xn = fma(omega, fma(tt, invC1, -xo), xo);
                                    dC = aC1;
                                } else {
                                    const double* cf = co[LAW == 0 ? r : 0][LAW == 0 ? j : 0];
                                    const double xE = j + 1 < CPT ? x[r][j + 1 < CPT ? j + 1 : j] : qs[r * W + c0 + CPT + 1];
                                    const double xW = j > 0 ? x[r][j > 0 ? j - 1 : 0] : qs[r * W + c0];
                                    double tt = bb;
                                    tt = fma(-cf[1], xE, tt);
                                    tt = fma(-cf[2], xW, tt);
                                    tt = fma(-cf[3], xN, tt);
                                    tt = fma(-cf[4], xS, tt);
                                    xn = fma(omega, fma(tt, cf[0], -xo), xo);
                                    dC = 1.0 / cf[0];
                                }
                                x[r][j] = xn;
                                if (j == 0 || j == CPT - 1) put_q(qs, r, j, xn, u[r][j]);
                                if (cc == 1 && lastm) {   // residual of a just-updated black point
                                    const double rr = dC * rfac * (xn - xo);
                                    rs2 = fma(rr, rr, rs2);
                                    rsm = fmax(rsm, fabs(rr));
                                }
                            }
                            if (i == (H > 1 ? 1 : 0)) {   // this colour's boundary values: side 0 row 0, side 1 row H-1
                                const unsigned f = qx + 1u;
                                #pragma unroll
                                for (int h = 0; h < HC; ++h) {
                                    if (cs >= 0) ll_put(xcell(myx, qx, 0, h), x[0][((PR0 + cc) & 1) + 2 * h], f);
                                    if (cn >= 0) ll_put(xcell(myx, qx, 1, h), x[H - 1][((PR0 + H - 1 + cc) & 1) + 2 * h], f);
                                }
                            }
                        }
                        if (cc == 1 && lastm) {
                            ac(4) += rs2;
                            ac(5) = fmax(ac(5), rsm);
                        }
                        lastx = (int)qx;
                        ++qx;
                        gbar();
                    }
                }
                mark(1);
                // ---- epilogue: U_{k+1}^n = U_k^n + du^n (du^n stays in x as the next carry)
                {
                    double* Un = S.U + (size_t)((k + 1) % B) * nt * ns + (size_t)(n - 1) * ns;
                    double d2 = 0.0, dm = 0.0;
                    #pragma unroll
                    for (int r = 0; r < H; ++r) {
                        #pragma unroll
                        for (int j = 0; j < CPT; j += 2) {
                            double2 v;
                            v.x = u[r][j] + x[r][j];
                            v.y = u[r][j + 1] + x[r][j + 1];
                            *reinterpret_cast<double2*>(Un + (size_t)(r0 + r) * NXU + c0 + j) = v;
                            d2 = fma(x[r][j], x[r][j], fma(x[r][j + 1], x[r][j + 1], d2));
                            dm = fmax(dm, fmax(fabs(x[r][j]), fabs(x[r][j + 1])));
                            if (r == 0 && cs >= 0) {
                                ll_put(ucell(myu, qu, 0, j), v.x, qu + 1u);
                                ll_put(ucell(myu, qu, 0, j + 1), v.y, qu + 1u);
                            }
                            if (r == H - 1 && cn >= 0) {
                                ll_put(ucell(myu, qu, 1, j), v.x, qu + 1u);
                                ll_put(ucell(myu, qu, 1, j + 1), v.y, qu + 1u);
                            }
                        }
                    }
                    ++qu;
                    ac(2) += d2;
                    ac(3) = fmax(ac(3), dm);
                    if (n == nt && S.carry_out && pass == 0 && p == 0)   // time slab: du_k of the last level
                        #pragma unroll
                        for (int r = 0; r < H; ++r)
                            #pragma unroll
                            for (int j = 0; j < CPT; j += 2)
                                *reinterpret_cast<double2*>(S.carry_out + (size_t)(r0 + r) * NXU + c0 + j) = make_double2(x[r][j], x[r][j + 1]);
                    gbar();                               // every thread's U_{k+1}^n rows are written
                    if (t == 0) {
                        __threadfence_block();
                        lvl_done[p] = n;                  // group p+1 may start level n
                    }
                }
                // ---- a-posteriori residual of the red points after the final black half-sweep (every chk-th level:
                //      it waits for the neighbours' final black rows, one more exchange on this group's chain)
                if (chkl) {
                    const unsigned qn = (unsigned)lastx;
                    double xs_h[HC], xn_h[HC];
                    #pragma unroll
                    for (int h = 0; h < HC; ++h) {
                        xs_h[h] = cs >= 0 ? ll_take(xcell(sx, qn, 1, h), ll_issue(xcell(sx, qn, 1, h)), qn + 1u) : 0.0;
                        xn_h[h] = cn >= 0 ? ll_take(xcell(nxq, qn, 0, h), ll_issue(xcell(nxq, qn, 0, h)), qn + 1u) : 0.0;
                    }
                    double rs2 = 0.0, rsm = 0.0, bb2 = 0.0;
                    #pragma unroll
                    for (int r = 0; r < H; ++r) {
                        #pragma unroll
                        for (int h = 0; h < HC; ++h) {
                            const int j = ((PR0 + r) & 1) + 2 * h;     // red points
                            const double xo = x[r][j];
                            const double xN = r + 1 < H ? x[r + 1 < H ? r + 1 : r][j] : xn_h[h];
                            const double xS = r > 0 ? x[r > 0 ? r - 1 : 0][j] : xs_h[h];
                            double rr = bsm(r, j);
                            if (LAW == 1) {
                                if (j + 1 < CPT) rr -= fma(ax, u[r][j + 1 < CPT ? j + 1 : j], -bx) * x[r][j + 1 < CPT ? j + 1 : j];
                                else rr -= qs[r * W + c0 + CPT + 1];
                                if (j > 0) rr -= fma(-ax, u[r][j > 0 ? j - 1 : 0], -bx) * x[r][j > 0 ? j - 1 : 0];
                                else rr -= qs[r * W + c0];
                                const double uNv = r + 1 < H ? u[r + 1 < H ? r + 1 : r][j] : hN[j];
                                const double uSv = r > 0 ? u[r > 0 ? r - 1 : 0][j] : hS[j];
                                rr -= fma(ay, uNv, -by) * xN + fma(-ay, uSv, -by) * xS + aC1 * xo;
                            } else {
                                const double* cf = co[LAW == 0 ? r : 0][LAW == 0 ? j : 0];
                                const double xE = j + 1 < CPT ? x[r][j + 1 < CPT ? j + 1 : j] : qs[r * W + c0 + CPT + 1];
                                const double xW = j > 0 ? x[r][j > 0 ? j - 1 : 0] : qs[r * W + c0];
                                rr -= cf[1] * xE + cf[2] * xW + cf[3] * xN + cf[4] * xS + xo / cf[0];
                            }
                            rs2 = fma(rr, rr, rs2);
                            rsm = fmax(rsm, fabs(rr));
                        }
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) bb2 = fma(bsm(r, j), bsm(r, j), bb2);
                    }
                    ac(4) += rs2;
                    ac(5) = fmax(ac(5), rsm);
                    ac(6) += bb2;
                }
                mark(3);
                // ---- iteration end: per-CTA partials, the last CTA reduces and decides
                if (n == nt) {
                    double a[NB_NP];
                    #pragma unroll
                    for (int j = 0; j < NB_NP; ++j) {
                        a[j] = ac(j);
                        ac(j) = 0.0;
                    }
                    #pragma unroll
                    for (int j = 0; j < NB_NP; ++j)
                        #pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const double y = __shfl_xor_sync(0xffffffffu, a[j], o);
                            a[j] = nb_is_max(j) ? fmax(a[j], y) : a[j] + y;
                        }
                    if ((t & 31) == 0)
                        #pragma unroll
                        for (int j = 0; j < NB_NP; ++j) red_s[p][t >> 5][j] = a[j];
                    gbar();
                    if (t == 0) {
                        double* hp = S.hpart + ((size_t)k * G + c) * NB_NP;
                        for (int j = 0; j < NB_NP; ++j) {
                            double v = red_s[p][0][j];
                            for (int w = 1; w < NW; ++w) v = nb_is_max(j) ? fmax(v, red_s[p][w][j]) : v + red_s[p][w][j];
                            hp[j] = v;
                        }
                        __threadfence();
                        s_last[p] = atomicAdd(S.arrive + k, 1u) == (unsigned)(G - 1);
                    }
                    gbar();
                    if (s_last[p] && t < 32) {   // last CTA of iteration k: reduce over CTAs, decide
                        __threadfence();
                        double g4[NB_NP] = {0, 0, 0, 0, 0, 0, 0};
                        for (int gg = t; gg < G; gg += 32) {
                            const double* hp = S.hpart + ((size_t)k * G + gg) * NB_NP;
                            #pragma unroll
                            for (int j = 0; j < NB_NP; ++j) {
                                const double v = __ldcg(hp + j);
                                g4[j] = nb_is_max(j) ? fmax(g4[j], v) : g4[j] + v;
                            }
                        }
                        #pragma unroll
                        for (int j = 0; j < NB_NP; ++j)
                            #pragma unroll
                            for (int o = 16; o > 0; o >>= 1) {
                                const double y = __shfl_xor_sync(0xffffffffu, g4[j], o);
                                g4[j] = nb_is_max(j) ? fmax(g4[j], y) : g4[j] + y;
                            }
                        if (t == 0) {
                            const double Ntot = (double)ns * (double)nt;
                            S.hist[4 * k + 0] = sqrt(g4[0] / Ntot);
                            S.hist[4 * k + 1] = g4[1];
                            S.hist[4 * k + 2] = sqrt(g4[2] / Ntot);
                            S.hist[4 * k + 3] = g4[3];
                            if (S.linres) {
                                S.linres[2 * k + 0] = g4[6] > 0.0 ? sqrt(g4[4] / g4[6]) : 0.0;
                                S.linres[2 * k + 1] = g4[5];
                            }
                            const double dn = S.stop_norm ? sqrt(g4[2] / Ntot) : g4[3];
                            double prev = INFINITY;
                            if (k >= 1) {
                                while (*((volatile unsigned*)(S.decided + k - 1)) == 0) __nanosleep(64);
                                __threadfence();
                                prev = S.stop_norm ? __ldcg(S.hist + 4 * (k - 1) + 2) : __ldcg(S.hist + 4 * (k - 1) + 3);
                            }
                            int st = 2;
                            bool finite = true;
                            #pragma unroll
                            for (int j = 0; j < NB_NP; ++j) finite = finite && isfinite(g4[j]);
                            if (!finite) st = -5;
                            else if (dn <= S.newton_tol) st = 0;
                            else if (k >= 1 && dn > 0.5 * prev && dn <= 1e3 * S.newton_tol) st = 1;
                            else if (k + 1 >= S.newton_max) st = -4;
                            __threadfence();
                            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(S.decided + k), "r"((unsigned)(16 + st)) : "memory");
                        }
                    }
                    mark(4);
                }
            }
            // ---- pass end: every group done; wait for the decisions of this pass's iterations
            __syncthreads();
            const int kl = min(pass * D + D, S.newton_max) - 1;
            if (threadIdx.x == 0) {
                unsigned v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(S.decided + kl) : "memory");
                    if (v) break;
                    __nanosleep(128);
                }
                int st = 2, kf = -1;
                for (int kk = pass * D; kk <= kl; ++kk) {
                    const int sk = (int)*((volatile unsigned*)(S.decided + kk)) - 16;
                    if (sk != 2) { st = sk; kf = kk + 1; break; }
                }
                s_dec[0] = st;
                s_dec[1] = kf;
                for (int i = 0; i < DM; ++i) lvl_done[i] = 0;
            }
            __syncthreads();
            mark(5);
            const int st = s_dec[0], kf = s_dec[1];
            if (st != 2) {
                const double* Uf = S.U + (size_t)(kf % B) * nt * ns;
                if (S.u_out)
                    for (int i = threadIdx.x; i < nt * H * (NXU / 2); i += NT) {
                        const int n = i / (H * (NXU / 2)), rr = (i / (NXU / 2)) % H, cc2 = i % (NXU / 2);
                        const size_t o = (size_t)n * ns + (size_t)(r0 + rr) * NXU + 2 * cc2;
                        *reinterpret_cast<double2*>(S.u_out + o) = ldcg2(Uf + o);
                    }
                if (trace && t == 0) {
                    tr[7] = clock64() - t_start;
                    for (int i = 0; i < NB_TR; ++i) S.trace[(size_t)c * NB_TR + i] = (unsigned long long)tr[i];
                }
                if (c == 0 && threadIdx.x == 0) {
                    S.info[0] = kf;
                    S.info[1] = st;
                    if (S.stats) {
                        S.stats[0] = levels; S.stats[1] = (long long)SW;
                        S.stats[2] = D; S.stats[3] = G; S.stats[4] = levels * SW; S.stats[5] = 0;
                    }
                }
                return;
            }
        }
    }
};

// Strip height h in {HB, HB + 1} and the parity of the first own row select the compile-time body.
template <int HB, int LAW, int NXU, int DM, int CPT>
__global__ void __launch_bounds__(DM * (NXU / CPT), 1) k_newton_nb(const NbParams S) {
    extern __shared__ double sm[];
    using E = NbEngine<HB, LAW, NXU, DM, CPT>;
    const int G = S.G, c = blockIdx.x;
    const int hb = S.P.nyu / G, hr = S.P.nyu % G;
    const int h = hb + (c < hr ? 1 : 0);
    const int pr0 = (c * hb + min(c, hr)) & 1;
    if (h == HB) {
        if (pr0) E::template run<HB, 1>(S, sm); else E::template run<HB, 0>(S, sm);
    } else {
        if (pr0) E::template run<HB + 1, 1>(S, sm); else E::template run<HB + 1, 0>(S, sm);
    }
}

}  // namespace pit
