// pit_newton_col.cuh — the COLUMN-BLOCKED on-chip engine (included by pit_kernels.cu after the strip engine).
//
// Same method, schedule, barriers, reductions and stop rule as k_newton_onchip; only the point layout of a
// strip changes.  A thread owns one grid COLUMN of (a sub-strip of) its CTA's rows, so
//   * the N/S neighbours of every matvec come from the thread's own registers (the register-blocked
//     5-point stencil), only E/W neighbours go through shared memory (2 loads + 1 store per point);
//   * u^n of the strip (one halo row each side) is staged once per step in shared memory and the
//     coefficients are recomputed from it (registers are kept for the Krylov vectors: 128 per thread);
//   * r/s and p are registers; x, r^0 (= b~ - A~ x0), v, t (and 1/a_C for the general law) are shared.
// Applies when nx (unknowns per row) is 256 or 512: 512 threads = 1 or 2 column groups; a column group
// splits the strip rows in two sub-strips whose boundary rows are exchanged through the shared operand.
#pragma once

namespace pit {

constexpr int BLOCK3 = 512;
constexpr int HALO_ROW = 512;                          // doubles per published row (nx <= 512)
constexpr int HALO_CTA = 2 * 6 * HALO_ROW;             // per CTA: {top, bottom} x {s, t, p, v, r, v2}
enum { HV_S = 0, HV_T = 1, HV_P = 2, HV_V = 3, HV_R = 4, HV_V2 = 5 };

// NXU (unknowns per row, 256 or 512) is a template parameter: the row pitch W and the column-group split are then
// compile-time constants, so every shared-memory offset of the stencil loops folds into an immediate (with a
// runtime pitch the 128-register budget forced the compiler to rematerialise the index arithmetic in every loop).
template <int V> struct IC { static constexpr int value = V; };   // compile-time strip height tag (0 = run time)

template <int RMAX, bool TRACE, int LAW, int NXU>
__global__ void __launch_bounds__(BLOCK3, 1) k_newton_col(SolveParams S) {
    extern __shared__ double smem[];
    const Prob P = S.P;
    const long long ns = P.ns;
    constexpr int nxu = NXU;
    const int nyu = P.nyu;
    const int G = S.G, g = blockIdx.x, tid = threadIdx.x;
    constexpr int W = nxu + 4;                         // row pitch of u_s / op_s: data at +2 (16-byte aligned rows)
    const int HM = S.hmax;
    double* const u_s = smem;                          // [HM+2][W] u of the strip rows + halo rows (+ ring / wrap columns)
    double* const op_s = u_s + (HM + 2) * W;           // [HM+2][W] matvec operand (E/W exchange, halo rows)
    double* const v_s = op_s + (HM + 2) * W;           // [RMAX][BLOCK3]
    double* const t_s = v_s + RMAX * BLOCK3;           // [RMAX][BLOCK3]
    double* const x_s = t_s + RMAX * BLOCK3;           // [RMAX][BLOCK3] BiCGSTAB iterate (-> du^n)
    double* const bt_s = x_s + RMAX * BLOCK3;          // [RMAX][BLOCK3] shadow residual r^0 (and b~)
    double* const ci_s = bt_s + RMAX * BLOCK3;         // [RMAX][BLOCK3] 1/a_C (LAW 0 only)
    __shared__ int sS[MAXK];
    __shared__ double red[NWARP2 * NPART];
    __shared__ double s_hp_big[4 * GMAX2];
    __shared__ double s_red[8];                        // bar_sync_reduce results (N <= 5)
    __shared__ double lacc[MAXD][4];                   // this CTA's norm partials per pipeline slot, summed over levels
    __shared__ double prevmax_s;
    // Newton norms of the pipeline slot e_slot per thread (sum r^2, max |r|, sum du^2, max |du|): reduced over the
    // CTA only when the slot's iteration finishes or the CTA changes slot, not in every step
    __shared__ double s_e[4][BLOCK3];
    s_e[0][tid] = 0.0; s_e[1][tid] = 0.0; s_e[2][tid] = 0.0; s_e[3][tid] = 0.0;
    // this CTA's share of a step with A active pairs (A = 1..MAXD), computed once: pair me, its CTA block [g0, g1),
    // the strip rows [r0, r1) and the CTAs owning the halo rows r0 - 1 / r1 (integer divisions kept off the step path)
    __shared__ int s_asg[MAXD + 1][8];
    __shared__ unsigned char s_kD[MAXK + 1], s_kB[MAXK + 1];   // k mod D (pipeline slot), k mod B (iterate buffer)
    for (int k = tid; k <= MAXK; k += BLOCK3) { s_kD[k] = (unsigned char)(k % S.D); s_kB[k] = (unsigned char)(k % S.B); }
    if (tid < MAXD) {
        const int A = tid + 1;
        int me = 0;
        while (me + 1 < A && (me + 1) * G / A <= g) ++me;                 // 32-bit: G * A < 2^31
        const int g0 = me * G / A, g1 = (me + 1) * G / A, C = g1 - g0, c = g - g0;
        const int r0 = c * nyu / C, r1 = (c + 1) * nyu / C;                // 32-bit: C * nyu < 2^31
        const int trow = r0 == 0 ? nyu - 1 : r0 - 1, brow = r1 == nyu ? 0 : r1;
        int* t = s_asg[A];
        t[0] = me; t[1] = g0; t[2] = g1; t[3] = r0; t[4] = r1;
        t[5] = g0 + ((trow + 1) * C - 1) / nyu;                             // owner of row r0 - 1 in the pair
        t[6] = g0 + ((brow + 1) * C - 1) / nyu;                             // owner of row r1
    }
    if (tid == 0) {
        const int D = S.D;
        for (int k = 0; k < S.newton_max; ++k) {
            int st = k == 0 ? 1 : sS[k - 1] + 1;
            if (k >= D && sS[k - D] + P.nt > st) st = sS[k - D] + P.nt;
            sS[k] = st;
        }
        prevmax_s = INFINITY;
    }
    if (tid < MAXD * 4) lacc[tid / 4][tid % 4] = 0.0;
    for (int i = tid; i < (HM + 2) * W; i += BLOCK3) op_s[i] = 0.0;   // Dirichlet: the dropped columns stay 0
    __syncthreads();

    unsigned ep = 0;
    int e_slot = -1;
    unsigned hi[2] = {0u, 0u};
    long long prof[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long t_last = clock64();
    auto flush_prof = [&]() {
        if (TRACE && tid == 0)
            for (int j = 0; j < 13; ++j) {
                atomicAdd(S.trace + j, (unsigned long long)prof[j]);
                S.trace[13 + 13 * g + j] = (unsigned long long)prof[j];    // per-CTA copy (tools/skew_run.py)
            }
    };
    const int newton_max = S.mode == 0 ? S.newton_max : 1;
    int set = 0, klo = 0, last_done = -1;
    long long total_inner = 0;
    const double rtol2 = S.lin_rtol * S.lin_rtol;
    const double atol2 = S.lin_atol * S.lin_atol * (double)P.ns;     // lin_atol bounds the RMS residual
    constexpr int Gr = BLOCK3 / nxu;                   // column groups (1 or 2)
    const int col = Gr == 1 ? tid : tid % nxu, grp = Gr == 1 ? 0 : tid / nxu;   // Gr = 1: R0 = 0 at compile time
    // E / W neighbours in the u_s / op_s rows: the next column, or the periodic wrap inside the row; Dirichlet
    // edges read the halo columns (u_s: the ring, staged every step; op_s: zeros, written once below)
    const int dE = (P.bc == 1 && col == nxu - 1) ? -(nxu - 1) : 1;
    const int dW = (P.bc == 1 && col == 0) ? (nxu - 1) : -1;
    const double ci_const = 1.0 / (1.0 + 2.0 * P.dt * P.m0 * (P.ihx2 + P.ihy2));   // LAW 1: a_C is constant

    for (int step = 1;; ++step) {
        while (klo < newton_max && step > sS[klo] + P.nt - 1) ++klo;
        // the active iterations are consecutive: k = kbase + a for pair a < A (no local array)
        int A = 0;
        for (int k = klo; k < newton_max && A < MAXD && sS[k] <= step; ++k) ++A;
        const int kbase = S.mode == 1 ? 0 : klo;
        if (S.mode == 1) A = S.nb;
        const int* const asg = s_asg[A];
        const int me = asg[0], g0 = asg[1], g1 = asg[2];
        const int kme = kbase + me;
        const int n = S.mode == 1 ? S.blev[me] : step - sS[kme] + 1;
        const int slot = s_kD[kme];
        const int buf = s_kB[kme], nbuf = s_kB[kme + 1];
        const Slot sl = slot_at(S.slotmem, ns, slot);
        double* const pX = sl.x;
        const int c = g - g0;
        const int r0 = asg[3], r1 = asg[4];
        const int h = r1 - r0;
        const double* Ulev = S.mode == 1 ? S.U + (long long)(n - 1) * ns : S.U + ((long long)buf * P.nt + (n - 1)) * ns;
        const double* uprev = n == 1 ? S.u0 : Ulev - ns;
        const double* ringn = S.ring ? S.ring + (long long)(n - 1) * P.ring_len : nullptr;
        double* Unew = S.mode == 1 ? nullptr : S.U + ((long long)nbuf * P.nt + (n - 1)) * ns;
        // this thread's sub-strip of rows [R0, R1) (strip-local), column col
        const int R0 = (grp * h) >> (Gr - 1), R1 = ((grp + 1) * h) >> (Gr - 1);   // Gr = 1 or 2
        const int hs = R1 - R0;
        const bool own_top = R0 == 0, own_bot = R1 == h;          // sub-strip touches the CTA's halo rows
        const bool top_valid = P.bc == 1 || r0 > 0, bot_valid = P.bc == 1 || r1 < nyu;
        // published boundary rows: own {top, bottom} slots, and the bottom slot of the CTA owning row r0 - 1 /
        // the top slot of the CTA owning row r1 (owner of row x in the pair: ((x + 1) C - 1) / nyu)
        double* const hb_own = S.halo + (long long)g * HALO_CTA + col;
        const double* const hb_S = S.halo + (long long)asg[5] * HALO_CTA + 6 * HALO_ROW + col;
        const double* const hb_N = S.halo + (long long)asg[6] * HALO_CTA + col;
        // halo values of the next phase, loaded right after the barrier that publishes them (bar_sync_reduce_pre):
        // phase 2 reads r, v2 -> hv[0], hv[1] (S) and hv[4], hv[5] (N); phase 1 reads s, t, p, v -> hv[0..3], hv[4..7]
        double hv[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const bool hasS = hs > 0 && own_top && top_valid, hasN = hs > 0 && own_bot && bot_valid;
        auto pre2 = [&]() {
            if (hasS) { hv[0] = __ldcg(hb_S + HV_R * HALO_ROW); hv[1] = __ldcg(hb_S + HV_V2 * HALO_ROW); }
            if (hasN) { hv[4] = __ldcg(hb_N + HV_R * HALO_ROW); hv[5] = __ldcg(hb_N + HV_V2 * HALO_ROW); }
        };
        auto pre1 = [&]() {
            if (hasS) {
                hv[0] = __ldcg(hb_S + HV_S * HALO_ROW); hv[1] = __ldcg(hb_S + HV_T * HALO_ROW);
                hv[2] = __ldcg(hb_S + HV_P * HALO_ROW); hv[3] = __ldcg(hb_S + HV_V * HALO_ROW);
            }
            if (hasN) {
                hv[4] = __ldcg(hb_N + HV_S * HALO_ROW); hv[5] = __ldcg(hb_N + HV_T * HALO_ROW);
                hv[6] = __ldcg(hb_N + HV_P * HALO_ROW); hv[7] = __ldcg(hb_N + HV_V * HALO_ROW);
            }
        };
        auto pub = [&](int R, int v, double val) {     // row R of the strip is a boundary row: publish
            if (R == 0) hb_own[v * HALO_ROW] = val;
            if (R == h - 1) hb_own[(6 + v) * HALO_ROW] = val;
        };
        const long long qc = (long long)(r0 + R0) * nxu + col;      // global index of the sub-strip's first point
        auto q_of = [&](int r) { return qc + (long long)r * nxu; };
        auto sidx = [&](int r) { return (R0 + r + 1) * W + col + 2; };   // op_s index of own point r
        auto uidx = [&](int r) { return (R0 + r + 1) * W + col + 2; };   // u_s index of own point r

        auto flush_e = [&]() {                         // CTA-uniform: s_e -> lacc[e_slot]
            double a4[4] = {s_e[0][tid], s_e[2][tid], s_e[1][tid], s_e[3][tid]};
            s_e[0][tid] = 0.0; s_e[1][tid] = 0.0; s_e[2][tid] = 0.0; s_e[3][tid] = 0.0;
            block_reduce2<2, 2, false>(a4, red);
            if (tid == 0) {
                lacc[e_slot][0] += a4[0];
                lacc[e_slot][1] = fmax(lacc[e_slot][1], a4[2]);
                lacc[e_slot][2] += a4[1];
                lacc[e_slot][3] = fmax(lacc[e_slot][3], a4[3]);
                if (!isfinite(a4[1])) atomicOr(&S.bs->err, 1u);   // a non-finite du makes the sum non-finite
            }
        };
        if (S.mode == 0 && slot != e_slot) {           // CTA-uniform: a new slot for this CTA
            if (e_slot >= 0) flush_e();
            e_slot = slot;
        }
        double sr[RMAX], pp[RMAX];
        auto X = [&](int r) -> double& { return x_s[r * BLOCK3 + tid]; };
        auto BT = [&](int r) -> double& { return bt_s[r * BLOCK3 + tid]; };

        PMARK(11);
        // ---- prologue -----------------------------------------------------------------------------
        // Fused with iteration 0's first half: the residual + Jacobian diagonal (kernel a), the carry,
        // r0 = b~ - A~ x0 (x0 = du^{n-1}), and v0 = A~ p0 with p0 = r0 are all formed before the first grid
        // barrier.  r0 on the two halo rows (needed by v0) is recomputed redundantly by the edge threads from
        // u (two rows deep), u^{n-1} and the carry, all of which are inputs of this step.
        const bool x0c = S.x0carry && S.mode == 0 && n > 1;
        // stage u of the strip, rows -1 .. h, in 16-byte pieces (cp.async.cg: every thread copies column pairs of
        // whole rows, independent of the column it owns; periodic rows wrap).  Dirichlet ring rows and the E/W halo
        // columns (the ring) are written with ordinary stores.
        {
            constexpr int lg = nxu == 512 ? 8 : 7, half = nxu >> 1;    // column pairs per row (nxu = 512 or 256)
            const int npairs = (h > 0 ? h + 2 : 0) << lg;
            for (int i = tid; i < npairs; i += BLOCK3) {
                const int rr = (i >> lg) - 1, cpair = i & (half - 1);
                int gr = r0 + rr;
                if (P.bc == 1) gr = gr < 0 ? gr + nyu : (gr >= nyu ? gr - nyu : gr);
                else if (gr < 0 || gr >= nyu) continue;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(u_s + (rr + 1) * W + 2 + 2 * cpair);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(Ulev + (long long)gr * nxu + 2 * cpair)
                             : "memory");
            }
            // mode 0: the own rows of u^{n-1} -> t_s and of the carry du^{n-1} -> x_s (= x0), same 16-byte pieces,
            // in the [row of the column group][thread] layout of the strip vectors
            if (S.mode == 0 && h > 0) {
                const bool cpx = n > 1;
                const int nq = h << lg, hh = h >> 1;
                for (int i = tid; i < nq; i += BLOCK3) {
                    const int j = i >> lg, cpair = i & (half - 1);             // strip row j
                    const int gsel = (Gr == 2 && j >= hh) ? 1 : 0;
                    const int soff = (j - (gsel ? hh : 0)) * BLOCK3 + gsel * nxu + 2 * cpair;
                    const long long q = (long long)(r0 + j) * nxu + 2 * cpair;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(t_s + soff)),
                                 "l"(uprev + q) : "memory");
                    if (cpx)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(x_s + soff)),
                                     "l"(pX + q) : "memory");
                }
            }
            if (P.bc != 1 && hs > 0) {
                for (int r = -1; r <= hs; ++r) {
                    const int ui = uidx(r), gr = r0 + R0 + r;
                    if (gr < 0 || gr >= nyu) u_s[ui] = node_ext(P, Ulev, ringn, gr, col);
                    if (col == 0) u_s[ui - 1] = node_ext(P, Ulev, ringn, gr, -1);
                    if (col == nxu - 1) u_s[ui + 1] = node_ext(P, Ulev, ringn, gr, nxu);
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        PMARK(12);
        auto rowq = [&](int gr) -> long long {                    // global index of (row gr, col), wrapped
            gr = gr < 0 ? gr + nyu : (gr >= nyu ? gr - nyu : gr);
            return (long long)gr * nxu + col;
        };
        auto carry_at = [&](int gr) -> double {                   // du^{n-1} at (gr, col); 0 outside (Dirichlet)
            if (S.mode == 1 || n == 1 || (P.bc != 1 && (gr < 0 || gr >= nyu))) return 0.0;
            return __ldcg(pX + rowq(gr));
        };
        if (S.mode == 1) {
            #pragma unroll
            for (int r = 0; r < RMAX; ++r) sr[r] = r < hs ? __ldcg(S.bptr[me] + q_of(r)) : 0.0;
        }
        // halo-point inputs: S halo (row r0-1) and N halo (row r1) of this column
        double hS_u2 = 0.0, hS_up = 0.0, hS_x = 0.0, hS_x2 = 0.0, hS_b = 0.0;
        double hN_u2 = 0.0, hN_up = 0.0, hN_x = 0.0, hN_x2 = 0.0, hN_b = 0.0;
        if (hasS) {
            hS_u2 = node_ext(P, Ulev, ringn, r0 - 2, col);
            if (S.mode == 1) hS_b = __ldcg(S.bptr[me] + rowq(r0 - 1));
            else hS_up = (n == 1 ? S.u0 : uprev)[rowq(r0 - 1)];
            hS_x = carry_at(r0 - 1);                                     // carry (enters b~)
            hS_x2 = x0c ? carry_at(r0 - 2) : 0.0;                        // x0 one row further
        }
        if (hasN) {
            hN_u2 = node_ext(P, Ulev, ringn, r1 + 1, col);
            if (S.mode == 1) hN_b = __ldcg(S.bptr[me] + rowq(r1));
            else hN_up = (n == 1 ? S.u0 : uprev)[rowq(r1)];
            hN_x = carry_at(r1);
            hN_x2 = x0c ? carry_at(r1 + 1) : 0.0;
        }
        // merged first iteration (S.merge): r0 two rows deep, i.e. at rows r0 - 2 and r1 + 1 (periodic): their u
        // E/W, the row beyond, u^{n-1}, and x0 (= the carry) E/W and beyond, loaded while the staging lands
        const bool mrg = S.merge != 0;                     // grid-uniform (host: mode 0, periodic, strips >= 3 rows)
        double fS[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, fN[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (mrg) {
            auto at = [&](const double* base, int gr, int gc) -> double {
                gr = gr < 0 ? gr + nyu : (gr >= nyu ? gr - nyu : gr);
                gc = gc < 0 ? gc + nxu : (gc >= nxu ? gc - nxu : gc);
                return __ldcg(base + (long long)gr * nxu + gc);
            };
            const bool cx = n > 1;
            if (hasS) {
                fS[0] = at(Ulev, r0 - 2, col + 1); fS[1] = at(Ulev, r0 - 2, col - 1); fS[2] = at(Ulev, r0 - 3, col);
                fS[3] = at(uprev, r0 - 2, col);
                if (cx) { fS[4] = at(pX, r0 - 2, col + 1); fS[5] = at(pX, r0 - 2, col - 1); fS[6] = at(pX, r0 - 3, col); }
            }
            if (hasN) {
                fN[0] = at(Ulev, r1 + 1, col + 1); fN[1] = at(Ulev, r1 + 1, col - 1); fN[2] = at(Ulev, r1 + 2, col);
                fN[3] = at(uprev, r1 + 1, col);
                if (cx) { fN[4] = at(pX, r1 + 1, col + 1); fN[5] = at(pX, r1 + 1, col - 1); fN[6] = at(pX, r1 + 2, col); }
            }
        }
        PMARK(7);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        // r0 = b~ - A~ x0 at a far halo row from its stencil values (u, u^{n-1}, carry; x0 = carry)
        auto r0_far = [&](double uc, double ue, double uw, double un, double us, double up, double xc, double xe,
                          double xw, double xn, double xs) -> double {
            const Vals v = {uc, ue, uw, un, us};
            double G, aC;
            res_diag<LAW>(P, v, up, G, aC);
            const double ci = LAW == 1 ? ci_const : 1.0 / aC;
            const double bt = (-G + (n == 1 ? 0.0 : xc)) * ci;
            if (!x0c) return bt;
            const Off o = offdiag_law<LAW>(P, v);
            return bt - (xc + ci * (o.e * xe + o.w * xw + o.n * xn + o.s * xs));
        };
        double rfS = 0.0, rfN = 0.0;                       // r0 at rows r0 - 2 and r1 + 1
        if (mrg && hasS)
            rfS = r0_far(hS_u2, fS[0], fS[1], u_s[uidx(-1)], fS[2], fS[3], hS_x2, fS[4], fS[5], hS_x, fS[6]);
        if (mrg && hasN)
            rfN = r0_far(hN_u2, fN[0], fN[1], fN[2], u_s[uidx(hs)], fN[3], hN_x2, fN[4], fN[5], fN[6], hN_x);
        if (S.mode == 0) {
            #pragma unroll
            for (int r = 0; r < RMAX; ++r) {
                sr[r] = (r < hs && n > 1) ? X(r) : 0.0;
            }
        }
        PMARK(8);
        // operand accessors: N/S from registers inside the sub-strip, shared memory across the column-group
        // boundary, the halo register across the CTA boundary; E/W from shared memory
        auto opS = [&](const double (&o)[RMAX], int r, double haloS) -> double {
            if (r > 0) return o[r - 1];
            return own_top ? haloS : op_s[sidx(r) - W];
        };
        auto opNh = [&](const double (&o)[RMAX], int r, double haloN, int H) -> double {   // H = hs
            if (r + 1 < H) return o[r + 1];
            return own_bot ? haloN : op_s[sidx(r) + W];
        };
        // the hot loops run with the strip height as a compile-time constant when it is RMAX or RMAX - 1 (every CTA
        // of a pair differs by at most one row); the guards of the unrolled loops then fold away.  Only with one
        // column group is hs CTA-uniform (the bodies contain __syncthreads), else it stays a run-time value.
        auto with_hs = [&](auto&& body) {
            if (Gr == 1 && hs == RMAX) body(IC<RMAX>{});
            else if (Gr == 1 && hs == RMAX - 1) body(IC<RMAX - 1>{});
            else body(IC<0>{});
        };
        auto put_op_at = [&](int si, double val) {
            op_s[si] = val;
        };
        auto put_op = [&](int r, double val) { put_op_at(sidx(r), val); };
        auto coef = [&](int r) -> Off {
            const int ui = uidx(r);
            const Vals uv = {u_s[ui], u_s[ui + dE], u_s[ui + dW], u_s[ui + W], u_s[ui - W]};
            return offdiag_law<LAW>(P, uv);
        };
        auto cinv = [&](int r) -> double { return LAW == 1 ? ci_const : ci_s[r * BLOCK3 + tid]; };
        double hS_r0 = 0.0, hN_r0 = 0.0;       // r0 = p0 on the halo rows
        {
            double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // sum r0^2, sum r^2, sum b~^2, sum r0 v0 | max |r|
            double am[4] = {0.0, 0.0, 0.0, 0.0};      // merged: (v0,v0), (r0,w0), (v0,w0), (w0,w0)
            with_hs([&](auto tag) {
                constexpr int HC = decltype(tag)::value;
                const int H = HC ? HC : hs, HH = (HC && Gr == 1) ? HC : h;
                #pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    pp[r] = 0.0;
                    if (r >= H) continue;
                    const int ui = uidx(r);
                    const Vals v = {u_s[ui], u_s[ui + dE], u_s[ui + dW], u_s[ui + W], u_s[ui - W]};
                    double G, aC;
                    res_diag<LAW>(P, v, S.mode == 0 ? t_s[r * BLOCK3 + tid] : 0.0, G, aC);   // u^{n-1} (staged)
                    double rhs;
                    if (S.mode == 1) {
                        rhs = sr[r];
                    } else {
                        const double res = -G;
                        a[1] += res * res;
                        a[4] = fmax(a[4], fabs(res));
                        rhs = res + sr[r];                 // r^n + du^{n-1}  (row n of Eq. 7)
                    }
                    const double ci = LAW == 1 ? ci_const : 1.0 / aC;
                    if (LAW != 1) ci_s[r * BLOCK3 + tid] = ci;
                    const double x0 = x0c ? sr[r] : 0.0;
                    if (!x0c) X(r) = 0.0;                  // x0c: x_s already holds x0 = du^{n-1} (staged)
                    sr[r] = rhs * ci;                      // b~ (r0 once the x0 matvec is subtracted)
                    a[2] += sr[r] * sr[r];
                    pp[r] = x0;
                    put_op(r, x0);
                }
                // b~ - diag part on the halo points (u stencil: own column rows from u_s, the far row in a register)
                double hS_ci = 0.0, hN_ci = 0.0, hS_bt = 0.0, hN_bt = 0.0;
                Off hS_o = {0.0, 0.0, 0.0, 0.0}, hN_o = {0.0, 0.0, 0.0, 0.0};
                if (hasS) {
                    const int ui = uidx(-1);
                    const Vals v = {u_s[ui], u_s[ui + dE], u_s[ui + dW], u_s[ui + W], hS_u2};
                    double G, aC;
                    res_diag<LAW>(P, v, hS_up, G, aC);
                    hS_ci = LAW == 1 ? ci_const : 1.0 / aC;
                    hS_bt = ((S.mode == 1 ? hS_b : -G + (n == 1 ? 0.0 : hS_x))) * hS_ci;
                    hS_o = offdiag_law<LAW>(P, v);
                    put_op_at(sidx(-1), x0c ? hS_x : 0.0);
                }
                if (hasN) {
                    const int ui = uidx(H);
                    const Vals v = {u_s[ui], u_s[ui + dE], u_s[ui + dW], hN_u2, u_s[ui - W]};
                    double G, aC;
                    res_diag<LAW>(P, v, hN_up, G, aC);
                    hN_ci = LAW == 1 ? ci_const : 1.0 / aC;
                    hN_bt = ((S.mode == 1 ? hN_b : -G + (n == 1 ? 0.0 : hN_x))) * hN_ci;
                    hN_o = offdiag_law<LAW>(P, v);
                    put_op_at(sidx(H), x0c ? hN_x : 0.0);
                }
                PMARK(9);
                __syncthreads();                           // op_s holds x0 on own rows + halo rows
                // r0 = b~ - A~ x0 on own points and on the halo points
                #pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    if (r >= H || !x0c) continue;
                    const int si = sidx(r);
                    const Off o = coef(r);
                    sr[r] -= pp[r] + cinv(r) * (o.e * op_s[si + dE] + o.w * op_s[si + dW] + o.n * opNh(pp, r, hN_x, H) +
                                                o.s * opS(pp, r, hS_x));     // x0c: hN_x/hS_x = x0 on the halo rows
                }
                if (hasS) {
                    const int si = sidx(-1);
                    hS_r0 = hS_bt - (x0c ? hS_x + hS_ci * (hS_o.e * op_s[si + dE] + hS_o.w * op_s[si + dW] +
                                                            hS_o.n * (H > 0 ? pp[0] : 0.0) + hS_o.s * hS_x2)
                                         : 0.0);
                }
                if (hasN) {
                    const int si = sidx(H);
                    double xN = 0.0;                       // x0 at the last own row (the halo point's S neighbour)
                    #pragma unroll
                    // (a select chain, not pp[hs - 1]: a dynamic index would move pp to local memory for the whole kernel)
                    #pragma unroll
                    for (int r = 0; r < RMAX; ++r) xN = fma(r == H - 1 ? 1.0 : 0.0, pp[r], xN);
                    hN_r0 = hN_bt - (x0c ? hN_x + hN_ci * (hN_o.e * op_s[si + dE] + hN_o.w * op_s[si + dW] +
                                                            hN_o.n * hN_x2 + hN_o.s * xN)
                                         : 0.0);
                }
                __syncthreads();                           // all reads of x0 done: op_s <- p0 = r0
                #pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    if (r >= H) continue;
                    BT(r) = sr[r];                         // r0, and the BiCGSTAB shadow vector r^0 = r0
                    pp[r] = sr[r];                         // p0 = r0
                    a[0] += sr[r] * sr[r];
                    put_op(r, sr[r]);
                }
                if (mrg) {                                 // r0 on the halo rows: E/W operands of v0 there
                    if (hasS) put_op_at(sidx(-1), hS_r0);
                    if (hasN) put_op_at(sidx(H), hN_r0);
                }
                __syncthreads();
                // v0 = A~ p0; publish r0, v0 of the boundary rows (the halo of phase 2)
                #pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    if (r >= H) continue;
                    const int si = sidx(r);
                    const Off o = coef(r);
                    const double vv = pp[r] + cinv(r) * (o.e * op_s[si + dE] + o.w * op_s[si + dW] + o.n * opNh(pp, r, hN_r0, H) +
                                                         o.s * opS(pp, r, hS_r0));
                    v_s[r * BLOCK3 + tid] = vv;
                    a[3] += sr[r] * vv;
                    am[0] += vv * vv;
                    const int R = R0 + r;
                    if (R == 0 || R == HH - 1) { pub(R, HV_R, sr[r]); pub(R, HV_V2, vv); }
                }
                if (mrg) {
                    // merged first iteration: v0 on the halo rows (r0 two rows deep), then w0 = A~ v0 on own rows, so
                    // that every dot product of the first iteration is a polynomial in alpha of one reduction
                    double v0S = 0.0, v0N = 0.0;
                    if (hasS) {
                        const int si = sidx(-1);
                        v0S = hS_r0 + hS_ci * (hS_o.e * op_s[si + dE] + hS_o.w * op_s[si + dW] + hS_o.n * sr[0] +
                                               hS_o.s * rfS);
                    }
                    if (hasN) {
                        const int si = sidx(H);
                        double rl = 0.0;                   // r0 at the last own row (select chain, no dynamic index)
                        #pragma unroll
                        for (int r = 0; r < RMAX; ++r) rl = fma(r == H - 1 ? 1.0 : 0.0, sr[r], rl);
                        v0N = hN_r0 + hN_ci * (hN_o.e * op_s[si + dE] + hN_o.w * op_s[si + dW] + hN_o.n * rfN +
                                               hN_o.s * rl);
                    }
                    __syncthreads();                       // all reads of r0 in op_s done
                    #pragma unroll
                    for (int r = 0; r < RMAX; ++r) {
                        if (r >= H) continue;
                        pp[r] = v_s[r * BLOCK3 + tid];
                        put_op(r, pp[r]);
                    }
                    if (hasS) put_op_at(sidx(-1), v0S);
                    if (hasN) put_op_at(sidx(H), v0N);
                    __syncthreads();
                    #pragma unroll
                    for (int r = 0; r < RMAX; ++r) {
                        if (r >= H) continue;
                        const int si = sidx(r);
                        const Off o = coef(r);
                        const double w0 = pp[r] + cinv(r) * (o.e * op_s[si + dE] + o.w * op_s[si + dW] +
                                                             o.n * opNh(pp, r, v0N, H) + o.s * opS(pp, r, v0S));
                        t_s[r * BLOCK3 + tid] = w0;
                        am[1] += sr[r] * w0; am[2] += pp[r] * w0; am[3] += w0 * w0;
                        const int R = R0 + r;
                        if (R == 0 || R == HH - 1) pub(R, HV_T, w0);
                    }
                }
            });
            PMARK(10);
            if (S.mode == 0) {                         // the residual norms go to the slot accumulators
                s_e[0][tid] += a[1];
                s_e[1][tid] = fmax(s_e[1][tid], a[4]);
            }
            if (mrg) {
                double a7[7] = {a[0], a[2], a[3], am[0], am[1], am[2], am[3]};
                block_reduce2<7, 0, false>(a7, red);
                if (tid == 0) {
                    double* pq = S.part + ((long long)set * G + g) * NPART;
                    for (int j = 0; j < 7; ++j) pq[j] = a7[j];
                }
            } else {
                double a3[3] = {a[0], a[2], a[3]};
                block_reduce2<3, 0, false>(a3, red);
                if (tid == 0) {
                    double* pq = S.part + ((long long)set * G + g) * NPART;
                    pq[0] = a3[0];
                    pq[1] = a3[1];
                    pq[2] = a3[2];
                }
            }
        }
        PMARK(0);
        double bnorm2, rho, r0v0;
        double o7[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        {
            if (mrg) {
                auto prem = [&]() {                    // the neighbours' r0, v0, w0 boundary rows
                    if (hasS) {
                        hv[0] = __ldcg(hb_S + HV_R * HALO_ROW); hv[1] = __ldcg(hb_S + HV_V2 * HALO_ROW);
                        hv[2] = __ldcg(hb_S + HV_T * HALO_ROW);
                    }
                    if (hasN) {
                        hv[4] = __ldcg(hb_N + HV_R * HALO_ROW); hv[5] = __ldcg(hb_N + HV_V2 * HALO_ROW);
                        hv[6] = __ldcg(hb_N + HV_T * HALO_ROW);
                    }
                };
                bar_sync_reduce_pre<7, 0>(S.bs, G, ep, true, hi, S.part + (long long)set * G * NPART, NPART, g0, g1, o7, s_red,
                                          prem);
            } else {
                double o[3];
                bar_sync_reduce_pre<3, 0>(S.bs, G, ep, true, hi, S.part + (long long)set * G * NPART, NPART, g0, g1, o, s_red,
                                          pre2);
                o7[0] = o[0]; o7[1] = o[1]; o7[2] = o[2];
            }
            PMARK(4);
            rho = o7[0];                               // (r^0, r0) = ||r0||^2
            bnorm2 = o7[1];                            // ||b~||^2: reference of the relative stopping test
            r0v0 = o7[2];                              // (r^0, v0)
        }
        PMARK(5);
        set ^= 1;
        double alpha = 0.0, omega = 1.0, beta = 0.0;
        bool conv = rho <= atol2 || rho <= rtol2 * bnorm2, pending = false, epi_done = false;
        if (!conv) {
            if (r0v0 == 0.0 || !isfinite(r0v0)) {
                if (tid == 0 && c == 0) atomicOr(&S.bs->err, 2u);
                conv = true;
            } else {
                alpha = rho / r0v0;
            }
        }
        int it = 0, maxit_step = 0;
        bool fused_first = true;                       // iteration 0's phase 1 happened in the prologue
        // the scalar update that follows a phase-2 reduction (t = A s): omega, the residual estimate, the stop test,
        // beta and the new rho (Jacobi-scaled BiCGSTAB)
        auto after_phase2 = [&](double ts, double tt2, double r0s, double r0t, double ss) {
            ++it;
            pending = true;
            if (tt2 == 0.0) {
                omega = 0.0;
                conv = true;
            } else {
                omega = ts / tt2;
                const double rhon = r0s - omega * r0t;
                const double rn2 = fmax(ss - 2.0 * omega * ts + omega * omega * tt2, 0.0);
                if (!isfinite(omega) || !isfinite(rn2)) {
                    if (tid == 0 && c == 0) atomicOr(&S.bs->err, 1u);
                    conv = true;
                } else if (rn2 <= rtol2 * bnorm2 || rn2 <= atol2 || it >= S.lin_max) {
                    conv = true;
                } else if (omega == 0.0 || rhon == 0.0) {
                    if (tid == 0 && c == 0) atomicOr(&S.bs->err, 2u);
                    conv = true;
                } else {
                    beta = (rhon / rho) * (alpha / omega);
                    rho = rhon;
                }
            }
        };
        if (mrg) {
            // merged first iteration: with s = r0 - alpha v0 and t = A~ s = v0 - alpha w0, every dot product of the
            // first phase 2 is a polynomial in alpha of the reduced (r0, v0, w0) products: no second barrier
            if (!conv) {
                const double vv = o7[3], rw = o7[4], vw = o7[5], ww = o7[6];
                after_phase2(r0v0 - alpha * vv - alpha * rw + alpha * alpha * vw,     // (t, s)
                             vv - 2.0 * alpha * vw + alpha * alpha * ww,                 // (t, t)
                             rho - alpha * r0v0,                                         // (r^0, s)
                             r0v0 - alpha * rw,                                          // (r^0, t)
                             rho - 2.0 * alpha * r0v0 + alpha * alpha * vv);             // (s, s)
                #pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    if (r >= hs) continue;
                    const int i = r * BLOCK3 + tid;
                    const double v0 = v_s[i];
                    sr[r] = sr[r] - alpha * v0;        // s
                    t_s[i] = v0 - alpha * t_s[i];      // t (t_s held w0)
                    pp[r] = BT(r);                     // p = r0
                }
                // the neighbours' boundary rows as the (s, t, p, v) the phase-1 slot expects
                #pragma unroll
                for (int side = 0; side < 2; ++side) {     // unrolled: hv stays in registers
                    const int b = 4 * side;
                    const double r0h = hv[b], v0h = hv[b + 1], w0h = hv[b + 2];
                    hv[b] = r0h - alpha * v0h; hv[b + 1] = v0h - alpha * w0h; hv[b + 2] = r0h; hv[b + 3] = v0h;
                }
                maxit_step = it;
            }
            fused_first = false;
        }

        // Control flow around every block / pair reduction is uniform across the CTA (converged pairs reduce
        // zeros).
        for (;;) {
            if (!fused_first) {
                // ============ phase-1 slot: p update + v = A p  |  epilogue of a pair that just converged ======
                double a[4] = {0.0, 0.0, 0.0, 0.0};        // (b~, v) | sum du^2 | max |du|, nonfinite
                const bool do_p1 = !conv, do_epi = conv && !epi_done;
                if (do_p1) {
                    const double* const hS = hv;       // pre-loaded after barrier B (pre1)
                    const double* const hN = hv + 4;
                    with_hs([&](auto tag) {
                        constexpr int HC = decltype(tag)::value;
                        const int H = HC ? HC : hs, HH = (HC && Gr == 1) ? HC : h;
                        #pragma unroll
                        for (int r = 0; r < RMAX; ++r) {
                            if (r >= H) continue;
                            const int i = r * BLOCK3 + tid;
                            const double rr = sr[r] - omega * t_s[i];
                            if (pending) x_s[i] += alpha * pp[r] + omega * sr[r];
                            const double pn = rr + beta * (pp[r] - omega * v_s[i]);
                            sr[r] = rr;
                            pp[r] = pn;
                            put_op(r, pn);
                        }
                        const double haloS = (hS[0] - omega * hS[1]) + beta * (hS[2] - omega * hS[3]);
                        const double haloN = (hN[0] - omega * hN[1]) + beta * (hN[2] - omega * hN[3]);
                        __syncthreads();
                        #pragma unroll
                        for (int r = 0; r < RMAX; ++r) {
                            if (r >= H) continue;
                            const int si = sidx(r);
                            const Off o = coef(r);
                            const double vv = pp[r] + cinv(r) * (o.e * op_s[si + dE] + o.w * op_s[si + dW] +
                                                                 o.n * opNh(pp, r, haloN, H) + o.s * opS(pp, r, haloS));
                            v_s[r * BLOCK3 + tid] = vv;
                            a[0] += BT(r) * vv;
                            const int R = R0 + r;
                            if (R == 0 || R == HH - 1) { pub(R, HV_R, sr[r]); pub(R, HV_V2, vv); }
                        }
                    });
                    pending = false;
                } else if (do_epi) {
                    with_hs([&](auto tag) {
                        constexpr int HC = decltype(tag)::value;
                        const int H = HC ? HC : hs;
                        #pragma unroll
                        for (int r = 0; r < RMAX; ++r) {
                            if (r >= H) continue;
                            double dx = X(r);
                            if (pending) dx += alpha * pp[r] + omega * sr[r];
                            const long long q = q_of(r);
                            if (S.mode == 1) S.xptr[me][q] = dx;
                            else {
                                pX[q] = dx;
                                Unew[q] = u_s[uidx(r)] + dx;
                            }
                            a[1] += dx * dx;
                            a[2] = fmax(a[2], fabs(dx));
                            if (!isfinite(dx)) a[3] = 1.0;
                        }
                    });
                    if (S.mode == 0) {
                        s_e[2][tid] += a[1];
                        s_e[3][tid] = fmax(s_e[3][tid], a[2]);
                    }
                    pending = false;
                }
                if (do_p1) {
                    double a1[1] = {a[0]};
                    block_reduce2<1, 0, false>(a1, red);
                    a[0] = a1[0];
                } else if (do_epi && S.mode == 1) {
                    block_reduce2<2, 2, false>(a, red);
                }
                if (tid == 0) {
                    if (do_p1) S.part[((long long)set * G + g) * NPART] = a[0];
                    if (do_epi && S.mode == 1 && a[3] != 0.0) atomicOr(&S.bs->err, 1u);
                }
                if (do_epi) epi_done = true;
                if (do_epi) PMARK(3); else PMARK(1);           // trace: epilogue slot vs phase-1 work
                double o1[1];
                const bool any = bar_sync_reduce_pre<1, 0>(S.bs, G, ep, !conv, hi, S.part + (long long)set * G * NPART,
                                                           NPART, g0, g1, o1, s_red, pre2);
                PMARK(4);
                if (!any) { set ^= 1; break; }
                const double r0v = o1[0];
                PMARK(5);
                set ^= 1;
                if (!conv) {
                    if (r0v == 0.0 || !isfinite(r0v)) {
                        if (tid == 0 && c == 0) atomicOr(&S.bs->err, 2u);
                        conv = true;
                    } else {
                        alpha = rho / r0v;
                    }
                }
            }
            fused_first = false;
            // ================= phase 2: s = r - alpha v, t = A s ====================================
            {
                double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};   // (t,s) (t,t) (b~,s) (b~,t) (s,s)
                if (!conv) {
                    const double* const hS = hv;       // pre-loaded after barrier A / the phase-1 barrier (pre2)
                    const double* const hN = hv + 4;
                    with_hs([&](auto tag) {
                        constexpr int HC = decltype(tag)::value;
                        const int H = HC ? HC : hs, HH = (HC && Gr == 1) ? HC : h;
                        #pragma unroll
                        for (int r = 0; r < RMAX; ++r) {
                            if (r >= H) continue;
                            const double sv = sr[r] - alpha * v_s[r * BLOCK3 + tid];
                            sr[r] = sv;
                            put_op(r, sv);
                        }
                        const double haloS = hS[0] - alpha * hS[1], haloN = hN[0] - alpha * hN[1];
                        __syncthreads();
                        #pragma unroll
                        for (int r = 0; r < RMAX; ++r) {
                            if (r >= H) continue;
                            const int si = sidx(r);
                            const Off o = coef(r);
                            const double sv = sr[r];
                            const double t = sv + cinv(r) * (o.e * op_s[si + dE] + o.w * op_s[si + dW] +
                                                             o.n * opNh(sr, r, haloN, H) + o.s * opS(sr, r, haloS));
                            t_s[r * BLOCK3 + tid] = t;
                            const double b0 = BT(r);
                            a[0] += t * sv; a[1] += t * t; a[2] += b0 * sv; a[3] += b0 * t; a[4] += sv * sv;
                            const int R = R0 + r;
                            if (R == 0 || R == HH - 1) {
                                pub(R, HV_S, sv); pub(R, HV_T, t); pub(R, HV_P, pp[r]); pub(R, HV_V, v_s[r * BLOCK3 + tid]);
                            }
                        }
                    });
                }
                block_reduce2<5, 0, false>(a, red);
                if (tid == 0 && !conv) {
                    double* pq = S.part + ((long long)set * G + g) * NPART;
                    for (int j = 0; j < 5; ++j) pq[j] = a[j];
                }
                PMARK(2);
            }
            {
                double o[5];
                bar_sync_reduce_pre<5, 0>(S.bs, G, ep, false, hi, S.part + (long long)set * G * NPART, NPART, g0, g1, o, s_red,
                                          pre1);
                PMARK(4);
                if (!conv) after_phase2(o[0], o[1], o[2], o[3], o[4]);
            }
            set ^= 1;
            maxit_step = it > maxit_step ? it : maxit_step;
            PMARK(5);
        }

        // ---- norms: every CTA accumulates its own partials per pipeline slot over the levels it serves; only
        // when an iteration finishes (at most one per step: start steps are distinct) are the accumulators
        // published and reduced over the grid (one extra barrier per iteration), then the stop rule -----------
        int stop_status = 2, stop_k = -1;
        int kc = -1;
        if (S.mode == 0)
            for (int aa = 0; aa < A; ++aa)
                if (step - sS[kbase + aa] + 1 == P.nt) kc = kbase + aa;
        if (kc >= 0 && e_slot == s_kD[kc]) {           // this CTA holds update norms of iteration kc
            flush_e();
            e_slot = -1;
        }
        if (S.mode == 0 && tid == 0) {
            if (kc >= 0) {
                const int sa = s_kD[kc];
                double* hq = S.hpart + ((long long)sa * G + g) * 4;
                for (int j = 0; j < 4; ++j) { hq[j] = lacc[sa][j]; lacc[sa][j] = 0.0; }
            }
        }
        if (kc >= 0) {
            bar_sync(S.bs, G, ep, false, hi);
            const double* hq = S.hpart + (long long)s_kD[kc] * G * 4;
            for (int j = tid; j < G * 4; j += BLOCK3) s_hp_big[j] = __ldcg(hq + j);
            __syncthreads();
            __shared__ int s_stop[3];                  // stop_status, stop_k, last_done (thread 0 -> all)
            if (tid < 32) {
                double a4[4] = {0.0, 0.0, 0.0, 0.0};
                for (int gg = tid; gg < G; gg += 32) {
                    a4[0] += s_hp_big[gg * 4 + 0]; a4[1] = fmax(a4[1], s_hp_big[gg * 4 + 1]);
                    a4[2] += s_hp_big[gg * 4 + 2]; a4[3] = fmax(a4[3], s_hp_big[gg * 4 + 3]);
                }
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    a4[0] += __shfl_xor_sync(0xffffffffu, a4[0], o);
                    a4[1] = fmax(a4[1], __shfl_xor_sync(0xffffffffu, a4[1], o));
                    a4[2] += __shfl_xor_sync(0xffffffffu, a4[2], o);
                    a4[3] = fmax(a4[3], __shfl_xor_sync(0xffffffffu, a4[3], o));
                }
                if (tid == 0) {
                    const int k = kc;
                    int st_ = 2, sk_ = -1;
                    const double Ntot = (double)ns * (double)P.nt;
                    const double dmax = S.stop_norm ? sqrt(a4[2] / Ntot) : a4[3];   // stop norm
                    if (g == 0) {
                        S.hist[4 * k + 0] = sqrt(a4[0] / Ntot);
                        S.hist[4 * k + 1] = a4[1];
                        S.hist[4 * k + 2] = sqrt(a4[2] / Ntot);
                        S.hist[4 * k + 3] = a4[3];
                    }
                    if (dmax <= S.newton_tol) { st_ = 0; sk_ = k; }
                    else if (k >= 1 && dmax > 0.5 * prevmax_s && dmax <= 1e3 * S.newton_tol) { st_ = 1; sk_ = k; }
                    else if (k + 1 >= newton_max) { st_ = -4; sk_ = k; }
                    prevmax_s = dmax;
                    s_stop[0] = st_; s_stop[1] = sk_; s_stop[2] = k;
                }
            }
            __syncthreads();
            stop_status = s_stop[0];
            stop_k = s_stop[1];
            last_done = s_stop[2];
        }
        if (g == 0 && tid == 0) total_inner += maxit_step;
        if (c == 0 && tid == 0 && S.stats && S.mode == 0) {
            atomicAdd((unsigned long long*)&S.stats[4], (unsigned long long)it);
            atomicAdd((unsigned long long*)&S.stats[8 + kme], (unsigned long long)it);
        }
        PMARK(6);
        if (S.mode == 1) {
            if (g == 0 && tid == 0) {
                S.info[0] = maxit_step;
                S.info[1] = *((volatile unsigned*)&S.bs->err) ? -5 : 0;
            }
            flush_prof();
            return;
        }
        // errors are raised only between a step's first and last barrier, so every CTA reads the same value here
        if (kc >= 0 && stop_status == 2 && *((volatile unsigned*)&S.bs->err)) { stop_status = -5; stop_k = last_done; }
        if (stop_status != 2) {
            const int kf = stop_k + 1;
            const double* Uf = S.U + (long long)(kf % S.B) * P.nt * ns;
            const long long N = ns * P.nt;
            if (S.u_out)
                for (long long q = (long long)g * BLOCK3 + tid; q < N; q += (long long)G * BLOCK3) S.u_out[q] = __ldcg(Uf + q);
            if (g == 0 && tid == 0) {
                S.info[0] = kf;
                S.info[1] = stop_status;
                if (S.stats) {
                    S.stats[0] = step; S.stats[1] = total_inner; S.stats[2] = S.D; S.stats[3] = G;
                    S.stats[5] = ep;                   // grid barriers every CTA passed
                }
            }
            flush_prof();
            return;
        }
    }
}

#undef PMARK

}  // namespace pit
