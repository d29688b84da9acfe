// pit_newton_ps0.cuh — engine 5 for the GENERAL LAW (mu(u) = m0 + m2 u^2: the nonlinear heat equation, Burgers with
// m2 > 0) on Dirichlet or periodic grids: the pipeline of CTA sets of pit_newton_ps.cuh (same schedule, same exchange
// cells, same level counters, same stop rule; read that file's header first) with the two things the general law
// changes:
//  * the coefficients of A_n = I + tau dF/du (Eq. (6)) depend on u at BOTH ends of a face
//    (mu((u_C + u_nb) / 2) and its derivative, R1), so a neighbour's contribution is not a function of the
//    neighbour alone: the four off-diagonal coefficients of every own point, divided by its diagonal, are formed once
//    per level in the residual pass (residual_jacobian_raw, pit_internal.cuh) and kept in shared memory in per-thread
//    slots (no bank conflicts, no sharing), and a half-sweep GATHERS: x <- (1 - omega) x + omega (b' - sum a' x_nb);
//  * Dirichlet boundaries (Eq. (2)): strips at the bottom / top of the grid have no neighbouring strip (their halo
//    row of u comes from the level's boundary ring, the increment du vanishes there), and the first / last column pair
//    has no x-neighbour thread (its travelling value is a zero slot of the warp-edge array; u from the ring).
// Rows of 256 unknowns (the coefficient slots of 512-wide strips do not fit in shared memory).
#pragma once
#include "pit_newton_ps.cuh"

namespace pit {

template <int NXU, int HE, bool PER, bool TRACE>
struct PsEngine0 {
    static constexpr int RG = 2;
    static constexpr int T = NXU / 2;          // threads per row group (two columns each)
    static constexpr int NW = T / 32;          // warps per row group
    static constexpr int NTH = RG * T;         // RG = 2: the lower and the upper half of the strip's rows
    static constexpr int HM = HE + 2;          // max strip height (strips have HE or HE + 2 rows, r0 even)
    static constexpr int HHM = HM / RG;        // max rows per thread
    static constexpr int UP = NXU + 2;         // ubuf row pitch: [even columns (T)][odd columns (T)][west boundary][east boundary]
    static constexpr int NWP = NW + 1;         // warp-edge slots per row: one per warp + a zero slot (no x-neighbour: Dirichlet)
    static constexpr size_t OFF_U = 0;                                    // ubuf [HM + 2][UP]: u^n rows r0-1 .. r0+H
    static constexpr size_t OFF_B = OFF_U + (size_t)(HM + 2) * UP;        // bs   [HHM][2][NTH] right-hand sides / a_C
    static constexpr size_t OFF_C = OFF_B + (size_t)HHM * 2 * NTH;        // cf   [4][HHM][2][NTH] a_partner, a_outside, a_N, a_S (each / a_C)
    static constexpr size_t OFF_A = OFF_C + (size_t)4 * HHM * 2 * NTH;    // acc  [NB_NP][NTH] per-thread norm partials
    static constexpr size_t OFF_E = OFF_A + (size_t)NB_NP * NTH;          // wedge [RG groups][2 kinds][HHM][NWP] warp-edge values of du
    static constexpr size_t OFF_G = OFF_E + (size_t)RG * 2 * HHM * NWP;   // gx   [2 colours][2][T] du across the row groups
    static constexpr size_t OFF_R = OFF_G + (size_t)4 * T;                // red  [RG NW][NB_NP]
    static constexpr size_t OFF_S = OFF_R + (size_t)RG * NW * NB_NP;      // scalars shared by the two code paths (16 words)
    static constexpr size_t SMEM = (OFF_S + 16) * sizeof(double);

    // HH = rows per thread (H = 2 HH rows per strip).  Row group g owns strip rows g HH .. g HH + HH - 1.  When HH is
    // odd the upper group starts on an odd row: its threads hold their two columns SWAPPED (local column jj = actual
    // column ^ f), so that the colour of local point (q, jj) is (q + jj) & 1 in both groups and every register
    // subscript stays compile-time; the E/W roles then mirror, which only flips the sign of ax and the shuffle
    // direction (per-thread constants).
    template <int HH, int GRP>
    __device__ __forceinline__ static void run(const PsParams& S, double* sm) {
        constexpr int H = RG * HH;
        const Prob P = S.P;
        const int Gs = S.Gs, c = blockIdx.x, p = c / Gs, s = c % Gs;
        const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
        constexpr int g = GRP;                              // the row group is compile-time (the kernel branches once, per warp)
        const int t = tid % T, wl = w % NW;
        const int nyu = P.nyu, nt = P.nt, D = S.D, B = S.B;
        const long long ns = P.ns;
        const int na = (nyu - HE * Gs) / 2;                 // strips 0 .. na-1 have HE + 2 rows
        const int r0 = s * HE + 2 * min(s, na);             // first row of the strip (even)
        // neighbouring strips (rows below / above); -1 = the grid's Dirichlet boundary
        const int ss = s > 0 ? s - 1 : (PER ? Gs - 1 : -1), sn = s + 1 < Gs ? s + 1 : (PER ? 0 : -1);
        const int nxp = P.nx + 1;                           // ring layout: bottom [nxp], top [nxp], left [ny-1], right [ny-1]
        constexpr int f = (g * HH) & 1;                     // column swap of this thread (upper group, HH odd)
        const int c0 = 2 * t;

        // The iterate this solve will probably end in (the previous solve's count, a device word: no host round trip)
        // is written straight into u_out; slot 0 (U_0 / a caller's guess) never is.  A wrong guess costs the final copy.
        // (kept in shared memory: the sweeps have no register to spare)
        long long* s_tr = reinterpret_cast<long long*>(sm + OFF_S);      // [PS_TR] cycle accounts
        long long* s_tm = s_tr + PS_TR;                                    // [2]
        int* s_dec = reinterpret_cast<int*>(s_tm + 2);                     // [2] the pass's decision
        int& s_last = s_dec[2];
        int& s_alias = s_dec[3];
        if (tid == 0) {
            const int hint = S.u_out ? __ldcg(S.hint) : 0;
            s_alias = (hint > 0 && hint % B != 0) ? hint % B : -1;
        }
        double* ubuf = sm + OFF_U;
        double* ub = ubuf + (size_t)(1 + g * HH) * UP;       // the thread's local row 0 (rows -1 and HH exist too)
        double* cfs = sm + OFF_C;
        double* bs = sm + OFF_B;
        double* accs = sm + OFF_A;
        double* wedge = sm + OFF_E + (size_t)g * 2 * HHM * NWP;  // this group's [2 kinds][HHM][NWP]
        double* gx0 = sm + OFF_G;                            // per colour: [0][t] lower group's top row -> upper, [1][t] upper's bottom row -> lower
        double* red_s = sm + OFF_R;

        // LL cells of a strip: [ring][side][t]; side 0 = its bottom row (published by the lower group), 1 = its top row
        unsigned long long* myx = S.llx + ((size_t)(p * Gs + s) * PS_RX * 2 * T) * 2;
        const unsigned long long* sbx = S.llx + ((size_t)(p * Gs + max(ss, 0)) * PS_RX * 2 * T) * 2;   // the strip below
        const unsigned long long* nbx = S.llx + ((size_t)(p * Gs + max(sn, 0)) * PS_RX * 2 * T) * 2;   // the strip above
        const bool has_nb = (g ? sn : ss) >= 0;              // this row group's side of the strip has a neighbouring strip
        auto mycell = [&](unsigned q, int side) { return myx + ((size_t)((q % PS_RX) * 2 + side) * T + t) * 2; };
        auto scell = [&](unsigned q) { return sbx + ((size_t)((q % PS_RX) * 2 + 1) * T + t) * 2; };   // its top row
        auto ncell = [&](unsigned q) { return nbx + ((size_t)((q % PS_RX) * 2 + 0) * T + t) * 2; };   // its bottom row

        const double omega = __ldcg(S.ctl);
        const int SW = (int)__ldcg(S.ctl + 1);
        const int chk = max(1, (int)__ldcg(S.ctl + 3));
        const double om1 = 1.0 - omega;                      // x <- om1 x + omega (b' - sum a' x_nb), a' = a / a_C
        const double rsc = om1 / omega;                      // (scaled) residual of a just-relaxed point: rsc (x_new - x_old)
        // kind A rows (other colour in local column 1): the product travels to thread t + 1 (f = 0) or t - 1 (f = 1);
        // kind B rows (other colour in local column 0): the opposite way.
        int srcA = (lane + (f ? 1 : 31)) & 31, srcB = (lane + (f ? 31 : 1)) & 31;
        asm volatile("" : "+r"(srcA), "+r"(srcB));
        const int edgeA = f ? 31 : 0, edgeB = f ? 0 : 31;    // lanes whose source lies in the neighbouring warp
        // the neighbouring warp's slot (periodic: wraps; Dirichlet: the first / last warp's outer side is the zero slot NW)
        const int wprev = wl > 0 ? wl - 1 : (PER ? NW - 1 : NW), wnext = wl + 1 < NW ? wl + 1 : (PER ? 0 : NW);
        const int wsA = f ? wnext : wprev, wsB = f ? wprev : wnext;
        double* wdA = wedge;                                 // [HHM][NWP]
        double* wdB = wedge + (size_t)HHM * NWP;
        int isA = lane == edgeA, isB = lane == edgeB;         // this lane's kind A / B source lies in the neighbouring warp
        int wrA = lane == 31 - edgeA, wrB = lane == 31 - edgeB;   // this lane's kind A / B product is a neighbouring warp's source
        unsigned wdA_w = (unsigned)__cvta_generic_to_shared(wdA + wl), wdB_w = (unsigned)__cvta_generic_to_shared(wdB + wl);   // rows are NWP apart
        // (opaque to the compiler, which otherwise rebuilds these from the thread index in every row of the sweeps)
        asm volatile("" : "+r"(isA), "+r"(isB), "+r"(wrA), "+r"(wrB), "+r"(wdA_w), "+r"(wdB_w));
        // ubuf rows are de-interleaved: [even columns (T)][odd columns (T)], so that a warp's loads of one local column
        // are contiguous (no bank conflicts).  Offsets of local columns 0 and 1, and of their out-of-thread x-neighbours
        // (actual column c0 - 1: odd, pair t - 1; actual column c0 + 2: even, pair t + 1; periodic).
        const int uo0 = f * T + t, uo1 = (1 - f) * T + t;
        const int cwest = t > 0 ? T + t - 1 : (PER ? 2 * T - 1 : NXU), ceast = t + 1 < T ? t + 1 : (PER ? 0 : NXU + 1);
        const int co0 = f ? ceast : cwest, co1 = f ? cwest : ceast;

        auto cbar = [&]() { __syncthreads(); };
        auto bsm = [&](int r, int j) -> double& { return bs[(size_t)(r * 2 + j) * NTH + tid]; };
        auto cfm = [&](int kind, int r, int j) -> double& { return cfs[(size_t)((kind * HHM + r) * 2 + j) * NTH + tid]; };   // 0 partner, 1 outside, 2 N, 3 S
        auto ac = [&](int j) -> double& { return accs[(size_t)j * NTH + tid]; };
        auto lswap = [&](double2 v) { return f ? make_double2(v.y, v.x) : v; };   // actual <-> local column order

        double x[HH][2];
        #pragma unroll
        for (int j = 0; j < NB_NP; ++j) ac(j) = 0.0;
        for (int i = tid; i < RG * 2 * HHM * NWP; i += NTH) (sm + OFF_E)[i] = 0.0;   // (the zero slots stay zero: nobody writes them)
        int lastx = -1;
        unsigned qx = 0;
        int levels = 0;
        const bool trace = TRACE && S.trace != nullptr && tid == 0;   // cycle accounts of thread 0, kept in shared memory
        if (trace) {
            for (int i = 0; i < PS_TR; ++i) s_tr[i] = 0;
            s_tm[0] = s_tm[1] = clock64();
        }
        auto mark = [&](int i) { if (trace) { const long long now = clock64(); s_tr[i] += now - s_tm[1]; s_tm[1] = now; } };
        auto take = [&](const unsigned long long* q, LLc cl, unsigned fl) -> double {
            if (TRACE && (S.dbg & 1)) return __hiloint2double((int)(unsigned)cl.w1, (int)(unsigned)cl.w0);   // timing experiment: no wait
            if (trace) {
                long long a = 0;
                const double v = ll_take_t(q, cl, fl, a);
                s_tr[3] += a;
                return v;
            }
            return ll_take(q, cl, fl);
        };

        // ---- thread 0's side jobs (no warp is set aside for them) ----
        const unsigned* fprev = p > 0 ? S.lvl + (size_t)(p - 1) * Gs : nullptr;   // set p-1's level counters
        unsigned* fmine = S.lvl + (size_t)p * Gs + s;
        int flag_lv = 0;        // thread 0: level whose U_{k+1} rows are written but not yet published (0 = none)
        int pf_lv = 0;          // thread 0: level whose U_k rows (set p-1) are still to be confirmed (0 = none)
        // One fence serves both jobs: it releases this strip's U_{k+1}^{flag_lv} rows (every thread stored them before
        // the last CTA barrier) ahead of the level counter, and it orders set p-1's counters (relaxed loads) before this
        // CTA's loads of their rows (which follow the next CTA barrier).
        auto service = [&](unsigned base) {
            unsigned v0 = 0xffffffffu, v1 = 0xffffffffu, v2 = 0xffffffffu;
            if (pf_lv && fprev) {
                v0 = ps::ld_rlx(fprev + s);
                if (ss >= 0) v1 = ps::ld_rlx(fprev + ss);
                if (sn >= 0) v2 = ps::ld_rlx(fprev + sn);
            }
            const bool ready = pf_lv && min(v0, min(v1, v2)) >= base + (unsigned)pf_lv;
            if ((flag_lv || (ready && fprev)) && !(TRACE && (S.dbg & 2))) __threadfence();   // (dbg bit 1: timing experiment without the fence)
            if (flag_lv) {
                asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(fmine), "r"(base + (unsigned)flag_lv) : "memory");
                flag_lv = 0;
            }
            if (ready) pf_lv = 0;
        };

        // tt[q] = b' - sum a' x_nb at the colour-cc point of every own row q (local column j = (q + cc) & 1), with the
        // point's own coefficients a' = a / a_C from its shared-memory slots.  Its x-neighbour inside the thread is the
        // other column of the row, the one outside travels by warp shuffle (warp edges through shared memory, the
        // grid's edge through the zero slot), the rows above / below are the thread's own registers, the other row
        // group's boundary row (shared memory) or the neighbouring strip's (LL cell; none at a Dirichlet boundary).
        auto gather = [&](const int cc, double (&tt)[HH], const bool svc, const unsigned fbase) {
            LLc hc;
            const unsigned qn = (unsigned)lastx;
            const bool ll = lastx >= 0 && has_nb;
            if (ll) hc = ll_issue(g ? ncell(qn) : scell(qn));
            if (svc && tid == 0 && (flag_lv | pf_lv)) service(fbase);
            double* gx = gx0 + (size_t)cc * 2 * T;           // double-buffered: a fast warp's next half-sweep writes the other half
            // (the loads of a row's right-hand side and coefficients run one row ahead of their use)
            double nb_ = bsm(0, cc & 1), n0_ = cfm(0, 0, cc & 1), n1_ = cfm(1, 0, cc & 1), n2_ = cfm(2, 0, cc & 1), n3_ = cfm(3, 0, cc & 1);
            #pragma unroll
            for (int q = 0; q < HH; ++q) {
                const int j = (q + cc) & 1, jn = 1 - j;
                const double xq = x[q][jn];                   // this row's point of the other colour
                const double cb = nb_, c0_ = n0_, c1_ = n1_, c2_ = n2_, c3_ = n3_;
                if (q + 1 < HH) {
                    const int j1 = (q + 1 + cc) & 1;
                    nb_ = bsm(q + 1, j1); n0_ = cfm(0, q + 1, j1); n1_ = cfm(1, q + 1, j1); n2_ = cfm(2, q + 1, j1); n3_ = cfm(3, q + 1, j1);
                }
                double acc = fma(-c0_, xq, cb);
                if (jn == 1) {               // kind A: the value travels as for the constant-viscosity law
                    const double in = __shfl_sync(0xffffffffu, xq, srcA);
                    if (!isA) acc = fma(-c1_, in, acc);
                    if (wrA) wdA[q * NWP + wl] = xq;
                } else {
                    const double in = __shfl_sync(0xffffffffu, xq, srcB);
                    if (!isB) acc = fma(-c1_, in, acc);
                    if (wrB) wdB[q * NWP + wl] = xq;
                }
                if (q + 1 < HH) acc = fma(-c2_, x[q + 1 < HH ? q + 1 : q][j], acc);
                if (q > 0) acc = fma(-c3_, x[q > 0 ? q - 1 : 0][j], acc);
                tt[q] = acc;
            }
            // this group's boundary row towards the other group: its point of the other colour (raw du)
            if (g == 0) gx[t] = x[HH - 1][1 - ((HH - 1 + cc) & 1)];
            else gx[T + t] = x[0][1 - (cc & 1)];
            cbar();
            if (isA) {
                #pragma unroll
                for (int q = 0; q < HH; ++q)
                    if (((q + cc) & 1) == 0) tt[q] = fma(-cfm(1, q, 0), wdA[q * NWP + wsA], tt[q]);      // kind A rows: active column 0
            }
            if (isB) {
                #pragma unroll
                for (int q = 0; q < HH; ++q)
                    if ((q + cc) & 1) tt[q] = fma(-cfm(1, q, 1), wdB[q * NWP + wsB], tt[q]);             // kind B rows: active column 1
            }
            // the row below local row 0 and the row above local row HH-1: the other row group or the neighbouring strip
            if (g == 0) {
                tt[HH - 1] = fma(-cfm(2, HH - 1, (HH - 1 + cc) & 1), gx[T + t], tt[HH - 1]);
                if (ll) tt[0] = fma(-cfm(3, 0, cc & 1), take(scell(qn), hc, qn + 1u), tt[0]);
            } else {
                tt[0] = fma(-cfm(3, 0, cc & 1), gx[t], tt[0]);
                if (ll) tt[HH - 1] = fma(-cfm(2, HH - 1, (HH - 1 + cc) & 1), take(ncell(qn), hc, qn + 1u), tt[HH - 1]);
            }
        };

        for (int pass = 0;; ++pass) {
            const int k = pass * D + p;
            const bool active = p < D && k < S.newton_max;
            // iterate k: the broadcast u^0 (every level reads the same rows) when no U_0 was materialised, else ring
            // buffer k % B — which lives in the caller's u_out for the slot the previous solve ended in

            const unsigned fbase = (unsigned)pass * (unsigned)nt;
            const int rg0 = r0 + g * HH;                         // global row of local row 0
            if (active) {
                #pragma unroll
                for (int r = 0; r < HH; ++r) {
                    x[r][0] = 0.0; x[r][1] = 0.0;
                    const double2 v = ldcg2(S.u0 + (size_t)(rg0 + r) * NXU + c0);     // u^{n-1} of level 1
                    ub[(size_t)r * UP + t] = v.x;
                    ub[(size_t)r * UP + T + t] = v.y;
                }
                lastx = -1;
                if (tid == 0) pf_lv = 1;
            }
            for (int n = 1; active && n <= nt; ++n) {
                ++levels;
                mark(6);
                // ---- set p-1 must have published U_k^n (normally confirmed by service() during the previous level)
                cbar();                                             // every thread has stored level n-1 and is done reading its u
                if (tid == 0) {
                    while (pf_lv) {
                        service(fbase);
                        if (pf_lv) __nanosleep(64);
                    }
                }
                cbar();
                // ---- prologue 1: b = du^{n-1} - (u^n - u^{n-1}); u^n replaces u^{n-1} in shared memory
                {
                    const double* un = (k == 0 && S.u0_bcast) ? S.u0 + c0 : ring_buf(S, s_alias, k % B) + (size_t)(n - 1) * ns + c0;
                    const double* rgn = (!PER && S.ring) ? S.ring + (size_t)(n - 1) * P.ring_len : nullptr;   // level n's boundary ring
                    double2 pf[HH + 1];                             // own rows, then this group's strip-halo row
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) pf[r] = ldcg2(un + (size_t)(rg0 + r) * NXU);
                    if (has_nb) {
                        pf[HH] = ldcg2(un + (size_t)(g ? (rg0 + HH) % nyu : (rg0 - 1 + nyu) % nyu) * NXU);
                    } else {                                        // Dirichlet: the ring's bottom (j = 0) / top (j = ny) row, i = c0 + 1, c0 + 2
                        const double* rr = rgn ? rgn + (g ? nxp : 0) + c0 + 1 : nullptr;
                        pf[HH] = rr ? make_double2(__ldcg(rr), __ldcg(rr + 1)) : make_double2(0.0, 0.0);
                    }
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        const double2 nw = lswap(pf[r]);
                        bsm(r, 0) = x[r][0] - (nw.x - ub[(size_t)r * UP + uo0]);
                        bsm(r, 1) = x[r][1] - (nw.y - ub[(size_t)r * UP + uo1]);
                        ub[(size_t)r * UP + t] = pf[r].x;
                        ub[(size_t)r * UP + T + t] = pf[r].y;
                    }
                    double* hrow = g ? ub + (size_t)HH * UP : ub - (ptrdiff_t)UP;
                    hrow[t] = pf[HH].x;
                    hrow[T + t] = pf[HH].y;
                    if (!PER && (t == 0 || t == T - 1)) {           // the level's left / right boundary values of the own rows
                        #pragma unroll
                        for (int r = 0; r < HH; ++r) {
                            const int jr = rg0 + r;
                            if (t == 0) ub[(size_t)r * UP + NXU] = rgn ? __ldcg(rgn + 2 * nxp + jr) : 0.0;
                            if (t == T - 1) ub[(size_t)r * UP + NXU + 1] = rgn ? __ldcg(rgn + 2 * nxp + (P.ny - 1) + jr) : 0.0;
                        }
                    }
                }
                cbar();
                if (tid == 0 && n < nt) pf_lv = n + 1;
                mark(0);
                // ---- prologue 2: r^n = -G^n, b = r^n + du^{n-1}, and the rows of A_n (Eq. (6)), everything divided by a_C
                {
                    double ar2 = 0.0, arm = 0.0;
                    double p0 = ub[-(ptrdiff_t)UP + uo0], p1 = ub[-(ptrdiff_t)UP + uo1];
                    double c0v = ub[uo0], c1v = ub[uo1];
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        const double n0 = ub[(size_t)(r + 1) * UP + uo0], n1 = ub[(size_t)(r + 1) * UP + uo1];
                        const double o0 = ub[(size_t)r * UP + co0], o1 = ub[(size_t)r * UP + co1];
                        // local column 0 is actual column f: its outside x-neighbour is W (f = 0) or E (f = 1), the partner the other
                        Vals v0, v1;
                        v0.c = c0v; v0.n = n0; v0.s = p0; v0.e = f ? o0 : c1v; v0.w = f ? c1v : o0;
                        v1.c = c1v; v1.n = n1; v1.s = p1; v1.e = f ? c0v : o1; v1.w = f ? o1 : c0v;
                        const RJ j0 = residual_jacobian_raw(P, v0, 0.0), j1 = residual_jacobian_raw(P, v1, 0.0);
                        const double f0 = j0.G - c0v, f1 = j1.G - c1v;                          // tau F(u^n)
                        const double b0 = bsm(r, 0), b1 = bsm(r, 1);
                        const double G0 = (x[r][0] - b0) + f0, G1 = (x[r][1] - b1) + f1;     // (u^n - u^{n-1}) + tau F(u^n)
                        const double i0 = 1.0 / j0.aC, i1 = 1.0 / j1.aC;
                        bsm(r, 0) = (b0 - f0) * i0;
                        bsm(r, 1) = (b1 - f1) * i1;
                        cfm(0, r, 0) = (f ? j0.aW : j0.aE) * i0;  cfm(1, r, 0) = (f ? j0.aE : j0.aW) * i0;
                        cfm(2, r, 0) = j0.aN * i0;                cfm(3, r, 0) = j0.aS * i0;
                        cfm(0, r, 1) = (f ? j1.aE : j1.aW) * i1;  cfm(1, r, 1) = (f ? j1.aW : j1.aE) * i1;
                        cfm(2, r, 1) = j1.aN * i1;                cfm(3, r, 1) = j1.aS * i1;
                        ar2 = fma(G0, G0, fma(G1, G1, ar2));
                        arm = fmax(arm, fmax(fabs(G0), fabs(G1)));
                        p0 = c0v; p1 = c1v; c0v = n0; c1v = n1;
                    }
                    ac(0) += ar2;
                    ac(1) = fmax(ac(1), arm);
                }
                mark(1);
                // ---- S red-black SOR sweeps, one neighbour exchange per half-sweep
                const bool chkl = (n % chk == 0) || n == nt;
                for (int m = 0; m < SW; ++m) {
                    const bool lastm = m == SW - 1 && chkl;
                    #pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        double tt[HH];
                        gather(cc, tt, true, fbase);
                        if (cc == 1 && lastm) {      // (CTA-uniform) the last black half-sweep of a checked level: also its residual
                            double rs2 = 0.0, rsm = 0.0;
                            #pragma unroll
                            for (int r = 0; r < HH; ++r) {
                                const int j = (r + cc) & 1;
                                const double xo = x[r][j], xn = fma(omega, tt[r], om1 * xo);
                                x[r][j] = xn;
                                const double rr = rsc * (xn - xo);
                                rs2 = fma(rr, rr, rs2);
                                rsm = fmax(rsm, fabs(rr));
                            }
                            if (has_nb) ll_put(mycell(qx, g), g ? x[HH - 1][(HH - 1 + cc) & 1] : x[0][cc & 1], qx + 1u);
                            ac(4) += rs2;
                            ac(5) = fmax(ac(5), rsm);
                        } else {
                            #pragma unroll
                            for (int i = 0; i < HH; ++i) {
                                const int r = i == 0 ? 0 : (i == 1 ? HH - 1 : i - 1);     // the two end rows first: one of them is the strip's boundary row
                                const int j = (r + cc) & 1;
                                const double xo = x[r][j];
                                x[r][j] = fma(omega, tt[r], om1 * xo);
                                if (i == (HH > 1 ? 1 : 0)) {     // publish the strip's boundary rows: local row 0 of the lower group, HH-1 of the upper
                                    if (has_nb) ll_put(mycell(qx, g), g ? x[HH - 1][(HH - 1 + cc) & 1] : x[0][cc & 1], qx + 1u);
                                }
                            }
                        }
                        lastx = (int)qx;
                        ++qx;
                    }
                }
                mark(2);
                // ---- epilogue: U_{k+1}^n = U_k^n + du^n (du^n stays in x as the next carry)
                {
                    double* Un = ring_buf(S, s_alias, (k + 1) % B) + (size_t)(n - 1) * ns;
                    double d2 = 0.0, dm = 0.0;
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        double2 v;
                        v.x = ub[(size_t)r * UP + uo0] + x[r][0];
                        v.y = ub[(size_t)r * UP + uo1] + x[r][1];
                        *reinterpret_cast<double2*>(Un + (size_t)(rg0 + r) * NXU + c0) = lswap(v);
                        d2 = fma(x[r][0], x[r][0], fma(x[r][1], x[r][1], d2));
                        dm = fmax(dm, fmax(fabs(x[r][0]), fabs(x[r][1])));
                    }
                    ac(2) += d2;
                    ac(3) = fmax(ac(3), dm);
                    if (tid == 0) flag_lv = n;                      // published by service() after the next CTA barrier
                }
                mark(4);
                // ---- a-posteriori residual of the red points after the final black half-sweep
                if (chkl) {
                    double tt[HH];
                    gather(0, tt, false, fbase);
                    double rs2 = 0.0, rsm = 0.0, bb2 = 0.0;
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        const double rr = tt[r] - x[r][r & 1];
                        rs2 = fma(rr, rr, rs2);
                        rsm = fmax(rsm, fabs(rr));
                        bb2 = fma(bsm(r, 0), bsm(r, 0), fma(bsm(r, 1), bsm(r, 1), bb2));
                    }
                    ac(4) += rs2;
                    ac(5) = fmax(ac(5), rsm);
                    ac(6) += bb2;
                    mark(5);
                }
                // ---- iteration end: per-CTA partials, the set's last CTA reduces and decides
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
                    if (lane == 0)
                        #pragma unroll
                        for (int j = 0; j < NB_NP; ++j) red_s[w * NB_NP + j] = a[j];
                    cbar();
                    if (tid == 0) {
                        service(fbase);                            // level nt's counter (fence inside)
                        double* hp = S.hpart + ((size_t)k * Gs + s) * NB_NP;
                        for (int j = 0; j < NB_NP; ++j) {
                            double v = red_s[j];
                            for (int ww = 1; ww < RG * NW; ++ww) v = nb_is_max(j) ? fmax(v, red_s[ww * NB_NP + j]) : v + red_s[ww * NB_NP + j];
                            hp[j] = v;
                        }
                        __threadfence();
                        s_last = atomicAdd(S.arrive + k, 1u) == (unsigned)(Gs - 1);
                    }
                    cbar();
                    if (s_last && tid < 32) {
                        __threadfence();
                        double g4[NB_NP] = {0, 0, 0, 0, 0, 0, 0};
                        for (int gg = tid; gg < Gs; gg += 32) {
                            const double* hp = S.hpart + ((size_t)k * Gs + gg) * NB_NP;
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
                        if (tid == 0) {
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
                }
            }
            // ---- pass end: every set done; wait for the decisions of this pass's iterations
            __syncthreads();          // (A)
            const int kl = min(pass * D + D, S.newton_max) - 1;
            if (tid == 0) {
                unsigned v;
                for (;;) {
                    v = ps::ld_acq(S.decided + kl);
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
            }
            __syncthreads();          // (B)
            if (s_dec[0] != 2) break;
        }
        if (trace) {
            s_tr[PS_TR - 1] = clock64() - s_tm[0];
            for (int i = 0; i < PS_TR; ++i) S.trace[(size_t)c * PS_TR + i] = (unsigned long long)s_tr[i];
        }
        if (c == 0 && tid == 0) {
            S.info[0] = s_dec[1];
            S.info[1] = s_dec[0];
            // speculative iterations past the deciding one leave no history
            for (int kk = s_dec[1]; kk < S.newton_max && kk < MAXK && __ldcg(S.decided + kk) != 0u; ++kk) {
                for (int j = 0; j < 4; ++j) S.hist[4 * kk + j] = 0.0;
                if (S.linres) { S.linres[2 * kk] = 0.0; S.linres[2 * kk + 1] = 0.0; }
            }
            if (S.stats) {
                S.stats[0] = levels; S.stats[1] = (long long)SW;
                S.stats[2] = D; S.stats[3] = (long long)D * Gs; S.stats[4] = (long long)levels * SW; S.stats[5] = 0;
            }
        }
        if (c == 0 && tid == 0) *S.hint = s_dec[1];         // the next solve keeps that ring slot in its u_out
        copy_out(S, s_alias, s_dec[1]);
    }

    // The converged iterate (buffer kf % B) copied to u_out by every CTA of the grid.
    __device__ __forceinline__ static double* ring_buf(const PsParams& S, int alias, int i) {
        return i == alias ? S.u_out : S.U + (size_t)i * S.P.nt * S.P.ns;
    }
    // The converged iterate (buffer kf % B) copied to u_out by every CTA of the grid (unless it was written in place).
    __device__ __forceinline__ static void copy_out(const PsParams& S, int alias, int kf) {
        if (!S.u_out || kf % S.B == alias) return;
        const long long n2 = (long long)S.P.nt * S.P.ns / 2;
        const double2* src = reinterpret_cast<const double2*>(ring_buf(S, alias, kf % S.B));
        double2* dst = reinterpret_cast<double2*>(S.u_out);
        const long long stride = (long long)S.D * S.Gs * NTH;
        for (long long i = (long long)blockIdx.x * NTH + threadIdx.x; i < n2; i += stride) __stcs(dst + i, __ldcg(src + i));
    }
};

template <int NXU, int HE, bool PER, bool TRACE>
__global__ void __launch_bounds__(NXU, 1) k_newton_ps0(const PsParams S) {
    extern __shared__ __align__(128) double sm_ps0[];
    using E = PsEngine0<NXU, HE, PER, TRACE>;
    if ((int)blockIdx.x >= S.D * S.Gs) return;
    const int s = blockIdx.x % S.Gs;
    const int na = (S.P.nyu - HE * S.Gs) / 2;
    const bool up = (int)threadIdx.x >= NXU / 2;                 // the upper row group (warp-uniform)
    if (s < na) { if (up) E::template run<(HE + 2) / 2, 1>(S, sm_ps0); else E::template run<(HE + 2) / 2, 0>(S, sm_ps0); }
    else { if (up) E::template run<HE / 2, 1>(S, sm_ps0); else E::template run<HE / 2, 0>(S, sm_ps0); }
}

}  // namespace pit
