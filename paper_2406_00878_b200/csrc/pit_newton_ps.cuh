// pit_newton_ps.cuh — engine 5: the all-at-once Newton solve (Eq. (5)) with the exact block inverse
// of Eq. (7) applied as the level recurrence du^n = A_n^{-1}(r^n + du^{n-1}), as a PIPELINE OF CTA
// SETS: set p (Gs CTAs, one per SM) runs Newton iteration k = pass * D + p over the levels n = 1..nt, one level
// behind set p - 1, so D Newton iterations are in flight on D * Gs SMs (the level wavefront of DESIGN.md §6.1 laid
// out in space instead of interleaved in every CTA as in engine 4).
//
// Per level a CTA holds its strip of H rows (c5: 22 rows of 512) ENTIRELY on chip: du (x) in registers (a thread owns
// two adjacent columns of one half of the strip's rows: two row groups of NXU / 2 threads), u^n (with its two halo rows)
// and the right-hand side b = r^n + du^{n-1} in shared memory.  HBM/L2 traffic per (level, iteration): U_k^n read once (into registers, issued before the
// previous level's epilogue; u^{n-1} is still in shared memory from the previous level) and U_{k+1}^n written once —
// the 16 B per DOF per Newton iteration of SURVEY §8(d).
//
// Level solves: S red-black SOR sweeps from the carry, Young's omega from the Jacobi bound (as engine 4, whose
// device set-up kernels k_nb_q / k_nb_ctl are reused).  A half-sweep first turns every point of the OTHER colour into
// its four products with the coefficients its neighbours apply to it (one load of u, seven flops) and scatters them
// into per-row accumulators, so every value of u and x is touched once per half-sweep.  Synchronisation:
// neighbouring strips of a set exchange their boundary rows through LL cells (no fences, pit_newton_nb.cuh) once per
// half-sweep — the loads are issued before the strip's own products and consumed after them, boundary rows are
// relaxed and published first; set p - 1 hands U_k^n to set p through per-strip level counters (release / acquire)
// that thread 0 publishes and polls where it would wait for its neighbours anyway.  Columns of neighbouring threads
// meet through warp shuffles (warp edges through a small shared array).
//
// This engine covers LAW 1 (viscous Burgers, constant viscosity) on periodic grids with an even number of rows per
// strip; everything else runs on engines 1-4.
#pragma once
#include "pit_newton_nb.cuh"
#include "pit_ps_params.cuh"

namespace pit {

namespace ps {
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_wait(unsigned addr, unsigned parity) {
    unsigned ok;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
}  // namespace ps

// TRACE: the developer build (PIT_TRACE: cycle accounts of thread 0, the PIT_PS_DBG timing experiments); the product
// build has none of it compiled in (c5 24.3 -> 23.9 ms, c4 3.66 -> 3.48 ms).
template <int NXU, int HE, int RG, bool TRACE>
struct PsEngine {
    static_assert(RG == 1 || RG == 2, "one or two row groups");
    static constexpr int T = NXU / 2;          // threads per row group (two columns each)
    static constexpr int NW = T / 32;          // warps per row group
    static constexpr int NTH = RG * T;         // RG = 2: the lower and the upper half of the strip's rows
    static constexpr int HM = HE + 2;          // max strip height (strips have HE or HE + 2 rows, r0 even)
    static constexpr int HHM = HM / RG;        // max rows per thread
    static constexpr size_t OFF_U = 0;                                    // ubuf [HM + 2][NXU]: u^n rows r0-1 .. r0+H
    static constexpr size_t OFF_B = OFF_U + (size_t)(HM + 2) * NXU;       // bs   [HHM][2][NTH]
    static constexpr size_t OFF_A = OFF_B + (size_t)HHM * 2 * NTH;        // acc  [NB_NP][NTH] per-thread norm partials
    static constexpr size_t OFF_E = OFF_A + (size_t)NB_NP * NTH;          // wedge [RG groups][2 kinds][HHM][NW] warp-edge E/W products
    static constexpr size_t OFF_G = OFF_E + (size_t)RG * 2 * HHM * NW;    // gx   [2 colours][2][T] N/S products across the row groups
    static constexpr size_t OFF_R = OFF_G + (size_t)4 * T;                // red  [RG NW][NB_NP]
    static constexpr size_t OFF_S = OFF_R + (size_t)RG * NW * NB_NP;      // scalars shared by the two code paths (16 words)
    static constexpr size_t SMEM = (OFF_S + 16) * sizeof(double);

    // HH = rows per thread (H = 2 HH rows per strip).  Row group g owns strip rows g HH .. g HH + HH - 1.  When HH is
    // odd the upper group starts on an odd row: its threads hold their two columns SWAPPED (local column jj = actual
    // column ^ f), so that the colour of local point (q, jj) is (q + jj) & 1 in both groups and every register
    // subscript stays compile-time; the E/W roles then mirror, which only flips the sign of ax and the shuffle
    // direction (per-thread constants).
    // The row group is a template parameter (the kernel branches once, per warp): the column swap, the strip side
    // and every sign it implies are compile-time in each of the two code paths.
    template <int HH, bool ISO, int GRP>
    __device__ __forceinline__ static void run(const PsParams& S, double* sm) {
        constexpr int H = RG * HH;
        const Prob P = S.P;
        const int Gs = S.Gs, c = blockIdx.x, p = c / Gs, s = c % Gs;
        const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
        constexpr int g = GRP;
        const int t = tid % T, wl = w % NW;
        const int nyu = P.nyu, nt = P.nt, D = S.D, B = S.B;
        const long long ns = P.ns;
        const int na = (nyu - HE * Gs) / 2;                 // strips 0 .. na-1 have HE + 2 rows
        const int r0 = s * HE + 2 * min(s, na);             // first row of the strip (even)
        const int ss = s > 0 ? s - 1 : Gs - 1, sn = s + 1 < Gs ? s + 1 : 0;   // periodic neighbours (rows below / above)
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
        double* ub = ubuf + (size_t)(1 + g * HH) * NXU;      // the thread's local row 0 (rows -1 and HH exist too)
        double* bs = sm + OFF_B;
        double* accs = sm + OFF_A;
        double* wedge = sm + OFF_E + (size_t)g * 2 * HHM * NW;   // this group's [2 kinds][HHM][NW]
        double* gx0 = sm + OFF_G;                            // per colour: [0][t] lower group's top row -> upper, [1][t] upper's bottom row -> lower
        double* red_s = sm + OFF_R;

        // LL cells of a strip: [ring][side][t]; side 0 = its bottom row (published by the lower group), 1 = its top row
        unsigned long long* myx = S.llx + ((size_t)(p * Gs + s) * PS_RX * 2 * T) * 2;
        const unsigned long long* sbx = S.llx + ((size_t)(p * Gs + ss) * PS_RX * 2 * T) * 2;   // the strip below
        const unsigned long long* nbx = S.llx + ((size_t)(p * Gs + sn) * PS_RX * 2 * T) * 2;   // the strip above
        auto mycell = [&](unsigned q, int side) { return myx + ((size_t)((q % PS_RX) * 2 + side) * T + t) * 2; };
        auto scell = [&](unsigned q) { return sbx + ((size_t)((q % PS_RX) * 2 + 1) * T + t) * 2; };   // its top row
        auto ncell = [&](unsigned q) { return nbx + ((size_t)((q % PS_RX) * 2 + 0) * T + t) * 2; };   // its bottom row

        const double omega = __ldcg(S.ctl);
        const int SW = (int)__ldcg(S.ctl + 1);
        const int chk = max(1, (int)__ldcg(S.ctl + 3));
#define bx (S.bx)
#define ay (S.ay)
#define by (S.by)
#define aC1 (S.aC1)
#define tau (S.P.dt)
        const double a1 = f ? -S.ax : S.ax;                  // ax seen through the column swap
        const double sx2 = f ? -P.i2hx : P.i2hx;             // 1/(2 hx) seen through the column swap (residual)
        const double oic = omega * S.invC1, om1 = 1.0 - omega;     // x <- om1 x + oic (b - offdiag x)
        const double rsc = aC1 * (om1 / omega);                      // residual of a just-relaxed point: rsc (x_new - x_old)
        // kind A rows (other colour in local column 1): the product travels to thread t + 1 (f = 0) or t - 1 (f = 1);
        // kind B rows (other colour in local column 0): the opposite way.
        // (kind A values come from lane - 1 (f = 0) or lane + 1 (f = 1), kind B values from the other side)
        const int edgeA = f ? 31 : 0, edgeB = f ? 0 : 31;    // lanes whose source lies in the neighbouring warp
        const int wsA = f ? (wl + 1) % NW : (wl + NW - 1) % NW, wsB = f ? (wl + NW - 1) % NW : (wl + 1) % NW;
        double* wdA = wedge;                                 // [HHM][NW]
        double* wdB = wedge + (size_t)HHM * NW;
        int isA = lane == edgeA, isB = lane == edgeB;         // this lane's kind A / B source lies in the neighbouring warp
        const double mA = isA ? 0.0 : 1.0, mB = isB ? 0.0 : 1.0;
        int wrA = lane == 31 - edgeA, wrB = lane == 31 - edgeB;   // this lane's kind A / B product is a neighbouring warp's source
        unsigned wdA_w = (unsigned)__cvta_generic_to_shared(wdA + wl), wdB_w = (unsigned)__cvta_generic_to_shared(wdB + wl);
        // (opaque to the compiler, which otherwise rebuilds these from the thread index in every row of the sweeps)
        asm volatile("" : "+r"(isA), "+r"(isB), "+r"(wrA), "+r"(wrB), "+r"(wdA_w), "+r"(wdB_w));
        // ubuf rows are de-interleaved: [even columns (T)][odd columns (T)], so that a warp's loads of one local column
        // are contiguous (no bank conflicts).  Offsets of local columns 0 and 1, and of their out-of-thread x-neighbours
        // (actual column c0 - 1: odd, pair t - 1; actual column c0 + 2: even, pair t + 1; periodic).
        const int uo0 = f * T + t, uo1 = (1 - f) * T + t;
        const int cwest = T + (t + T - 1) % T, ceast = (t + 1) % T;
        const int co0 = f ? ceast : cwest, co1 = f ? cwest : ceast;

        auto cbar = [&]() { __syncthreads(); };
        auto bsm = [&](int r, int j) -> double& { return bs[(size_t)(r * 2 + j) * NTH + tid]; };
        auto ac = [&](int j) -> double& { return accs[(size_t)j * NTH + tid]; };
        auto lswap = [&](double2 v) { return f ? make_double2(v.y, v.x) : v; };   // actual <-> local column order

        double x[HH][2];
        #pragma unroll
        for (int j = 0; j < NB_NP; ++j) ac(j) = 0.0;
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
            if (pf_lv && fprev) { v0 = ps::ld_rlx(fprev + s); v1 = ps::ld_rlx(fprev + ss); v2 = ps::ld_rlx(fprev + sn); }
            const bool ready = pf_lv && min(v0, min(v1, v2)) >= base + (unsigned)pf_lv;
            if ((flag_lv || (ready && fprev)) && !(TRACE && (S.dbg & 2))) __threadfence();   // (dbg bit 1: timing experiment without the fence)
            if (flag_lv) {
                asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(fmine), "r"(base + (unsigned)flag_lv) : "memory");
                flag_lv = 0;
            }
            if (ready) pf_lv = 0;
        };

        // tt[q] = b - (off-diagonal part of A_n) x at the colour-cc point of every own row q (local column (q + cc) & 1).
        // Every point of the other colour is turned into its products with the coefficients its four neighbours apply
        // to it: a_E = ax u - bx (seen from its W neighbour), a_W = -ax u - bx, a_N = ay u - by (seen from the row
        // below), a_S = -ay u - by.  The product for the neighbouring THREAD travels by warp shuffle (warp edges through
        // shared memory), the one for the other row group through shared memory, and the neighbouring strip's row
        // arrives in an LL cell.
        auto gather = [&](const int cc, double (&tt)[HH], const bool svc, const unsigned fbase) {
            LLc hcs, hcn;                                    // RG = 2: a thread has one neighbouring strip (hcs holds its cell)
            const unsigned qn = (unsigned)lastx;
            if (lastx >= 0) {
                if constexpr (RG == 1) {
                    hcs = ll_issue(scell(qn));
                    hcn = ll_issue(ncell(qn));
                } else {
                    hcs = ll_issue(g ? ncell(qn) : scell(qn));
                }
            }
            if (svc && tid == 0 && (flag_lv | pf_lv)) service(fbase);
            double* gx = gx0 + (size_t)cc * 2 * T;           // double-buffered: a fast warp's next half-sweep writes the other half
            tt[0] = bsm(0, cc & 1);
            double bnext = HH > 1 ? bsm(1, (1 + cc) & 1) : 0.0;      // (right-hand sides run one row ahead, like u)
            double unext = ub[(1 - (cc & 1)) ? uo1 : uo0];       // (the loads of u run one row ahead of their use: c5 23.9 -> 23.2 ms)
            #pragma unroll
            for (int q = 0; q < HH; ++q) {
                const int jn = 1 - ((q + cc) & 1);               // the other colour's local column in this row
                const double uq = unext, xq = x[q][jn];
                if (q + 1 < HH) unext = ub[(size_t)(q + 1) * NXU + ((1 - ((q + 1 + cc) & 1)) ? uo1 : uo0)];
                if (q + 1 < HH) tt[q + 1 < HH ? q + 1 : q] = bnext;
                if (q + 2 < HH) bnext = bsm(q + 2, (q + 2 + cc) & 1);
                // (a1 u - bx) x and (-a1 u - bx) x = -(a1 u - bx) x - 2 bx x; the same in y (on an isotropic grid the y
                // products ARE the x products: the +a form is pa unless the columns are swapped)
                const double pa = fma(a1, uq, -bx) * xq, pb = fma(-2.0 * bx, xq, -pa);
                double pn, psv;
                if (ISO) {
                    pn = f ? pb : pa;
                    psv = f ? pa : pb;
                } else {
                    pn = fma(ay, uq, -by) * xq;
                    psv = fma(-2.0 * by, xq, -pn);
                }
                // the travelling product goes to the neighbouring thread at once (shuffle); the lanes whose source lies in
                // the neighbouring warp take theirs from shared memory behind the barrier instead
                if (jn == 1) {               // kind A: in-thread term pa, travelling term pb
                    const double in = f ? __shfl_down_sync(0xffffffffu, pb, 1) : __shfl_up_sync(0xffffffffu, pb, 1);
                    tt[q] -= pa;
                    tt[q] = fma(-mA, in, tt[q]);             // (mA = 0 on the lane whose source lies in the neighbouring warp)
                    if (wrA) wdA[q * NW + wl] = pb;
                } else {                     // kind B: in-thread term pb, travelling term pa
                    const double in = f ? __shfl_up_sync(0xffffffffu, pa, 1) : __shfl_down_sync(0xffffffffu, pa, 1);
                    tt[q] -= pb;
                    tt[q] = fma(-mB, in, tt[q]);
                    if (wrB) wdB[q * NW + wl] = pa;
                }
                if (q > 0) tt[q > 0 ? q - 1 : 0] -= pn;
                else if (RG == 2 && g == 1) gx[T + t] = pn;  // to the lower group's top row
                if (q + 1 < HH) tt[q + 1 < HH ? q + 1 : q] -= psv;
                else if (RG == 2 && g == 0) gx[t] = psv;     // to the upper group's bottom row
            }
            cbar();
            // the edge lanes' travelling products, from the neighbouring warp (every lane loads the broadcast value; the
            // complementary 0/1 factor keeps it out of the other lanes: no divergent branch)
            #pragma unroll
            for (int q = 0; q < HH; ++q) {
                if ((q + cc) & 1) tt[q] = fma(mB - 1.0, wdB[q * NW + wsB], tt[q]);      // kind B rows
                else tt[q] = fma(mA - 1.0, wdA[q * NW + wsA], tt[q]);                   // kind A rows: other colour in local column 1
            }
            // the row below local row 0 and the row above local row HH-1: the other row group or the neighbouring strip
            if (RG == 2) {
                if (g == 0) tt[HH - 1] -= gx[T + t]; else tt[0] -= gx[t];
            }
            if (lastx >= 0) {
                if constexpr (RG == 1) {
                    const double xs = take(scell(qn), hcs, qn + 1u), xn = take(ncell(qn), hcn, qn + 1u);
                    const double us = ub[-(ptrdiff_t)NXU + ((cc & 1) ? uo1 : uo0)];
                    const double un = ub[(size_t)HH * NXU + (((HH - 1 + cc) & 1) ? uo1 : uo0)];
                    tt[0] = fma(-fma(-ay, us, -by), xs, tt[0]);
                    tt[HH - 1] = fma(-fma(ay, un, -by), xn, tt[HH - 1]);
                } else if (g == 0) {
                    const double xh = take(scell(qn), hcs, qn + 1u);
                    const double uh = ub[-(ptrdiff_t)NXU + ((cc & 1) ? uo1 : uo0)];
                    tt[0] = fma(-fma(-ay, uh, -by), xh, tt[0]);
                } else {
                    const double xh = take(ncell(qn), hcs, qn + 1u);
                    const double uh = ub[(size_t)HH * NXU + (((HH - 1 + cc) & 1) ? uo1 : uo0)];
                    tt[HH - 1] = fma(-fma(ay, uh, -by), xh, tt[HH - 1]);
                }
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
                    ub[(size_t)r * NXU + t] = v.x;
                    ub[(size_t)r * NXU + T + t] = v.y;
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
                    double2 pf[HH + RG % 2 + 1];                    // own rows, then the strip's halo row(s) this thread stores
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) pf[r] = ldcg2(un + (size_t)(rg0 + r) * NXU);
                    if constexpr (RG == 1) {
                        pf[HH] = ldcg2(un + (size_t)((rg0 - 1 + nyu) % nyu) * NXU);
                        pf[HH + 1] = ldcg2(un + (size_t)((rg0 + HH) % nyu) * NXU);
                    } else {
                        pf[HH] = ldcg2(un + (size_t)(g ? (rg0 + HH) % nyu : (rg0 - 1 + nyu) % nyu) * NXU);
                    }
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        const double2 nw = lswap(pf[r]);
                        bsm(r, 0) = x[r][0] - (nw.x - ub[(size_t)r * NXU + uo0]);
                        bsm(r, 1) = x[r][1] - (nw.y - ub[(size_t)r * NXU + uo1]);
                        ub[(size_t)r * NXU + t] = pf[r].x;
                        ub[(size_t)r * NXU + T + t] = pf[r].y;
                    }
                    if constexpr (RG == 1) {
                        ub[-(ptrdiff_t)NXU + t] = pf[HH].x;
                        ub[-(ptrdiff_t)NXU + T + t] = pf[HH].y;
                        ub[(size_t)HH * NXU + t] = pf[HH + 1].x;
                        ub[(size_t)HH * NXU + T + t] = pf[HH + 1].y;
                    } else {
                        double* hrow = g ? ub + (size_t)HH * NXU : ub - (ptrdiff_t)NXU;
                        hrow[t] = pf[HH].x;
                        hrow[T + t] = pf[HH].y;
                    }
                }
                cbar();
                if (tid == 0 && n < nt) pf_lv = n + 1;
                mark(0);
                // ---- prologue 2: r^n = -G^n, b = r^n + du^{n-1} (local column order: the x-differences carry sx2)
                {
                    double ar2 = 0.0, arm = 0.0;
                    double p0 = ub[-(ptrdiff_t)NXU + uo0], p1 = ub[-(ptrdiff_t)NXU + uo1];
                    double c0v = ub[uo0], c1v = ub[uo1];
                    #pragma unroll
                    for (int r = 0; r < HH; ++r) {
                        const double n0 = ub[(size_t)(r + 1) * NXU + uo0], n1 = ub[(size_t)(r + 1) * NXU + uo1];
                        const double o0 = ub[(size_t)r * NXU + co0], o1 = ub[(size_t)r * NXU + co1];
                        // local column 0: x-neighbours o0 (outside) and c1v; local column 1: c0v and o1 (outside)
                        const double conv0 = 0.5 * ((c1v * c1v - o0 * o0) * sx2 + (n0 * n0 - p0 * p0) * P.i2hy);
                        const double visc0 = P.m0 * ((c1v - 2.0 * c0v + o0) * P.ihx2 + (n0 - 2.0 * c0v + p0) * P.ihy2);
                        const double conv1 = 0.5 * ((o1 * o1 - c0v * c0v) * sx2 + (n1 * n1 - p1 * p1) * P.i2hy);
                        const double visc1 = P.m0 * ((o1 - 2.0 * c1v + c0v) * P.ihx2 + (n1 - 2.0 * c1v + p1) * P.ihy2);
                        const double f0 = tau * (conv0 - visc0), f1 = tau * (conv1 - visc1);
                        const double b0 = bsm(r, 0), b1 = bsm(r, 1);
                        const double G0 = (x[r][0] - b0) + f0, G1 = (x[r][1] - b1) + f1;     // (u^n - u^{n-1}) + tau F(u^n)
                        bsm(r, 0) = b0 - f0;
                        bsm(r, 1) = b1 - f1;
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
                                const double xo = x[r][j], xn = fma(oic, tt[r], om1 * xo);
                                x[r][j] = xn;
                                const double rr = rsc * (xn - xo);
                                rs2 = fma(rr, rr, rs2);
                                rsm = fmax(rsm, fabs(rr));
                            }
                            if constexpr (RG == 1) {
                                ll_put(mycell(qx, 0), x[0][cc & 1], qx + 1u);
                                ll_put(mycell(qx, 1), x[HH - 1][(HH - 1 + cc) & 1], qx + 1u);
                            } else {
                                ll_put(mycell(qx, g), g ? x[HH - 1][(HH - 1 + cc) & 1] : x[0][cc & 1], qx + 1u);
                            }
                            ac(4) += rs2;
                            ac(5) = fmax(ac(5), rsm);
                        } else {
                            #pragma unroll
                            for (int i = 0; i < HH; ++i) {
                                const int r = i == 0 ? 0 : (i == 1 ? HH - 1 : i - 1);     // the two end rows first: one of them is the strip's boundary row
                                const int j = (r + cc) & 1;
                                const double xo = x[r][j];
                                x[r][j] = fma(oic, tt[r], om1 * xo);
                                if (i == (HH > 1 ? 1 : 0)) {     // publish the strip's boundary rows: local row 0 of the lower group, HH-1 of the upper
                                    if constexpr (RG == 1) {
                                        ll_put(mycell(qx, 0), x[0][cc & 1], qx + 1u);
                                        ll_put(mycell(qx, 1), x[HH - 1][(HH - 1 + cc) & 1], qx + 1u);
                                    } else {
                                        ll_put(mycell(qx, g), g ? x[HH - 1][(HH - 1 + cc) & 1] : x[0][cc & 1], qx + 1u);
                                    }
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
                        v.x = ub[(size_t)r * NXU + uo0] + x[r][0];
                        v.y = ub[(size_t)r * NXU + uo1] + x[r][1];
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
                        const double rr = tt[r] - aC1 * x[r][r & 1];
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
#undef bx
#undef ay
#undef by
#undef aC1
#undef tau
    }

    // The converged iterate (buffer kf % B) copied to u_out by every CTA of the grid.
    // Ring buffer i of the iterate ring; slot `alias` (if any) is the caller's u_out.
    __device__ __forceinline__ static double* ring_buf(const PsParams& S, int alias, int i) {
        return i == alias ? S.u_out : S.U + (size_t)i * S.P.nt * S.P.ns;
    }
    __device__ __forceinline__ static void copy_out(const PsParams& S, int alias, int kf) {
        if (!S.u_out || kf % S.B == alias) return;        // the final iterate was written in place
        const long long n2 = (long long)S.P.nt * S.P.ns / 2;
        const double2* src = reinterpret_cast<const double2*>(ring_buf(S, alias, kf % S.B));
        double2* dst = reinterpret_cast<double2*>(S.u_out);
        const long long stride = (long long)S.D * S.Gs * NTH;
        long long i = (long long)blockIdx.x * NTH + threadIdx.x;
        for (; i + 3 * stride < n2; i += 4 * stride) {
            const double2 a = __ldcg(src + i), b = __ldcg(src + i + stride), cc = __ldcg(src + i + 2 * stride), d = __ldcg(src + i + 3 * stride);
            __stcs(dst + i, a); __stcs(dst + i + stride, b); __stcs(dst + i + 2 * stride, cc); __stcs(dst + i + 3 * stride, d);
        }
        for (; i < n2; i += stride) __stcs(dst + i, __ldcg(src + i));
    }
};

template <int NXU, int HE, int RG, bool TRACE>
__global__ void __launch_bounds__(RG * NXU / 2, 1) k_newton_ps(const PsParams S) {
    extern __shared__ __align__(128) double sm_ps[];
    using E = PsEngine<NXU, HE, RG, TRACE>;
    if ((int)blockIdx.x >= S.D * S.Gs) return;
    const int s = blockIdx.x % S.Gs;
    const int na = (S.P.nyu - HE * S.Gs) / 2;
    const bool iso = S.ax == S.ay && S.bx == S.by;      // hx = hy: the y products of the sweeps are the x products
    const bool up = RG == 2 && (int)threadIdx.x >= NXU / 2;      // the upper row group (warp-uniform)
    if (s < na) {
        if (iso) { if (up) E::template run<(HE + 2) / RG, true, RG - 1>(S, sm_ps); else E::template run<(HE + 2) / RG, true, 0>(S, sm_ps); }
        else { if (up) E::template run<(HE + 2) / RG, false, RG - 1>(S, sm_ps); else E::template run<(HE + 2) / RG, false, 0>(S, sm_ps); }
    } else {
        if (iso) { if (up) E::template run<HE / RG, true, RG - 1>(S, sm_ps); else E::template run<HE / RG, true, 0>(S, sm_ps); }
        else { if (up) E::template run<HE / RG, false, RG - 1>(S, sm_ps); else E::template run<HE / RG, false, 0>(S, sm_ps); }
    }
}

}  // namespace pit
