// pit_newton_onchip.cuh — the ON-CHIP engine of the persistent Newton kernel (included by pit_kernels.cu).
//
// Same method and same wavefront schedule as k_newton (see pit_kernels.cu), re-laid out so that a
// per-level BiCGSTAB solve keeps its whole state in registers and shared memory for the duration of a
// wavefront step:
//   * one 256-thread CTA per SM (up to 255 registers per thread); a (level, iteration) pair owns a contiguous block of CTAs and every CTA
//     owns a strip of whole rows [r0, r1) of that level;
//   * per point, x, b~, r/s live in registers (PPT points per thread), p, v, t, 1/a_C in shared memory;
//   * u^n of the strip plus one halo row above/below and one halo column left/right (Dirichlet ring
//     or periodic wrap) is staged once per step in shared memory; the Jacobian coefficients of the
//     matvec are recomputed from it (Burgers: one FMA each), so no coefficient array exists at all;
//   * the matvec operand (p or s) is staged in shared memory; the two halo rows owned by neighbouring
//     CTAs are recomputed from the 4 (resp. 2) values those CTAs published for their boundary rows
//     before the last grid barrier, so each BiCGSTAB iteration needs exactly 2 grid barriers;
//   * grid barrier = one red.release.gpu per CTA on a monotonic counter + ld.acquire spin (1.2 us on
//     B200, profiles/r01_v1/microbench.txt), carrying an OR flag for the step-termination test;
//   * a pair that converges does its epilogue (U_{k+1}^n = U_k^n + du^n, carry) in the next phase
//     slot, overlapped with still-iterating pairs; the step ends at the first barrier where no pair is
//     left iterating: 2 * (max BiCGSTAB iterations of the step) + 2 grid barriers per wavefront step.
#pragma once

namespace pit {

constexpr int BLOCK2 = 512;
constexpr int NWARP2 = BLOCK2 / 32;

template <int NS, int NM, bool BCAST = true>
__device__ __forceinline__ void block_reduce2(double (&a)[NS + NM], double* sm) {
    // butterfly inside each warp, then warp 0 combines the NWARP2 per-warp values with a second (fixed)
    // butterfly: no serial loop over warps.  Result valid in thread 0.
    constexpr int N = NS + NM;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    auto op = [](int vi, double x, double y) { return vi < NS ? x + y : fmax(x, y); };
    if constexpr (N >= 4 && N <= 8 && NWARP2 == 16) {
        // transposed butterfly: every exchange halves the values a lane carries (padded to 8 with 0, which is
        // neutral for the sums and for the maxima of non-negative values): 4 + 2 + 1 + 1 + 1 shuffles instead
        // of 5 N; lane l ends with value 4 b4 + 2 b3 + b2 (b = bits of l) reduced over the warp
        const int h4 = (l >> 4) & 1, h3 = (l >> 3) & 1, h2 = (l >> 2) & 1;
        double c[4];
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double lo = j < N ? a[j] : 0.0, hi = j + 4 < N ? a[j + 4] : 0.0;
            c[j] = op(4 * h4 + j, h4 ? hi : lo, __shfl_xor_sync(0xffffffffu, h4 ? lo : hi, 16));
        }
        double d[2];
        #pragma unroll
        for (int j = 0; j < 2; ++j)
            d[j] = op(4 * h4 + 2 * h3 + j, h3 ? c[j + 2] : c[j], __shfl_xor_sync(0xffffffffu, h3 ? c[j] : c[j + 2], 8));
        const int vi = 4 * h4 + 2 * h3 + h2;
        double e = op(vi, h2 ? d[1] : d[0], __shfl_xor_sync(0xffffffffu, h2 ? d[0] : d[1], 4));
        e = op(vi, e, __shfl_xor_sync(0xffffffffu, e, 2));
        e = op(vi, e, __shfl_xor_sync(0xffffffffu, e, 1));
        if ((l & 3) == 0 && vi < N) sm[w * N + vi] = e;
        __syncthreads();
        if (w == 0) {
            // lane l: value i = l / 4 over warps l % 4, + 4, + 8, + 12 in that order, then a 4-lane butterfly;
            // value i ends in lane 4 i and is broadcast to the warp
            const int i = l >> 2, q = l & 3;
            double v = 0.0;
            if (i < N) {
                v = sm[q * N + i];
                #pragma unroll
                for (int m = 1; m < 4; ++m) v = op(i, v, sm[(q + 4 * m) * N + i]);
            }
            v = op(i, v, __shfl_xor_sync(0xffffffffu, v, 2));
            v = op(i, v, __shfl_xor_sync(0xffffffffu, v, 1));
            #pragma unroll
            for (int ii = 0; ii < N; ++ii) a[ii] = __shfl_sync(0xffffffffu, v, 4 * ii);
        }
        if (BCAST) __syncthreads();
        return;
    }
    if constexpr (N >= 3 && N <= 4 && NWARP2 == 16) {
        // the same for 3..4 values padded to 4: 2 + 1 + 1 + 1 + 1 shuffles; lane l ends with value 2 b4 + b3
        const int h4 = (l >> 4) & 1, h3 = (l >> 3) & 1;
        double c[2];
        #pragma unroll
        for (int j = 0; j < 2; ++j) {
            const double lo = a[j], hi = j + 2 < N ? a[j + 2] : 0.0;
            c[j] = op(2 * h4 + j, h4 ? hi : lo, __shfl_xor_sync(0xffffffffu, h4 ? lo : hi, 16));
        }
        const int vi = 2 * h4 + h3;
        double e = op(vi, h3 ? c[1] : c[0], __shfl_xor_sync(0xffffffffu, h3 ? c[0] : c[1], 8));
        e = op(vi, e, __shfl_xor_sync(0xffffffffu, e, 4));
        e = op(vi, e, __shfl_xor_sync(0xffffffffu, e, 2));
        e = op(vi, e, __shfl_xor_sync(0xffffffffu, e, 1));
        if ((l & 7) == 0 && vi < N) sm[w * N + vi] = e;
        __syncthreads();
        if (w == 0) {
            // lane l: value i = l / 8 over warps l % 8 and + 8, then an 8-lane butterfly; value i ends in lane 8 i
            const int i = l >> 3, q = l & 7;
            double v = 0.0;
            if (i < N) v = op(i, sm[q * N + i], sm[(q + 8) * N + i]);
            v = op(i, v, __shfl_xor_sync(0xffffffffu, v, 4));
            v = op(i, v, __shfl_xor_sync(0xffffffffu, v, 2));
            v = op(i, v, __shfl_xor_sync(0xffffffffu, v, 1));
            #pragma unroll
            for (int ii = 0; ii < N; ++ii) a[ii] = __shfl_sync(0xffffffffu, v, 8 * ii);
        }
        if (BCAST) __syncthreads();
        return;
    }
    #pragma unroll
    for (int i = 0; i < N; ++i)
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, a[i], o);
            a[i] = i < NS ? a[i] + y : fmax(a[i], y);
        }
    if (l == 0)
        #pragma unroll
        for (int i = 0; i < N; ++i) sm[w * N + i] = a[i];
    __syncthreads();
    if (w == 0) {
        #pragma unroll
        for (int i = 0; i < N; ++i) {
            double v = l < NWARP2 ? sm[l * N + i] : (i < NS ? 0.0 : 0.0);
            #pragma unroll
            for (int o = NWARP2 / 2; o > 0; o >>= 1) {
                const double y = __shfl_xor_sync(0xffffffffu, v, o);
                v = i < NS ? v + y : fmax(v, y);
            }
            a[i] = v;
        }
    }
    if (BCAST) __syncthreads();   // without it only warp 0 (thread 0) holds the result; sm is reused after a later barrier
}

// Fixed-order reduction of the per-CTA partials of CTAs [g0, g1) (NS sums then NM maxima), in ONE L2
// round trip: thread t loads CTA g0 + t's partials (C <= BLOCK2), warp 0 combines them in lane order.
constexpr int GMAX2 = 160;                         // max CTAs (= SMs) of the on-chip engine

template <int NS, int NM>
__device__ __forceinline__ void pair_reduce2(const double* part, int stride, int g0, int g1, double (&out)[NS + NM],
                                             double* sm /* >= GMAX2 * (NS + NM) + NS + NM */) {
    constexpr int N = NS + NM;
    const int C = g1 - g0;
    if ((int)threadIdx.x < C) {
        const double* pg = part + (long long)(g0 + threadIdx.x) * stride;
        #pragma unroll
        for (int i = 0; i < N; ++i) sm[i * GMAX2 + threadIdx.x] = __ldcg(pg + i);
    }
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {                      // warp 0 (a warp-uniform condition)
        double a[N];
        #pragma unroll
        for (int i = 0; i < N; ++i) a[i] = 0.0;
        for (int t = threadIdx.x; t < C; t += 32)
            #pragma unroll
            for (int i = 0; i < N; ++i) {
                const double y = sm[i * GMAX2 + t];
                a[i] = i < NS ? a[i] + y : fmax(a[i], y);
            }
        #pragma unroll
        for (int i = 0; i < N; ++i)
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double y = __shfl_xor_sync(0xffffffffu, a[i], o);
                a[i] = i < NS ? a[i] + y : fmax(a[i], y);
            }
        if (threadIdx.x == 0)
            #pragma unroll
            for (int i = 0; i < N; ++i) sm[N * GMAX2 + i] = a[i];
    }
    __syncthreads();
    #pragma unroll
    for (int i = 0; i < N; ++i) out[i] = sm[N * GMAX2 + i];
}

// Grid barrier of the on-chip engine, after the sm_70+ cooperative-groups pattern (bar.sync + one
// atom.release.gpu per CTA + ld.acquire.gpu polling + bar.sync), extended to carry an OR flag for free:
// two 64-bit monotonic counters alternate by episode parity; a CTA adds 1 + (flag << 32), so the low
// word counts arrivals and the high word counts flags.  Episode ep completes when the low word of
// ctr[ep & 1] reaches (ep / 2 + 1) * G; nothing else is added to that counter until every CTA has
// arrived at episode ep + 1, so the high word read at completion is exactly the flag count through
// episode ep and its increment over the previous same-parity episode is this episode's flag count.
__device__ __forceinline__ bool bar_sync(BarState* b, unsigned G, unsigned& ep, bool flag, unsigned (&hi)[2]) {
    __shared__ unsigned s_any;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* ctr = b->ctr + 16 * (ep & 1);
        const unsigned long long add = 1ull | ((unsigned long long)(flag ? 1u : 0u) << 32);
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(add) : "memory");
        const unsigned target = (ep / 2 + 1) * G;
        unsigned long long v;
        for (;;) {                                     // 32 ns back-off between polls (tools/barrier_bench.cu)
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if ((unsigned)v >= target) break;
            __nanosleep(32);
        }
        const unsigned h = (unsigned)(v >> 32);
        // static indices (a dynamic hi[ep & 1] would put the pair in local memory, on every barrier's path)
        const bool odd = (ep & 1) != 0;
        s_any = h != (odd ? hi[1] : hi[0]);
        if (odd) hi[1] = h; else hi[0] = h;
    }
    ++ep;
    __syncthreads();
    return s_any;
}

// bar_sync fused with the pair reduction: after thread 0's acquire, warps 0..N-1 each reduce one of the N values
// over the pair's CTAs [g0, g1): lane l loads the partials of CTAs g0 + l, g0 + l + 32, ... (all loads issued
// together: one L2 round trip) and sums them in that order, then a fixed butterfly — the same order for every
// value as a single-warp loop, so results are bit-identical run to run.  C = g1 - g0 <= GMAX2 = 160.
// pre() runs in every thread right after the barrier completes, before the partial loads: loads that only need
// the barrier (the halo rows the next phase reads) then share the partials' L2 round trip.
template <int NS, int NM, class Pre>
__device__ __forceinline__ bool bar_sync_reduce_pre(BarState* b, unsigned G, unsigned& ep, bool flag, unsigned (&hi)[2],
                                                    const double* part, int stride, int g0, int g1,
                                                    double (&out)[NS + NM], double* sm, Pre&& pre) {
    constexpr int N = NS + NM;
    constexpr int J = GMAX2 / 32;
    __shared__ unsigned s_any2;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* ctr = b->ctr + 16 * (ep & 1);
        const unsigned long long add = 1ull | ((unsigned long long)(flag ? 1u : 0u) << 32);
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(add) : "memory");
        const unsigned target = (ep / 2 + 1) * G;
        unsigned long long v;
        for (;;) {                                     // 32 ns back-off between polls (tools/barrier_bench.cu)
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if ((unsigned)v >= target) break;
            __nanosleep(32);
        }
        const unsigned h = (unsigned)(v >> 32);
        // static indices (a dynamic hi[ep & 1] would put the pair in local memory, on every barrier's path)
        const bool odd = (ep & 1) != 0;
        s_any2 = h != (odd ? hi[1] : hi[0]);
        if (odd) hi[1] = h; else hi[0] = h;
    }
    __syncthreads();
    pre();
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (w < N) {                                        // a warp-uniform condition
        double y[J];
        #pragma unroll
        for (int j = 0; j < J; ++j) {
            const int t = g0 + l + 32 * j;
            y[j] = t < g1 ? __ldcg(part + (long long)t * stride + w) : 0.0;
        }
        double a = 0.0;
        #pragma unroll
        for (int j = 0; j < J; ++j) a = w < NS ? a + y[j] : fmax(a, y[j]);
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double z = __shfl_xor_sync(0xffffffffu, a, o);
            a = w < NS ? a + z : fmax(a, z);
        }
        if (l == 0) sm[w] = a;
    }
    const bool any = s_any2;
    ++ep;
    __syncthreads();
    #pragma unroll
    for (int i = 0; i < N; ++i) out[i] = sm[i];
    return any;
}

template <int NS, int NM>
__device__ __forceinline__ bool bar_sync_reduce(BarState* b, unsigned G, unsigned& ep, bool flag, unsigned (&hi)[2],
                                                const double* part, int stride, int g0, int g1, double (&out)[NS + NM],
                                                double* sm) {
    return bar_sync_reduce_pre<NS, NM>(b, G, ep, flag, hi, part, stride, g0, g1, out, sm, [] {});
}

// u at unknown (gc, gr) of level n, extended by the Dirichlet ring (Eq. 2) or the periodic wrap.
__device__ __forceinline__ double node_ext(const Prob& P, const double* __restrict__ U, const double* __restrict__ ringn,
                                           int gr, int gc) {
    if (P.bc == 1) {
        gr = gr < 0 ? gr + P.nyu : (gr >= P.nyu ? gr - P.nyu : gr);
        gc = gc < 0 ? gc + P.nxu : (gc >= P.nxu ? gc - P.nxu : gc);
        return __ldcg(U + (long long)gr * P.nxu + gc);
    }
    const bool in_r = gr >= 0 && gr < P.nyu, in_c = gc >= 0 && gc < P.nxu;
    if (in_r && in_c) return __ldcg(U + (long long)gr * P.nxu + gc);
    if (!ringn || (!in_r && !in_c)) return 0.0;          // corners are never used by the 5-point stencil
    const int nxp = P.nx + 1;
    if (gr < 0) return __ldcg(ringn + gc + 1);                         // bottom, paper node (gc+1, 0)
    if (gr >= P.nyu) return __ldcg(ringn + nxp + gc + 1);              // top, (gc+1, ny)
    if (gc < 0) return __ldcg(ringn + 2 * nxp + gr);                   // left, (0, gr+1)
    return __ldcg(ringn + 2 * nxp + (P.ny - 1) + gr);                  // right, (nx, gr+1)
}

// Off-diagonal Jacobian coefficients for the matvec.  LAW 1 = viscous Burgers with constant viscosity
// (f = g = u^2/2, mu = m0: a_E = tau (u_E / 2h - mu / h^2), ...), LAW 0 = the general law of Eq. (1).
template <int LAW>
__device__ __forceinline__ Off offdiag_law(const Prob& P, const Vals& v) {
    if (LAW == 1) {
        const double cx = P.dt * P.i2hx, cy = P.dt * P.i2hy, dx = P.dt * P.m0 * P.ihx2, dy = P.dt * P.m0 * P.ihy2;
        Off o;
        o.e = fma(cx, v.e, -dx);
        o.w = fma(-cx, v.w, -dx);
        o.n = fma(cy, v.n, -dy);
        o.s = fma(-cy, v.s, -dy);
        return o;
    }
    return offdiag(P, v);
}

// ---- hot per-point loops, as functions with __restrict__ shared-memory operands (the strip arrays are
// disjoint regions of one dynamic shared buffer; without the qualifier every store would fence the next
// point's loads) ----------------------------------------------------------------------------------------
template <int LAW>
__device__ __forceinline__ double scaled_matvec(const Prob& P, int c0, int l, int W, const double* __restrict__ u_s,
                                                const double* __restrict__ op_s, const double* __restrict__ ci_s) {
    const Vals uv = {u_s[c0], u_s[c0 + 1], u_s[c0 - 1], u_s[c0 + W], u_s[c0 - W]};
    const Off o = offdiag_law<LAW>(P, uv);
    return op_s[c0] + ci_s[l] * (o.e * op_s[c0 + 1] + o.w * op_s[c0 - 1] + o.n * op_s[c0 + W] + o.s * op_s[c0 - W]);
}

// phase 1, own points: r = s - omega t, x += alpha p + omega s (pending), p = r + beta (p - omega v)
template <int PPT>
__device__ __forceinline__ void p_update(int tid, int W, const int (&lrr)[PPT], double (&x)[PPT], double (&sr)[PPT],
                                         const double (&bt)[PPT], bool first, bool pending, double alpha, double omega,
                                         double beta, double* __restrict__ p_s, const double* __restrict__ v_s,
                                         const double* __restrict__ t_s, double* __restrict__ op_s) {
    #pragma unroll
    for (int m = 0; m < PPT; ++m) {
        const int l = tid + m * BLOCK2;
        const int lr = lrr[m];
        if (lr < 0) continue;
        double pn;
        if (first) {
            pn = bt[m];
        } else {
            const double pold = p_s[l];
            const double r = sr[m] - omega * t_s[l];
            if (pending) x[m] += alpha * pold + omega * sr[m];
            pn = r + beta * (pold - omega * v_s[l]);
            sr[m] = r;
        }
        p_s[l] = pn;
        op_s[l + 2 * lr + W + 1] = pn;
    }
}

// phase 1 matvec pass (interior rows, or the two boundary rows): v = D^{-1} A p, (b~, v), publish r, v
template <int PPT, int LAW>
__device__ __forceinline__ void v_pass(bool boundary, const Prob& P, int tid, int h, int W, const int (&lrr)[PPT],
                                       const double (&bt)[PPT], const double (&sr)[PPT], long long qbase,
                                       const double* __restrict__ u_s, const double* __restrict__ op_s,
                                       const double* __restrict__ ci_s, double* __restrict__ v_s,
                                       double* __restrict__ pR, double* __restrict__ pV2, double& acc) {
    #pragma unroll
    for (int m = 0; m < PPT; ++m) {
        const int l = tid + m * BLOCK2;
        const int lr = lrr[m];
        if (lr < 0 || (lr == 0 || lr == h - 1) != boundary) continue;
        const double vv = scaled_matvec<LAW>(P, l + 2 * lr + W + 1, l, W, u_s, op_s, ci_s);
        v_s[l] = vv;
        acc += bt[m] * vv;
        if (boundary) {
            pR[qbase + l] = sr[m];
            pV2[qbase + l] = vv;
        }
    }
}

// phase 2, own points: s = r - alpha v
template <int PPT>
__device__ __forceinline__ void s_update(int tid, int W, const int (&lrr)[PPT], double (&sr)[PPT], double alpha,
                                         const double* __restrict__ v_s, double* __restrict__ op_s) {
    #pragma unroll
    for (int m = 0; m < PPT; ++m) {
        const int l = tid + m * BLOCK2;
        const int lr = lrr[m];
        if (lr < 0) continue;
        const double s = sr[m] - alpha * v_s[l];
        sr[m] = s;
        op_s[l + 2 * lr + W + 1] = s;
    }
}

// phase 2 matvec pass: t = D^{-1} A s, the five dots, publish s, t, p, v of the boundary rows
template <int PPT, int LAW>
__device__ __forceinline__ void t_pass(bool boundary, const Prob& P, int tid, int h, int W, const int (&lrr)[PPT],
                                       const double (&bt)[PPT], const double (&sr)[PPT], long long qbase,
                                       const double* __restrict__ u_s, const double* __restrict__ op_s,
                                       const double* __restrict__ ci_s, double* __restrict__ t_s,
                                       const double* __restrict__ p_s, const double* __restrict__ v_s,
                                       double* __restrict__ pS, double* __restrict__ pT, double* __restrict__ pP,
                                       double* __restrict__ pV, double (&a)[5]) {
    #pragma unroll
    for (int m = 0; m < PPT; ++m) {
        const int l = tid + m * BLOCK2;
        const int lr = lrr[m];
        if (lr < 0 || (lr == 0 || lr == h - 1) != boundary) continue;
        const double s = sr[m];
        const double t = scaled_matvec<LAW>(P, l + 2 * lr + W + 1, l, W, u_s, op_s, ci_s);
        t_s[l] = t;
        a[0] += t * s; a[1] += t * t; a[2] += bt[m] * s; a[3] += bt[m] * t; a[4] += s * s;
        if (boundary) {
            const long long q = qbase + l;
            pS[q] = s; pT[q] = t; pP[q] = p_s[l]; pV[q] = v_s[l];
        }
    }
}

// Optional cycle accounting (S.trace != nullptr, env PIT_TRACE=1): per-CTA clock64 time per category,
// summed over CTAs: 0 prologue, 1 phase-1 work, 2 phase-2 work, 3 epilogue, 4 grid barriers,
// 5 scalar reductions after barriers, 6 end-of-step bookkeeping.
#define PMARK(cat)                                                       \
    do {                                                                 \
        if (TRACE) {                                                     \
            const long long t_ = clock64();                              \
            prof[cat] += t_ - t_last;                                    \
            t_last = t_;                                                 \
        }                                                                \
    } while (0)

template <int PPT, bool TRACE, int LAW>
__global__ void __launch_bounds__(BLOCK2, 1) k_newton_onchip(SolveParams S) {
    static_assert(BLOCK2 * NPART >= 4 * MAXD, "pair results live in red[]");
    extern __shared__ double smem[];
    const Prob P = S.P;
    const long long ns = P.ns;
    const int nxu = P.nxu, nyu = P.nyu;
    const int G = S.G, g = blockIdx.x, tid = threadIdx.x;
    const int W = nxu + 2;                         // shared row pitch: halo column each side
    const int HR = S.hmax + 2;                     // shared rows: halo row each side
    double* u_s = smem;                            // [HR][W]  u^n_k of the strip (+ halo / ring)
    double* op_s = u_s + HR * W;                   // [HR][W]  matvec operand
    double* p_s = op_s + HR * W;                   // [PPT][BLOCK2]
    double* v_s = p_s + PPT * BLOCK2;
    double* ci_s = v_s + PPT * BLOCK2;             // 1 / a_C
    double* t_s = ci_s + PPT * BLOCK2;             // t = A s (lives from phase 2 to the next phase 1)
    __shared__ int sS[MAXK];
    __shared__ double red[NWARP2 * NPART];
    __shared__ double s_hp_big[4 * GMAX2];        // end-of-step norm partials of all CTAs
    __shared__ double s_red[5 * GMAX2 + 8];       // pair_reduce2 staging
    __shared__ double pr[NPART];
    __shared__ double hacc[MAXD][4];
    __shared__ double prevmax_s;
    if (tid == 0) {
        const int D = S.D;
        for (int k = 0; k < S.newton_max; ++k) {
            int st = k == 0 ? 1 : sS[k - 1] + 1;
            if (k >= D && sS[k - D] + P.nt > st) st = sS[k - D] + P.nt;
            sS[k] = st;
        }
        prevmax_s = INFINITY;
    }
    if (tid < MAXD * 4) hacc[tid / 4][tid % 4] = 0.0;
    __syncthreads();

    unsigned ep = 0;
    unsigned hi[2] = {0u, 0u};                    // thread 0: flag counts seen at the last barriers
    long long prof[7] = {0, 0, 0, 0, 0, 0, 0};
    long long t_last = clock64();
    auto flush_prof = [&]() {
        if (TRACE && tid == 0)
            for (int j = 0; j < 7; ++j) atomicAdd(S.trace + j, (unsigned long long)prof[j]);
    };
    const int newton_max = S.mode == 0 ? S.newton_max : 1;
    int set = 0, klo = 0, last_done = -1;
    long long total_inner = 0;
    const double rtol2 = S.lin_rtol * S.lin_rtol;
    const double atol2 = S.lin_atol * S.lin_atol * (double)P.ns;     // lin_atol bounds the RMS residual

    for (int step = 1;; ++step) {
        while (klo < newton_max && step > sS[klo] + P.nt - 1) ++klo;
        int ks[MAXD];
        int A = 0;
        for (int k = klo; k < newton_max && A < MAXD && sS[k] <= step; ++k) ks[A++] = k;
        if (S.mode == 1) { A = S.nb; for (int a = 0; a < A; ++a) ks[a] = a; }
        int me = 0;
        while (me + 1 < A && (long long)(me + 1) * G / A <= g) ++me;
        const int g0 = (int)((long long)me * G / A), g1 = (int)((long long)(me + 1) * G / A);
        const int kme = ks[me];
        const int n = S.mode == 1 ? S.blev[me] : step - sS[kme] + 1;
        const int slot = kme % S.D;
        const int buf = kme % S.B, nbuf = (kme + 1) % S.B;
        const Slot sl = slot_at(S.slotmem, ns, slot);
        // published boundary-row values (full-level arrays, only strip boundary rows are touched)
        double* const pBT = sl.bt;  double* const pX = sl.x;
        double* const pS = sl.s;    double* const pT = sl.t;  double* const pP = sl.p[0];  double* const pV = sl.v[0];
        double* const pR = sl.r;    double* const pV2 = sl.v[1];
        const int c = g - g0, C = g1 - g0;
        const int r0 = (int)((long long)c * nyu / C), r1 = (int)((long long)(c + 1) * nyu / C);
        const int h = r1 - r0, npts = h * nxu;
        const double* Ulev = S.mode == 1 ? S.U + (long long)(n - 1) * ns : S.U + ((long long)buf * P.nt + (n - 1)) * ns;
        const double* uprev = n == 1 ? S.u0 : Ulev - ns;
        const double* ringn = S.ring ? S.ring + (long long)(n - 1) * P.ring_len : nullptr;
        double* Unew = S.mode == 1 ? nullptr : S.U + ((long long)nbuf * P.nt + (n - 1)) * ns;
        double* hp = S.hpart + (long long)(step & 1) * G * 4;
        const bool top_valid = P.bc == 1 || r0 > 0, bot_valid = P.bc == 1 || r1 < nyu;
        const int top_row = r0 == 0 ? nyu - 1 : r0 - 1, bot_row = r1 == nyu ? 0 : r1;

        double x[PPT], bt[PPT], sr[PPT];
        int lrr[PPT];                              // strip-local row of point m (-1: no point)
        #pragma unroll
        for (int m = 0; m < PPT; ++m) {
            const int l = tid + m * BLOCK2;
            lrr[m] = l < npts ? l / nxu : -1;
        }
        const long long qbase = (long long)r0 * nxu;   // global index of point m = qbase + l

        // ---- prologue: stage u, fused residual + Jacobian diagonal (kernel a), carry, scaling ----
        // Every global read of the prologue is issued before the first wait: u rows r0-1 .. r1 by cp.async,
        // u^{n-1} and the carry of the own points and the carry halo rows into registers.
        const bool x0c = S.x0carry && S.mode == 0 && n > 1;
        for (int idx = tid; idx < (h + 2) * W; idx += BLOCK2) {
            const int srow = idx / W, scol = idx - srow * W;
            int gr = r0 - 1 + srow, gc = scol - 1;
            bool inside = true;
            if (P.bc == 1) {
                gr = gr < 0 ? gr + nyu : (gr >= nyu ? gr - nyu : gr);
                gc = gc < 0 ? gc + nxu : (gc >= nxu ? gc - nxu : gc);
            } else {
                inside = gr >= 0 && gr < nyu && gc >= 0 && gc < nxu;
                if (scol == 0 || scol == W - 1) op_s[idx] = 0.0;   // Dirichlet: dropped columns stay 0
            }
            if (inside) {
                const unsigned dst = (unsigned)__cvta_generic_to_shared(u_s + idx);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(Ulev + (long long)gr * nxu + gc)
                             : "memory");
            } else {
                u_s[idx] = node_ext(P, Ulev, ringn, r0 - 1 + srow, scol - 1);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        double xh[2] = {0.0, 0.0};                 // carry on the halo rows (x0 = du^{n-1} operand)
        #pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int idx = tid + j * BLOCK2;
            if (x0c && h > 0 && idx < 2 * nxu) {
                const int side = idx >= nxu, col = side ? idx - nxu : idx;
                if (side ? bot_valid : top_valid) xh[j] = __ldcg(pX + (long long)(side ? bot_row : top_row) * nxu + col);
            }
        }
        {
            double a[4] = {0.0, 0.0, 0.0, 0.0};  // sum r0^2, sum r^2, sum b~^2 | max |r|   (r0 = b~ - A~ x0)
            #pragma unroll
            for (int m = 0; m < PPT; ++m) {
                const long long q = qbase + tid + m * BLOCK2;
                bt[m] = 0.0; sr[m] = 0.0;
                if (lrr[m] >= 0) {
                    if (S.mode == 1) {
                        sr[m] = __ldcg(S.bptr[me] + q);
                    } else {
                        bt[m] = __ldcg(uprev + q);
                        sr[m] = n == 1 ? 0.0 : __ldcg(pX + q);
                    }
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            #pragma unroll
            for (int m = 0; m < PPT; ++m) {
                const int l = tid + m * BLOCK2;
                x[m] = 0.0;
                if (lrr[m] >= 0) {
                    const int lr = lrr[m];
                    const int c0 = l + 2 * lr + W + 1;
                    const long long q = qbase + l;
                    const Vals v = {u_s[c0], u_s[c0 + 1], u_s[c0 - 1], u_s[c0 + W], u_s[c0 - W]};
                    const RJ o = residual_jacobian_raw(P, v, bt[m]);
                    double rhs;
                    if (S.mode == 1) {
                        rhs = sr[m];
                    } else {
                        const double r = -o.G;
                        a[1] += r * r;
                        a[3] = fmax(a[3], fabs(r));
                        rhs = r + sr[m];                   // r^n + du^{n-1}  (row n of Eq. 7)
                    }
                    const double ci = 1.0 / o.aC;
                    ci_s[l] = ci;
                    x[m] = x0c ? sr[m] : 0.0;              // initial guess: the carry du^{n-1}, or 0
                    bt[m] = rhs * ci;                      // b~ (kept in bt until r0 is known)
                    a[2] += bt[m] * bt[m];
                    if (x0c) op_s[c0] = x[m];
                }
            }
            if (x0c) {
                // r0 = b~ - A~ x0 with x0 = du^{n-1}: the operand halo rows are the carry of the
                // neighbouring strips (written for every point by the previous step's epilogue)
                #pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int idx = tid + j * BLOCK2;
                    if (h > 0 && idx < 2 * nxu) {
                        const int side = idx >= nxu, col = side ? idx - nxu : idx;
                        op_s[(side ? h + 1 : 0) * W + col + 1] = xh[j];
                    }
                }
                __syncthreads();
                if (P.bc == 1)
                    for (int rr = tid; rr < h + 2; rr += BLOCK2) {
                        op_s[rr * W] = op_s[rr * W + nxu];
                        op_s[rr * W + nxu + 1] = op_s[rr * W + 1];
                    }
                __syncthreads();
            }
            #pragma unroll
            for (int m = 0; m < PPT; ++m) {
                const int l = tid + m * BLOCK2;
                if (lrr[m] >= 0) {
                    const int lr = lrr[m];
                    const int c0 = l + 2 * lr + W + 1;
                    if (x0c) {
                        const Vals uv = {u_s[c0], u_s[c0 + 1], u_s[c0 - 1], u_s[c0 + W], u_s[c0 - W]};
                        const Off o = offdiag_law<LAW>(P, uv);
                        bt[m] -= op_s[c0] + ci_s[l] * (o.e * op_s[c0 + 1] + o.w * op_s[c0 - 1] + o.n * op_s[c0 + W] +
                                                       o.s * op_s[c0 - W]);
                    }
                    sr[m] = bt[m];                         // r0, and the BiCGSTAB shadow vector r^0 = r0
                    a[0] += bt[m] * bt[m];
                    if (lr == 0 || lr == h - 1) pBT[qbase + l] = bt[m];
                }
            }
            block_reduce2<3, 1>(a, red);
            if (tid == 0) {
                S.part[((long long)set * G + g) * NPART] = a[0];
                S.part[((long long)set * G + g) * NPART + 1] = a[2];
                hp[g * 4 + 0] = a[1];
                hp[g * 4 + 1] = a[3];
            }
        }
        PMARK(0);
        bar_sync(S.bs, G, ep, false, hi);
        PMARK(4);
        double bnorm2, rho;
        {
            double o[2];
            pair_reduce2<2, 0>(S.part + (long long)set * G * NPART, NPART, g0, g1, o, s_red);
            rho = o[0];                          // (r^0, r0) = ||r0||^2
            bnorm2 = o[1];                       // ||b~||^2: reference of the relative stopping test
        }
        PMARK(5);
        set ^= 1;
        double alpha = 0.0, omega = 1.0, beta = 0.0;
        bool conv = rho <= atol2 || rho <= rtol2 * bnorm2, pending = false, epi_done = false;
        int it = 0, maxit_step = 0;

        // periodic halo columns of the strip's own rows (the halo rows' wrap cells are never read)
        auto fill_wrap_own = [&]() {
            if (P.bc == 1)
                for (int rr = 1 + tid; rr <= h; rr += BLOCK2) {
                    op_s[rr * W] = op_s[rr * W + nxu];
                    op_s[rr * W + nxu + 1] = op_s[rr * W + 1];
                }
        };
        // scaled matvec (D^{-1} A op) at own point l of strip row lr; A_n recomputed from the staged u
        auto matvec_at = [&](int l, int lr) -> double {
            const int c0 = l + 2 * lr + W + 1;
            const Vals uv = {u_s[c0], u_s[c0 + 1], u_s[c0 - 1], u_s[c0 + W], u_s[c0 - W]};
            const Off o = offdiag_law<LAW>(P, uv);
            return op_s[c0] + ci_s[l] * (o.e * op_s[c0 + 1] + o.w * op_s[c0 - 1] + o.n * op_s[c0 + W] + o.s * op_s[c0 - W]);
        };
        // operand halo rows + periodic halo columns, then the scaled matvec y = D^{-1} A op at own points
        auto fill_wrap = [&]() {
            if (P.bc == 1)
                for (int rr = tid; rr < h + 2; rr += BLOCK2) {
                    op_s[rr * W] = op_s[rr * W + nxu];
                    op_s[rr * W + nxu + 1] = op_s[rr * W + 1];
                }
        };

        for (;;) {
            // ================= phase-1 slot: p update + v = A p  |  epilogue of converged pairs ======
            if (!conv) {
                double a[1] = {0.0};
                // halo operand (2 rows owned by the neighbour CTAs): issue the L2 loads first so their
                // latency overlaps the own-point update below (2 nxu <= 4 BLOCK2: <= 4 per thread)
                double hq[2][4];
                #pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int idx = tid + j * BLOCK2;
                    hq[j][0] = hq[j][1] = hq[j][2] = hq[j][3] = 0.0;
                    if (h > 0 && idx < 2 * nxu) {
                        const int side = idx >= nxu, col = side ? idx - nxu : idx;
                        if (side ? bot_valid : top_valid) {
                            const long long q = (long long)(side ? bot_row : top_row) * nxu + col;
                            if (it == 0) {
                                hq[j][0] = __ldcg(pBT + q);
                            } else {
                                hq[j][0] = __ldcg(pS + q); hq[j][1] = __ldcg(pT + q);
                                hq[j][2] = __ldcg(pP + q); hq[j][3] = __ldcg(pV + q);
                            }
                        }
                    }
                }
                p_update<PPT>(tid, W, lrr, x, sr, bt, it == 0, pending, alpha, omega, beta, p_s, v_s, t_s, op_s);
                pending = false;
                __syncthreads();
                fill_wrap_own();
                __syncthreads();
                // interior rows first: their neighbours are all local, so the L2 latency of the halo loads
                // issued at the top of the phase is hidden behind this pass
                auto vpass = [&](bool boundary) {
                    v_pass<PPT, LAW>(boundary, P, tid, h, W, lrr, bt, sr, qbase, u_s, op_s, ci_s, v_s, pR, pV2, a[0]);
                };
                vpass(false);
                #pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int idx = tid + j * BLOCK2;
                    if (h > 0 && idx < 2 * nxu) {
                        const int side = idx >= nxu, col = side ? idx - nxu : idx;
                        const double val = it == 0 ? hq[j][0]
                                                   : (hq[j][0] - omega * hq[j][1]) + beta * (hq[j][2] - omega * hq[j][3]);
                        op_s[(side ? h + 1 : 0) * W + col + 1] = val;
                    }
                }
                __syncthreads();
                vpass(true);
                block_reduce2<1, 0>(a, red);
                if (tid == 0) S.part[((long long)set * G + g) * NPART] = a[0];
                PMARK(1);
            } else if (!epi_done) {
                // epilogue: du^n = x (+ the pending last update), U_{k+1}^n = U_k^n + du^n, carry
                double a[3] = {0.0, 0.0, 0.0};
                #pragma unroll
                for (int m = 0; m < PPT; ++m) {
                    const int l = tid + m * BLOCK2;
                    if (lrr[m] >= 0) {
                        const int lr = lrr[m];
                        const int i = l;
                        const long long q = qbase + l;
                        double dx = x[m];
                        if (pending) dx += alpha * p_s[i] + omega * sr[m];
                        if (S.mode == 1) S.xptr[me][q] = dx;
                        else {
                            pX[q] = dx;
                            Unew[q] = u_s[l + 2 * lr + W + 1] + dx;
                        }
                        a[0] += dx * dx;
                        a[1] = fmax(a[1], fabs(dx));
                        if (!isfinite(dx)) a[2] = 1.0;
                    }
                }
                block_reduce2<1, 2>(a, red);
                if (tid == 0) {
                    hp[g * 4 + 2] = a[0];
                    hp[g * 4 + 3] = a[1];
                    if (a[2] != 0.0) atomicOr(&S.bs->err, 1u);
                }
                epi_done = true;
                pending = false;
                PMARK(3);
            }
            const bool any = bar_sync(S.bs, G, ep, !conv, hi);
            PMARK(4);
            if (!any) { set ^= 1; break; }
            double r0v = 0.0;
            if (!conv) {
                double o[1];
                pair_reduce2<1, 0>(S.part + (long long)set * G * NPART, NPART, g0, g1, o, s_red);
                r0v = o[0];
            }
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
            // ================= phase 2: s = r - alpha v, t = A s ====================================
            if (!conv) {
                double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};   // (t,s) (t,t) (b~,s) (b~,t) (s,s)
                double hq[2][2];
                #pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int idx = tid + j * BLOCK2;
                    hq[j][0] = hq[j][1] = 0.0;
                    if (h > 0 && idx < 2 * nxu) {
                        const int side = idx >= nxu, col = side ? idx - nxu : idx;
                        if (side ? bot_valid : top_valid) {
                            const long long q = (long long)(side ? bot_row : top_row) * nxu + col;
                            hq[j][0] = __ldcg(pR + q); hq[j][1] = __ldcg(pV2 + q);
                        }
                    }
                }
                s_update<PPT>(tid, W, lrr, sr, alpha, v_s, op_s);
                __syncthreads();
                fill_wrap_own();
                __syncthreads();
                auto tpass = [&](bool boundary) {
                    t_pass<PPT, LAW>(boundary, P, tid, h, W, lrr, bt, sr, qbase, u_s, op_s, ci_s, t_s, p_s, v_s, pS, pT, pP,
                                     pV, a);
                };
                tpass(false);
                #pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int idx = tid + j * BLOCK2;
                    if (h > 0 && idx < 2 * nxu) {
                        const int side = idx >= nxu, col = side ? idx - nxu : idx;
                        op_s[(side ? h + 1 : 0) * W + col + 1] = hq[j][0] - alpha * hq[j][1];
                    }
                }
                __syncthreads();
                tpass(true);
                block_reduce2<5, 0>(a, red);
                if (tid == 0) {
                    double* pp = S.part + ((long long)set * G + g) * NPART;
                    for (int j = 0; j < 5; ++j) pp[j] = a[j];
                }
                PMARK(2);
            }
            bar_sync(S.bs, G, ep, false, hi);
            PMARK(4);
            if (!conv) {
                double o[5];
                pair_reduce2<5, 0>(S.part + (long long)set * G * NPART, NPART, g0, g1, o, s_red);
                const double ts = o[0], tt2 = o[1], r0s = o[2], r0t = o[3], ss = o[4];
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
            }
            set ^= 1;
            maxit_step = it > maxit_step ? it : maxit_step;
            PMARK(5);
        }
        // the epilogue of a pair that was converged from the start happened in the first phase slot

        // ---- norms of the finished levels -> per-iteration accumulators; stop rule (as k_newton) ----
        const unsigned err = *((volatile unsigned*)&S.bs->err);
        int stop_status = 2, stop_k = -1;
        // one round trip: all CTAs' norm partials -> shared, then one warp per pair reduces its range
        {
            double* s_hp = red;                              // G * 4 doubles fit? (G <= 160 -> 640)
            for (int j = tid; j < G * 4; j += BLOCK2) s_hp_big[j] = __ldcg(hp + j);
            __syncthreads();
            const int w = tid >> 5, lane = tid & 31;
            if (w < A) {
                const int ga0 = (int)((long long)w * G / A), ga1 = (int)((long long)(w + 1) * G / A);
                double a4[4] = {0.0, 0.0, 0.0, 0.0};
                for (int gg = ga0 + lane; gg < ga1; gg += 32) {
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
                if (lane == 0) for (int j = 0; j < 4; ++j) s_hp[w * 4 + j] = a4[j];
            }
            __syncthreads();
            (void)s_hp;
        }
        for (int a = 0; a < A; ++a) {
            const double o[4] = {red[a * 4 + 0], red[a * 4 + 1], red[a * 4 + 2], red[a * 4 + 3]};
            const int k = ks[a];
            const int na = S.mode == 1 ? 1 : step - sS[k] + 1;
            const int sa = k % S.D;
            if (tid == 0) {
                if (na == 1) { hacc[sa][0] = hacc[sa][1] = hacc[sa][2] = hacc[sa][3] = 0.0; }
                hacc[sa][0] += o[0]; hacc[sa][1] = fmax(hacc[sa][1], o[1]);
                hacc[sa][2] += o[2]; hacc[sa][3] = fmax(hacc[sa][3], o[3]);
            }
            __syncthreads();
            if (S.mode == 0 && na == P.nt) {
                last_done = k;
                const double Ntot = (double)ns * (double)P.nt;
                const double dmax = S.stop_norm ? sqrt(hacc[sa][2] / Ntot) : hacc[sa][3];   // stop norm
                if (g == 0 && tid == 0) {
                    S.hist[4 * k + 0] = sqrt(hacc[sa][0] / Ntot);
                    S.hist[4 * k + 1] = hacc[sa][1];
                    S.hist[4 * k + 2] = sqrt(hacc[sa][2] / Ntot);
                    S.hist[4 * k + 3] = hacc[sa][3];
                }
                if (dmax <= S.newton_tol) { stop_status = 0; stop_k = k; }
                else if (k >= 1 && dmax > 0.5 * prevmax_s && dmax <= 1e3 * S.newton_tol) { stop_status = 1; stop_k = k; }
                else if (k + 1 >= newton_max) { stop_status = -4; stop_k = k; }
                __syncthreads();
                if (tid == 0) prevmax_s = dmax;
                __syncthreads();
            }
        }
        __syncthreads();
        if (g == 0 && tid == 0) total_inner += maxit_step;
        if (c == 0 && tid == 0 && S.stats && S.mode == 0) {          // per-pair iteration accounting
            atomicAdd((unsigned long long*)&S.stats[4], (unsigned long long)it);
            atomicAdd((unsigned long long*)&S.stats[8 + kme], (unsigned long long)it);
        }
        PMARK(6);
        if (S.mode == 1) {
            if (g == 0 && tid == 0) {
                S.info[0] = maxit_step;
                S.info[1] = err ? -5 : 0;
            }
            flush_prof();
            return;
        }
        if (err && stop_status == 2) { stop_status = -5; stop_k = last_done; }
        if (stop_status != 2) {
            const int kf = stop_k + 1;
            const double* Uf = S.U + (long long)(kf % S.B) * P.nt * ns;
            const long long N = ns * P.nt;
            if (S.u_out)
                for (long long q = (long long)g * BLOCK2 + tid; q < N; q += (long long)G * BLOCK2) S.u_out[q] = __ldcg(Uf + q);
            if (g == 0 && tid == 0) {
                S.info[0] = kf;
                S.info[1] = stop_status;
                if (S.stats) { S.stats[0] = step; S.stats[1] = total_inner; S.stats[2] = S.D; S.stats[3] = G; }
            }
            flush_prof();
            return;
        }
    }
}


}  // namespace pit
