// pit_kernels.cu — the hot path of libpit on sm_100a, fp64.
//
//   (a) k_resjac        : space-time residual of Eq. (5) + diagonal of every A_n (Eq. 6), all levels at
//                         once, fused norm reduction (HBM-streaming stencil kernel).
//   (b)+(c)+(d) k_newton: ONE persistent cooperative kernel per solve that runs the whole all-at-once
//                         Newton iteration on the device:
//        - the exact blockwise inverse of Eq. (7), applied as its row recursion
//              du^n = A_n^{-1} (r^n + du^{n-1})                    (Theorem 1's proof)
//          which keeps the level coupling on the device as a recurrence over levels (the literal
//          product form of Theorem 1 loses cond(A)^n digits);
//        - a Newton-iteration WAVEFRONT: U_{k+1}^n depends only on U_k^{<=n}, so level n of iteration k
//          and level n-1 of iteration k+1 run concurrently (pipeline depth D);
//        - every ready (level, iteration) pair is solved by Jacobi-scaled BiCGSTAB with 2 grid barriers
//          per iteration (neighbour values of p and s are recomputed redundantly from the state the
//          owning CTA wrote before the last barrier), deterministic fixed-order reductions;
//        - the per-level residual/Jacobian of kernel (a) is fused into each solve's prologue, the update
//          U_{k+1} = U_k + dU and the norms into its epilogue; the stop rule is evaluated on the device.
#include "pit_internal.cuh"

namespace pit {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier (all CTAs co-resident: cooperative launch).  Returns the OR of `flag` over CTAs.
__device__ __forceinline__ unsigned grid_sync(GridBar* b, unsigned nblocks, unsigned& gen, unsigned flag) {
    __shared__ unsigned s_flag;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (flag) atomicOr(&b->flag_acc, 1u);
        __threadfence();
        const unsigned arrived = atomicAdd(&b->count, 1u);
        if (arrived == nblocks - 1) {
            b->flag_out[(gen + 1) & 1] = atomicExch(&b->flag_acc, 0u);
            atomicExch(&b->count, 0u);
            __threadfence();
            atomicExch(&b->gen, gen + 1);
        } else {
            while (ld_acquire_u32(&b->gen) == gen) { }
        }
        __threadfence();
        s_flag = *((volatile unsigned*)&b->flag_out[(gen + 1) & 1]);
        gen += 1;
    }
    __syncthreads();
    return s_flag;
}

// Sum (NS entries) / max (NM entries) of the per-CTA partials of CTAs [g0, g1) in a fixed order.
// Called by all threads; result returned in every thread.
template <int NS, int NM>
__device__ __forceinline__ void pair_reduce(const double* part, int stride, int g0, int g1, double (&out)[NS + NM],
                                            double* sm) {
    constexpr int N = NS + NM;
    if (threadIdx.x < 32) {
        double a[N];
        #pragma unroll
        for (int i = 0; i < N; ++i) a[i] = 0.0;
        for (int g = g0 + (int)threadIdx.x; g < g1; g += 32) {
            const double* pg = part + (long long)g * stride;
            #pragma unroll
            for (int i = 0; i < N; ++i) {
                const double y = *((volatile const double*)(pg + i));
                a[i] = i < NS ? a[i] + y : fmax(a[i], y);
            }
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
            for (int i = 0; i < N; ++i) sm[i] = a[i];
    }
    __syncthreads();
    #pragma unroll
    for (int i = 0; i < N; ++i) out[i] = sm[i];
    __syncthreads();
}

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// ----------------------------------------------------------------------------------------------------
// (a) all-level residual + diagonal, fused partial norms.  One thread per unknown (grid-stride over
// the [nt][ns] space-time array); the stencil neighbours and u^{n-1} are L1/L2 hits.
// ----------------------------------------------------------------------------------------------------
// Residual and diagonal coefficient only (kernel a).  LAW 1 = Burgers with constant viscosity (m2 = 0):
// G = u_C - u_prev + tau[(u_E^2 - u_W^2)/(4h_x) + (u_N^2 - u_S^2)/(4h_y) - m0 (Laplacian)], a_C constant.
template <int LAW>
__device__ __forceinline__ void res_diag(const Prob& P, const Vals& v, double uprev, double& G, double& aC) {
    if (LAW == 1) {
        const double conv = 0.5 * ((v.e * v.e - v.w * v.w) * P.i2hx + (v.n * v.n - v.s * v.s) * P.i2hy);
        const double lap = (v.e + v.w - 2.0 * v.c) * P.ihx2 + (v.n + v.s - 2.0 * v.c) * P.ihy2;
        G = (v.c - uprev) + P.dt * (conv - P.m0 * lap);
        aC = 1.0 + 2.0 * P.dt * P.m0 * (P.ihx2 + P.ihy2);
        return;
    }
    const RJ o = residual_jacobian_raw(P, v, uprev);
    G = o.G;
    aC = o.aC;
}

template <int LAW>
__global__ void __launch_bounds__(BLOCK) k_resjac(Prob P, const double* __restrict__ U, const double* __restrict__ u0,
                                                  const double* __restrict__ ring, double* __restrict__ R,
                                                  double* __restrict__ diag, double* __restrict__ part) {
    constexpr int RB = 4;                      // rows per iteration: all their loads are issued before any use
    __shared__ double red[NWARP * 2];
    const int nxu = P.nxu, nyu = P.nyu;
    const int nxp = P.nx + 1;
    const int rows = P.nt * nyu;
    const int groups = (rows + RB - 1) / RB;
    double a[2] = {0.0, 0.0};
    for (int grp = blockIdx.x; grp < groups; grp += gridDim.x) {
        for (int i = threadIdx.x; i < nxu; i += BLOCK) {
            const bool he = P.bc == 1 || i + 1 < nxu, hw = P.bc == 1 || i > 0;
            const int ie = i + 1 < nxu ? i + 1 : 0, iw = i > 0 ? i - 1 : nxu - 1;
            Vals v[RB];
            double up[RB];
            long long q[RB];
            #pragma unroll
            for (int t = 0; t < RB; ++t) {
                const int row = min(grp * RB + t, rows - 1);
                const int n = row / nyu, j = row - n * nyu;             // level n (0-based), row j
                const double* Ul = U + (long long)n * P.ns;
                const double* Up = n == 0 ? u0 : Ul - P.ns;
                const double* ringn = ring ? ring + (long long)n * P.ring_len : nullptr;
                const long long rb = (long long)j * nxu;
                const bool hn = P.bc == 1 || j + 1 < nyu, hs = P.bc == 1 || j > 0;
                const long long rn = j + 1 < nyu ? rb + nxu : 0, rs = j > 0 ? rb - nxu : (long long)(nyu - 1) * nxu;
                v[t].c = __ldg(Ul + rb + i);
                v[t].e = he ? __ldg(Ul + rb + ie) : (ringn ? __ldg(ringn + 2 * nxp + (P.ny - 1) + j) : 0.0);
                v[t].w = hw ? __ldg(Ul + rb + iw) : (ringn ? __ldg(ringn + 2 * nxp + j) : 0.0);
                v[t].n = hn ? __ldg(Ul + rn + i) : (ringn ? __ldg(ringn + nxp + i + 1) : 0.0);
                v[t].s = hs ? __ldg(Ul + rs + i) : (ringn ? __ldg(ringn + i + 1) : 0.0);
                up[t] = __ldg(Up + rb + i);
                q[t] = (long long)n * P.ns + rb + i;
            }
            #pragma unroll
            for (int t = 0; t < RB; ++t) {
                if (grp * RB + t >= rows) continue;
                double G, aC;
                res_diag<LAW>(P, v[t], up[t], G, aC);
                const double r = -G;
                __stcs(R + q[t], r);                                   // streaming stores: R, diag not re-read here
                if (diag) __stcs(diag + q[t], aC);
                a[0] += r * r;
                a[1] = fmax(a[1], fabs(r));
            }
        }
    }
    block_reduce<1, 1>(a, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = a[0];
        part[2 * blockIdx.x + 1] = a[1];
    }
}

// (a) TMA-staged variant: persistent CTAs walk row tiles (level n, rows [j0, j0 + R)) in level-major order.
// One elected thread stages, per tile, the R + 2 rows of u^n (with the N/S halo rows, wrapped on periodic grids)
// and the R rows of u^{n-1} into shared memory with 1-D bulk copies (cp.async.bulk, completion on an mbarrier),
// S tiles ahead; all threads then evaluate the stencil from shared memory and stream R and diag(A_n) out.
// DRAM: u^n once (u^{n-1} rows were staged nyu / R tiles earlier and hit L2), R and diag written once:
// 24 B per DOF.  Needs nxu even (16-byte rows) and 16-byte aligned U / u0 (the host checks; else k_resjac).
constexpr int BLOCKA = 512;
constexpr int MAXSTAGE = 8;

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    unsigned done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(a), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}

// Warp-specialised: warp NWA (the last) is the producer (one lane issues the bulk copies of tile it + NS once
// the consumers released the stage on its `empty` mbarrier); warps 0..NWA-1 consume (stencil from shared
// memory, streaming stores) and release each stage with one arrive per warp.  No CTA-wide barrier per tile.
constexpr int NWA = BLOCKA / 32;                   // consumer warps

template <int LAW>
__global__ void __launch_bounds__(BLOCKA + 32, 1) k_resjac_bulk(Prob P, const double* __restrict__ U,
                                                               const double* __restrict__ u0, const double* __restrict__ ring,
                                                               double* __restrict__ R, double* __restrict__ diag,
                                                               double* __restrict__ part, int RT, int NS) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long full[MAXSTAGE], empty[MAXSTAGE];
    __shared__ double red[NWA * 2];
    const int nxu = P.nxu, nyu = P.nyu, tid = threadIdx.x, warp = tid >> 5;
    const bool per = P.bc == 1;
    const int tpl = (nyu + RT - 1) / RT;                       // tiles per level
    const long long ntiles = (long long)P.nt * tpl;
    const int stage = (2 * RT + 2) * nxu;                      // doubles per stage: u^n rows -1..RT, u^{n-1} rows 0..RT-1
    const unsigned rowb = (unsigned)nxu * 8u;
    const int nxp = P.nx + 1;
    const long long stride = gridDim.x;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWA); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NWA) {                                         // ---- producer ----
        if ((tid & 31) == 0) {
            int it = 0;
            for (long long t = blockIdx.x; t < ntiles; t += stride, ++it) {
                const int s = it % NS;
                if (it >= NS) mbar_wait(&empty[s], (unsigned)(it / NS - 1) & 1u);
                const int n = (int)(t / tpl), j0 = (int)(t % tpl) * RT;
                const int rows = min(RT, nyu - j0);
                double* cur = sm + (long long)s * stage;
                double* prv = cur + (RT + 2) * nxu;
                const double* Ul = U + (long long)n * P.ns;
                const double* Up = n == 0 ? u0 : Ul - P.ns;
                const bool hasS = per || j0 > 0, hasN = per || j0 + rows < nyu;
                const unsigned bytes = rowb * (unsigned)(2 * rows + (hasS ? 1 : 0) + (hasN ? 1 : 0));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&full[s], bytes);
                if (hasS) bulk_g2s(cur, Ul + (long long)(j0 == 0 ? nyu - 1 : j0 - 1) * nxu, rowb, &full[s]);
                bulk_g2s(cur + nxu, Ul + (long long)j0 * nxu, rowb * rows, &full[s]);
                if (hasN) bulk_g2s(cur + (rows + 1) * nxu, Ul + (long long)(j0 + rows == nyu ? 0 : j0 + rows) * nxu, rowb, &full[s]);
                bulk_g2s(prv, Up + (long long)j0 * nxu, rowb * rows, &full[s]);
            }
        }
        return;
    }
    double a[2] = {0.0, 0.0};                                  // ---- consumers ----
    int it = 0;
    for (long long t = blockIdx.x; t < ntiles; t += stride, ++it) {
        const int s = it % NS;
        mbar_wait(&full[s], (unsigned)(it / NS) & 1u);
        const int n = (int)(t / tpl), j0 = (int)(t % tpl) * RT;
        const int rows = min(RT, nyu - j0);
        const double* cur = sm + (long long)s * stage;
        const double* prv = cur + (RT + 2) * nxu;
        const double* ringn = ring ? ring + (long long)n * P.ring_len : nullptr;
        double* Rl = R + (long long)n * P.ns + (long long)j0 * nxu;
        double* Dl = diag ? diag + (long long)n * P.ns + (long long)j0 * nxu : nullptr;
        int r = tid / nxu, i = tid - r * nxu;
        const int di = BLOCKA % nxu, dr = BLOCKA / nxu;
        for (; r < rows;) {
            const int e = r * nxu + i, j = j0 + r;
            const double* row = cur + (r + 1) * nxu;
            Vals v;
            v.c = row[i];
            if (i + 1 < nxu) v.e = row[i + 1];
            else v.e = per ? row[0] : (ringn ? __ldg(ringn + 2 * nxp + (P.ny - 1) + j) : 0.0);
            if (i > 0) v.w = row[i - 1];
            else v.w = per ? row[nxu - 1] : (ringn ? __ldg(ringn + 2 * nxp + j) : 0.0);
            if (per || j + 1 < nyu) v.n = row[nxu + i];
            else v.n = ringn ? __ldg(ringn + nxp + i + 1) : 0.0;
            if (per || j > 0) v.s = row[i - nxu];
            else v.s = ringn ? __ldg(ringn + i + 1) : 0.0;
            double G, aC;
            res_diag<LAW>(P, v, prv[e], G, aC);
            const double rr = -G;
            __stcs(Rl + e, rr);
            if (Dl) __stcs(Dl + e, aC);
            a[0] += rr * rr;
            a[1] = fmax(a[1], fabs(rr));
            i += di; r += dr;
            if (i >= nxu) { i -= nxu; ++r; }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
    #pragma unroll
    for (int k = 0; k < 2; ++k)
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, a[k], o);
            a[k] = k == 0 ? a[k] + y : fmax(a[k], y);
        }
    if ((tid & 31) == 0) { red[warp * 2] = a[0]; red[warp * 2 + 1] = a[1]; }
    asm volatile("bar.sync 1, %0;" ::"r"(BLOCKA) : "memory");   // consumers only (the producer warp has left)
    if (tid == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < NWA; ++w) { s0 += red[2 * w]; s1 = fmax(s1, red[2 * w + 1]); }
        part[2 * blockIdx.x] = s0;
        part[2 * blockIdx.x + 1] = s1;
    }
}

__global__ void k_finish_norms(const double* __restrict__ part, int nparts, long long N, double* __restrict__ norms) {
    __shared__ double red[NWARP * 2];
    double a[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += BLOCK) { a[0] += part[2 * i]; a[1] = fmax(a[1], part[2 * i + 1]); }
    block_reduce<1, 1>(a, red);
    if (threadIdx.x == 0) { norms[0] = sqrt(a[0] / (double)N); norms[1] = a[1]; }
}


// ----------------------------------------------------------------------------------------------------
// (b2) building blocks of the literal Theorem 1 product form inside a Section 7 window.
// ----------------------------------------------------------------------------------------------------
struct MatvecJobs {
    int n;
    int lev[MAXD];                // A_lev (1-based level), taken at the iterate U
    const double* x[MAXD];
    double* y[MAXD];              // y = A_lev x   (may not alias x)
};

// y_j = A_{lev_j} x_j for a batch of vectors: the true (unscaled) diagonal block of Eq. (6) at U.
__global__ void __launch_bounds__(BLOCK) k_matvec_batch(Prob P, const double* __restrict__ U, const double* __restrict__ ring,
                                                        MatvecJobs J) {
    const int j = blockIdx.y;
    const int n = J.lev[j];
    const double* Ul = U + (long long)(n - 1) * P.ns;
    const double* ringn = ring ? ring + (long long)(n - 1) * P.ring_len : nullptr;
    const double* x = J.x[j];
    double* y = J.y[j];
    for (long long p = (long long)blockIdx.x * BLOCK + threadIdx.x; p < P.ns; p += (long long)gridDim.x * BLOCK) {
        const Nbr nb = neighbours(P, p);
        const Vals v = stencil_values(P, Ul, ringn, p, nb);
        const RJ o = residual_jacobian(P, v, nb, 0.0);
        y[p] = o.aC * x[p] + o.aE * x[nb.e] + o.aW * x[nb.w] + o.aN * x[nb.n] + o.aS * x[nb.s];
    }
}

// r~^m = sum_{j <= m} y^j over the window's levels, in place (the level scan of the RHS recursion,
// r~^{n+1} = P^n r^{n+1} + r~^n).
__global__ void k_level_prefix(long long ns, int L, double* __restrict__ Y) {
    for (long long p = (long long)blockIdx.x * BLOCK + threadIdx.x; p < ns; p += (long long)gridDim.x * BLOCK) {
        double acc = 0.0;
        for (int m = 0; m < L; ++m) {
            acc += Y[(long long)m * ns + p];
            Y[(long long)m * ns + p] = acc;
        }
    }
}

// ||A_n||_inf (max absolute row sum) of levels n0..n0+L-1 at U: the Section 7 gate (R13 of
// SURVEY: Gershgorin bound on the forward chain prod ||A_i||).  part[L][gridDim.x] partial maxima.
__global__ void __launch_bounds__(BLOCK) k_anorm(Prob P, const double* __restrict__ U, const double* __restrict__ ring,
                                                 int n0, double* __restrict__ part) {
    __shared__ double red[NWARP * 1];
    const int n = n0 + blockIdx.y;
    const double* Ul = U + (long long)(n - 1) * P.ns;
    const double* ringn = ring ? ring + (long long)(n - 1) * P.ring_len : nullptr;
    double a[1] = {0.0};
    for (long long p = (long long)blockIdx.x * BLOCK + threadIdx.x; p < P.ns; p += (long long)gridDim.x * BLOCK) {
        const Nbr nb = neighbours(P, p);
        const Vals v = stencil_values(P, Ul, ringn, p, nb);
        const RJ o = residual_jacobian(P, v, nb, 0.0);
        a[0] = fmax(a[0], fabs(o.aC) + fabs(o.aE) + fabs(o.aW) + fabs(o.aN) + fabs(o.aS));
    }
    block_reduce<0, 1>(a, red);
    if (threadIdx.x == 0) part[(long long)blockIdx.y * gridDim.x + blockIdx.x] = a[0];
}

// U += dU over all levels, fused norm partials of dU (sum dU^2, max |dU|, nonfinite flag).
__global__ void __launch_bounds__(BLOCK) k_update(long long N, double* __restrict__ U, const double* __restrict__ dU,
                                                  double* __restrict__ part) {
    __shared__ double red[NWARP * 3];
    double a[3] = {0.0, 0.0, 0.0};
    for (long long q = (long long)blockIdx.x * BLOCK + threadIdx.x; q < N; q += (long long)gridDim.x * BLOCK) {
        const double d = dU[q];
        U[q] += d;
        a[0] += d * d;
        a[1] = fmax(a[1], fabs(d));
        if (!isfinite(d)) a[2] = 1.0;
    }
    block_reduce<1, 2>(a, red);
    if (threadIdx.x == 0) { part[3 * blockIdx.x] = a[0]; part[3 * blockIdx.x + 1] = a[1]; part[3 * blockIdx.x + 2] = a[2]; }
}

// U_0: the caller's guess, or u^0 at every level.
__global__ void k_init_iterate(long long ns, int nt, const double* u0, const double* guess,
                               double* U) {
    const long long N = ns * nt;
    for (long long q = (long long)blockIdx.x * BLOCK + threadIdx.x; q < N; q += (long long)gridDim.x * BLOCK)
        U[q] = guess ? guess[q] : u0[q % ns];
}

// ----------------------------------------------------------------------------------------------------
// The persistent Newton kernel.
// ----------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK) k_newton(SolveParams S) {
    const Prob P = S.P;
    const long long ns = P.ns;
    const int G = S.G, g = blockIdx.x;
    __shared__ int sS[MAXK];                   // start step of iteration k
    __shared__ double red[NWARP * NPART];
    __shared__ double pr[NPART];
    __shared__ double hacc[MAXD][4];           // per-slot norm accumulators of the in-flight iterations
    __shared__ double prevmax_s;
    unsigned gen = 0;
    if (threadIdx.x == 0) {
        gen = ld_acquire_u32(&S.bar->gen);
        const int D = S.D;
        for (int k = 0; k < S.newton_max; ++k) {
            int st = k == 0 ? 1 : sS[k - 1] + 1;
            if (k >= D && sS[k - D] + P.nt > st) st = sS[k - D] + P.nt;
            sS[k] = st;
        }
        prevmax_s = INFINITY;
    }
    if (threadIdx.x < MAXD * 4) hacc[threadIdx.x / 4][threadIdx.x % 4] = 0.0;
    __syncthreads();

    const int newton_max = S.mode == 0 ? S.newton_max : 1;
    int set = 0;                               // partial-array parity, flips after every barrier
    int klo = 0;
    int last_done = -1;                        // last completed Newton iteration
    long long total_inner = 0;
    const double rtol2 = S.lin_rtol * S.lin_rtol;
    const double atol2 = S.lin_atol * S.lin_atol * (double)P.ns;     // lin_atol bounds the RMS residual

    for (int step = 1;; ++step) {
        // ---- active (level, iteration) pairs of this wavefront step, iteration ascending ----
        while (klo < newton_max && step > sS[klo] + P.nt - 1) ++klo;
        int ks[MAXD];
        int A = 0;
        for (int k = klo; k < newton_max && A < MAXD && sS[k] <= step; ++k) ks[A++] = k;
        if (S.mode == 1) { A = S.nb; for (int a = 0; a < A; ++a) ks[a] = a; }
        // my pair = the one whose contiguous CTA block [a G / A, (a+1) G / A) contains g
        int me = 0;
        while (me + 1 < A && (long long)(me + 1) * G / A <= g) ++me;
        const int g0 = (int)((long long)me * G / A), g1 = (int)((long long)(me + 1) * G / A);
        const int kme = ks[me];
        const int n = S.mode == 1 ? S.blev[me] : step - sS[kme] + 1;       // 1-based level
        const int slot = kme % S.D;
        const int buf = kme % S.B, nbuf = (kme + 1) % S.B;
        const Slot sl = slot_at(S.slotmem, ns, slot);
        const long long c = g - g0, C = g1 - g0;
        const long long p0 = c * ns / C, p1 = (c + 1) * ns / C;
        const double* Ulev = S.mode == 1 ? S.U + (long long)(n - 1) * ns : S.U + ((long long)buf * P.nt + (n - 1)) * ns;
        const double* uprev = n == 1 ? S.u0 : Ulev - ns;
        const double* ringn = S.ring ? S.ring + (long long)(n - 1) * P.ring_len : nullptr;
        double* partS = S.part + (long long)set * G * NPART;
        double* hp = S.hpart + (long long)(step & 1) * G * 4;

        // ---- prologue: fused residual + Jacobian of level n (kernel a), carry, Jacobi scaling ----
        {
            double a[3] = {0.0, 0.0, 0.0};   // sum bt^2, sum r^2 | max |r|
            for (long long p = p0 + threadIdx.x; p < p1; p += BLOCK) {
                const Nbr nb = neighbours(P, p);
                const Vals v = stencil_values(P, Ulev, ringn, p, nb);
                const RJ o = residual_jacobian(P, v, nb, S.mode == 1 ? 0.0 : uprev[p]);
                double rhs;
                if (S.mode == 1) {
                    rhs = S.bptr[me][p];
                } else {
                    const double r = -o.G;                               // Newton rhs of Eq. (5)
                    a[1] += r * r;
                    a[2] = fmax(a[2], fabs(r));
                    rhs = r + (n == 1 ? 0.0 : sl.x[p]);                  // r^n + du^{n-1}  (Eq. 7 row n)
                }
                const double inv = 1.0 / o.aC;
                const double bt = rhs * inv;
                sl.cE[p] = o.aE * inv; sl.cW[p] = o.aW * inv; sl.cN[p] = o.aN * inv; sl.cS[p] = o.aS * inv;
                sl.bt[p] = bt;
                sl.r[p] = bt;
                sl.x[p] = 0.0;
                a[0] += bt * bt;
            }
            block_reduce<2, 1>(a, red);
            if (threadIdx.x == 0) {
                partS[(long long)g * NPART + 0] = a[0];
                hp[g * 4 + 0] = a[1];
                hp[g * 4 + 1] = a[2];
            }
        }
        grid_sync(S.bar, G, gen, 0);
        double bnorm2, rho, alpha = 0.0, omega = 1.0, beta = 0.0;
        {
            double o[1];
            pair_reduce<1, 0>(S.part + (long long)set * G * NPART, NPART, g0, g1, o, pr);
            bnorm2 = o[0];
        }
        set ^= 1;
        rho = bnorm2;
        bool conv = bnorm2 <= atol2;            // zero (or negligible) right-hand side
        bool pending = false;                   // x misses the last iteration's alpha p + omega s update
        int it = 0;
        int maxit_step = 0;

        // ---- BiCGSTAB iterations (2 grid barriers each) ----
        for (;;) {
            const int par = it & 1;
            if (!conv) {
                double a[1] = {0.0};
                const double* pold = sl.p[par ^ 1];
                const double* vold = sl.v[par ^ 1];
                double* pnew = sl.p[par];
                double* vnew = sl.v[par];
                for (long long p = p0 + threadIdx.x; p < p1; p += BLOCK) {
                    const Nbr nb = neighbours(P, p);
                    double pc, pe, pw, pn, ps;
                    if (it == 0) {
                        pc = sl.bt[p];
                        pe = sl.bt[nb.e]; pw = sl.bt[nb.w]; pn = sl.bt[nb.n]; ps = sl.bt[nb.s];
                    } else {
                        const double sc = sl.s[p], tc = sl.t[p];
                        const double rn = sc - omega * tc;
                        if (pending) sl.x[p] += alpha * pold[p] + omega * sc;
                        sl.r[p] = rn;
                        pc = rn + beta * (pold[p] - omega * vold[p]);
                        auto pq = [&](long long q) {
                            return (sl.s[q] - omega * sl.t[q]) + beta * (pold[q] - omega * vold[q]);
                        };
                        pe = pq(nb.e); pw = pq(nb.w); pn = pq(nb.n); ps = pq(nb.s);
                    }
                    const double vv = pc + sl.cE[p] * pe + sl.cW[p] * pw + sl.cN[p] * pn + sl.cS[p] * ps;
                    pnew[p] = pc;
                    vnew[p] = vv;
                    a[0] += sl.bt[p] * vv;
                }
                block_reduce<1, 0>(a, red);
                if (threadIdx.x == 0) S.part[((long long)set * G + g) * NPART + 0] = a[0];
                pending = false;
            }
            const unsigned any = grid_sync(S.bar, G, gen, conv ? 0u : 1u);
            if (!any) { set ^= 1; break; }     // every pair had converged before this phase
            double r0v = 0.0;
            if (!conv) {
                double o[1];
                pair_reduce<1, 0>(S.part + (long long)set * G * NPART, NPART, g0, g1, o, pr);
                r0v = o[0];
            }
            set ^= 1;
            if (!conv) {
                if (r0v == 0.0 || !finite(r0v)) {
                    if (threadIdx.x == 0 && c == 0) atomicOr(&S.bar->err, 2u);
                    conv = true;
                } else {
                    alpha = rho / r0v;
                }
            }
            if (!conv) {
                double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};   // (t,s) (t,t) (r0,s) (r0,t) (s,s)
                const double* vv = sl.v[par];
                for (long long p = p0 + threadIdx.x; p < p1; p += BLOCK) {
                    const Nbr nb = neighbours(P, p);
                    const double sc = sl.r[p] - alpha * vv[p];
                    auto sq = [&](long long q) { return sl.r[q] - alpha * vv[q]; };
                    const double tc = sc + sl.cE[p] * sq(nb.e) + sl.cW[p] * sq(nb.w) + sl.cN[p] * sq(nb.n) +
                                      sl.cS[p] * sq(nb.s);
                    sl.s[p] = sc;
                    sl.t[p] = tc;
                    const double b0 = sl.bt[p];
                    a[0] += tc * sc; a[1] += tc * tc; a[2] += b0 * sc; a[3] += b0 * tc; a[4] += sc * sc;
                }
                block_reduce<5, 0>(a, red);
                if (threadIdx.x == 0) {
                    double* pp = S.part + ((long long)set * G + g) * NPART;
                    for (int i = 0; i < 5; ++i) pp[i] = a[i];
                }
            }
            grid_sync(S.bar, G, gen, 0);
            if (!conv) {
                double o[5];
                pair_reduce<5, 0>(S.part + (long long)set * G * NPART, NPART, g0, g1, o, pr);
                const double ts = o[0], tt = o[1], r0s = o[2], r0t = o[3], ss = o[4];
                ++it;
                pending = true;
                if (tt == 0.0) {                          // t = A s = 0  =>  s = 0: exact solution
                    omega = 0.0;
                    conv = true;
                } else {
                    omega = ts / tt;
                    const double rhon = r0s - omega * r0t;
                    const double rn2 = fmax(ss - 2.0 * omega * ts + omega * omega * tt, 0.0);
                    if (!finite(omega) || !finite(rn2)) {
                        if (threadIdx.x == 0 && c == 0) atomicOr(&S.bar->err, 1u);
                        conv = true;
                    } else if (rn2 <= rtol2 * bnorm2 || rn2 <= atol2 || it >= S.lin_max) {
                        conv = true;
                    } else if (omega == 0.0 || rhon == 0.0) {
                        if (threadIdx.x == 0 && c == 0) atomicOr(&S.bar->err, 2u);
                        conv = true;
                    } else {
                        beta = (rhon / rho) * (alpha / omega);
                        rho = rhon;
                    }
                }
            }
            set ^= 1;
            maxit_step = it > maxit_step ? it : maxit_step;
        }

        // ---- epilogue: final x update, U_{k+1}^n = U_k^n + du^n, carry, norms ----
        {
            double a[3] = {0.0, 0.0, 0.0};   // sum du^2, max |du|, nonfinite
            const int lp = (it - 1) & 1;
            double* Unew = S.mode == 1 ? nullptr : S.U + ((long long)nbuf * P.nt + (n - 1)) * ns;
            for (long long p = p0 + threadIdx.x; p < p1; p += BLOCK) {
                double dx = sl.x[p];
                if (pending) dx += alpha * sl.p[lp][p] + omega * sl.s[p];
                sl.x[p] = dx;                        // du^n: the carry of level n+1 (same slot)
                if (S.mode == 1) {
                    S.xptr[me][p] = dx;
                } else {
                    Unew[p] = Ulev[p] + dx;
                }
                a[0] += dx * dx;
                a[1] = fmax(a[1], fabs(dx));
                if (!finite(dx)) a[2] = 1.0;
            }
            block_reduce<1, 2>(a, red);
            if (threadIdx.x == 0) {
                hp[g * 4 + 2] = a[0];
                hp[g * 4 + 3] = a[1];
                if (a[2] != 0.0) atomicOr(&S.bar->err, 1u);
            }
        }
        // the step's inner iteration count is the max over its pairs (all pairs share the barriers)
        grid_sync(S.bar, G, gen, 0);
        // ---- norms of the finished levels -> per-iteration accumulators; stop rule ----
        const unsigned err = *((volatile unsigned*)&S.bar->err);
        int stop_status = 2;     // 2 = continue
        int stop_k = -1;
        for (int a = 0; a < A; ++a) {
            const int ga0 = (int)((long long)a * G / A), ga1 = (int)((long long)(a + 1) * G / A);
            double oa[2], ob[2];
            pair_reduce<1, 1>(hp, 4, ga0, ga1, oa, pr);
            pair_reduce<1, 1>(hp + 2, 4, ga0, ga1, ob, pr);
            const double o[4] = {oa[0], oa[1], ob[0], ob[1]};
            const int k = ks[a];
            const int na = S.mode == 1 ? 1 : step - sS[k] + 1;
            const int sa = k % S.D;
            if (threadIdx.x == 0) {
                if (na == 1) { hacc[sa][0] = hacc[sa][1] = hacc[sa][2] = hacc[sa][3] = 0.0; }
                hacc[sa][0] += o[0]; hacc[sa][1] = fmax(hacc[sa][1], o[1]);
                hacc[sa][2] += o[2]; hacc[sa][3] = fmax(hacc[sa][3], o[3]);
            }
            __syncthreads();
            if (S.mode == 0 && na == P.nt) {          // iteration k complete: record and test
                last_done = k;
                const double Ntot = (double)ns * (double)P.nt;
                const double dmax = S.stop_norm ? sqrt(hacc[sa][2] / Ntot) : hacc[sa][3];   // stop norm
                if (g == 0 && threadIdx.x == 0) {
                    S.hist[4 * k + 0] = sqrt(hacc[sa][0] / Ntot);
                    S.hist[4 * k + 1] = hacc[sa][1];
                    S.hist[4 * k + 2] = sqrt(hacc[sa][2] / Ntot);
                    S.hist[4 * k + 3] = hacc[sa][3];
                }
                if (dmax <= S.newton_tol) { stop_status = 0; stop_k = k; }
                else if (k >= 1 && dmax > 0.5 * prevmax_s && dmax <= 1e3 * S.newton_tol) { stop_status = 1; stop_k = k; }
                else if (k + 1 >= newton_max) { stop_status = -4; stop_k = k; }
                __syncthreads();
                if (threadIdx.x == 0) prevmax_s = dmax;
                __syncthreads();
            }
        }
        if (g == 0 && threadIdx.x == 0) total_inner += maxit_step;
        if (S.mode == 1) {
            if (g == 0 && threadIdx.x == 0) {
                S.info[0] = maxit_step;
                S.info[1] = err ? -5 : 0;
            }
            return;
        }
        if (err && stop_status == 2) {            // NaN/Inf or breakdown: stop with the last complete iterate
            stop_status = -5;
            stop_k = last_done;                    // last completed iteration (-1: U_0)
        }
        if (stop_status != 2) {
            const int kf = stop_k + 1;              // the returned iterate U_{k+1}
            const double* Uf = S.U + (long long)(kf % S.B) * P.nt * ns;
            const long long N = ns * P.nt;
            if (S.u_out)
                for (long long q = (long long)g * BLOCK + threadIdx.x; q < N; q += (long long)G * BLOCK)
                    S.u_out[q] = Uf[q];
            if (g == 0 && threadIdx.x == 0) {
                S.info[0] = kf;
                S.info[1] = stop_status;
                if (S.stats) {
                    S.stats[0] = step;
                    S.stats[1] = total_inner;
                    S.stats[2] = S.D;
                    S.stats[3] = G;
                }
            }
            return;
        }
    }
}

}  // namespace pit

#include "pit_newton_onchip.cuh"
#include "pit_newton_col.cuh"
