// pit_guess.cuh — the paper's all-at-once initial guess, on the device.
//
// "we initialize the solution by solving Eq. (FDS) sequentially on a coarse grid and interpolating this
// coarse-grid-solution to the original fine mesh by using a 1-D cubic spline along each spatial coordinate.
// ... the original grid is coarsened in both each spatial direction and time by the same factor c_f."
//
// Device pipeline (pit_api.cu drives it, one stream, no host round trip):
//   k_restrict_u0 / k_restrict_ring  inject u^0 and the Dirichlet ring at the coarse nodes (fine node c_f i,
//                                    fine level c_f m)
//   coarse solve                     the same all-at-once engine on the coarse problem (its converged solution
//                                    is the sequential BDF1 solution, Theorem 1 / PAPER.md:204-207)
//   k_spline<0>  along x             every coarse level m >= 1 and coarse node row -> fine unknown columns
//   k_spline<1>  along y             every coarse level and fine column           -> fine unknown rows
//   k_spline<2>  along t             every fine unknown: knots u^0 (t = 0) and the m >= 1 levels -> levels 1..nt
// Splines (R22): C^2 cubic on uniform knots, periodic along periodic directions, not-a-knot otherwise
// and in time.  With m_k = M_k H^2 / 6 the continuity equations read m_{k-1} + 4 m_k + m_{k+1} = F_{k+1} - 2 F_k
// + F_{k-1}; a thread owns one line (Thomas algorithm, Sherman-Morrison for the cyclic system), the
// line-independent factors come from k_spline_setup.
#pragma once

namespace pit {

struct GuessParams {
    int cf, bc;
    int nx, ny, nt, nxu, nyu;
    long long ns;
    int nxc, nyc, ntc, nxuc, nyuc, ring_len_c;
    long long nsc;
    const double* u0f;       // fine u^0 [ns]
    const double* cU;        // coarse solution [ntc][nsc]
    const double* cring;     // coarse rings [ntc][ring_len_c] or nullptr (Dirichlet homogeneous / periodic)
    double* Tx;              // [ntc][NR][nxu]
    double* Ty;              // [ntc][ns]
    double* tmp;             // [K][lines] moments of the current pass
    const double* fac;       // [2][K] from k_spline_setup: Thomas inverse pivots, cyclic correction z
    double* U0;              // [nt][ns] the fine initial iterate
};

__global__ void k_restrict_u0(GuessParams g, double* u0c) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.nsc; q += (long long)gridDim.x * blockDim.x) {
        const int icu = (int)(q % g.nxuc), jcu = (int)(q / g.nxuc);
        long long f;
        if (g.bc == 1) f = (long long)(g.cf * jcu) * g.nxu + g.cf * icu;
        else f = (long long)(g.cf * (jcu + 1) - 1) * g.nxu + (g.cf * (icu + 1) - 1);
        u0c[q] = g.u0f[f];
    }
}

// coarse ring of level m = fine ring of level c_f m at the nodes c_f i (ABI ring order, include/pit.h)
__global__ void k_restrict_ring(GuessParams g, const double* __restrict__ ringf, double* ringc) {
    const long long total = (long long)g.ntc * g.ring_len_c;
    const int rlf = 2 * (g.nx + g.ny);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int m = (int)(t / g.ring_len_c) + 1, e = (int)(t % g.ring_len_c);
        const double* rf = ringf + (long long)(g.cf * m - 1) * rlf;
        const int nb = g.nxc + 1;
        int f;
        if (e < nb) f = g.cf * e;                                                    // bottom, ic = e
        else if (e < 2 * nb) f = (g.nx + 1) + g.cf * (e - nb);                      // top
        else if (e < 2 * nb + g.nyc - 1) f = 2 * (g.nx + 1) + g.cf * (e - 2 * nb + 1) - 1;           // left, jc >= 1
        else f = 2 * (g.nx + 1) + (g.ny - 1) + g.cf * (e - 2 * nb - (g.nyc - 1) + 1) - 1;            // right
        ringc[t] = rf[f];
    }
}

// Line-independent factors of the spline system with K knots: fac[0..K) inverse Thomas pivots, fac[K..2K) the
// cyclic correction z (periodic only).  Not-a-knot: the K-4 interior unknowns m_2..m_{K-3} have pivots
// 4 - 1/w; periodic: T = tridiag(1, b', 1) with b'_0 = 4 - gamma = 8, b'_{K-1} = 4 - 1/gamma = 4.25 (gamma = -4)
// and T z = (gamma, 0, .., 0, 1) (Sherman-Morrison).
__global__ void k_spline_setup(int K, int periodic, double* fac) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    if (periodic) {
        double w = 0.0;
        for (int k = 0; k < K; ++k) {
            const double b = k == 0 ? 8.0 : (k == K - 1 ? 4.25 : 4.0);
            w = 1.0 / (b - (k == 0 ? 0.0 : w));
            fac[k] = w;
        }
        double d = 0.0;
        for (int k = 0; k < K; ++k) {
            const double u = k == 0 ? -4.0 : (k == K - 1 ? 1.0 : 0.0);
            d = (u - (k == 0 ? 0.0 : d)) * fac[k];
            fac[K + k] = d;
        }
        for (int k = K - 2; k >= 0; --k) fac[K + k] -= fac[k] * fac[K + k + 1];
    } else {
        double w = 0.0;
        for (int k = 0; k < K - 4; ++k) {
            w = 1.0 / (4.0 - (k == 0 ? 0.0 : w));
            fac[k] = w;
        }
    }
}

// Moments m_k (stored at tmp[k * ls]) of the spline through F(k), k = 0..K-1.
// Periodic: stores y (T y = r); the caller adds the cyclic correction -fct z_k when evaluating.
template <class F>
__device__ __forceinline__ double spline_moments_line(int K, bool periodic, F fetch, double* tmp, long long ls,
                                                      const double* __restrict__ fac) {
    if (periodic) {
        double fm = fetch(K - 1), f0 = fetch(0), d = 0.0;
        for (int k = 0; k < K; ++k) {
            const double fp = fetch(k + 1 < K ? k + 1 : 0);
            const double r = fp - 2.0 * f0 + fm;
            d = (r - (k == 0 ? 0.0 : d)) * fac[k];
            tmp[k * ls] = d;
            fm = f0; f0 = fp;
        }
        double y = d, y_last = d;
        for (int k = K - 2; k >= 0; --k) {
            y = tmp[k * ls] - fac[k] * y;
            tmp[k * ls] = y;
        }
        const double* z = fac + K;
        return (y - 0.25 * y_last) / (1.0 + z[0] - 0.25 * z[K - 1]);      // Sherman-Morrison factor
    }
    if (K <= 2) {
        for (int k = 0; k < K; ++k) tmp[k * ls] = 0.0;
        return 0.0;
    }
    auto r_at = [&](int k) { return fetch(k + 1) - 2.0 * fetch(k) + fetch(k - 1); };
    if (K == 3) {
        const double m = r_at(1) / 6.0;
        tmp[0] = m; tmp[ls] = m; tmp[2 * ls] = m;
        return 0.0;
    }
    const double m1 = r_at(1) / 6.0, mK2 = r_at(K - 2) / 6.0;       // rows 0/1 and K-2/K-1 combined
    tmp[1 * ls] = m1;
    tmp[(K - 2) * ls] = mK2;
    const int n = K - 4;                                             // interior unknowns m_2 .. m_{K-3}
    if (n > 0) {
        double fm = fetch(1), f0 = fetch(2), d = 0.0;
        for (int i = 0; i < n; ++i) {
            const int k = i + 2;
            const double fp = fetch(k + 1);
            double r = fp - 2.0 * f0 + fm;
            if (i == 0) r -= m1;
            if (i == n - 1) r -= mK2;
            d = (r - (i == 0 ? 0.0 : d)) * fac[i];
            tmp[k * ls] = d;
            fm = f0; f0 = fp;
        }
        double x = d;
        for (int i = n - 2; i >= 0; --i) {
            x = tmp[(i + 2) * ls] - fac[i] * x;
            tmp[(i + 2) * ls] = x;
        }
    }
    tmp[0] = 2.0 * m1 - tmp[2 * ls];
    tmp[(K - 1) * ls] = 2.0 * mK2 - tmp[(K - 3) * ls];
    return 0.0;
}

// S(p) at fine position p (knot k at p = cf k): (1-th) F_k + th F_{k+1} + ((1-th)^3 - (1-th)) m_k + (th^3 - th) m_{k+1}
template <class F>
__device__ __forceinline__ double spline_eval_at(int p, int cf, int K, bool periodic, F fetch, const double* tmp,
                                                 long long ls, double fct, const double* __restrict__ z) {
    const int k = p / cf, r = p - k * cf;
    const int kk = periodic && k >= K ? k - K : k;
    if (r == 0) return fetch(kk);
    const int k1 = periodic && kk + 1 >= K ? 0 : kk + 1;
    const double th = (double)r / (double)cf, a = 1.0 - th;
    double m0 = tmp[kk * ls], m1 = tmp[k1 * ls];
    if (periodic) { m0 -= fct * z[kk]; m1 -= fct * z[k1]; }
    return a * fetch(kk) + th * fetch(k1) + (a * a * a - a) * m0 + (th * th * th - th) * m1;
}

// PASS 0: x, lines (m, coarse node row jc), knots = coarse node columns; PASS 1: y, lines (m, fine unknown column),
// knots = coarse node rows; PASS 2: t, lines = fine unknowns, knots = levels 0 (u^0) .. ntc.
template <int PASS>
__global__ void __launch_bounds__(256) k_spline(GuessParams g) {
    const bool per = PASS < 2 && g.bc == 1;
    const int NR = g.bc == 1 ? g.nyc : g.nyc + 1;                 // coarse node rows
    const int NC = g.bc == 1 ? g.nxc : g.nxc + 1;                 // coarse node columns
    const int i0 = g.bc == 1 ? 0 : 1;                             // fine node of the first unknown
    const long long lines = PASS == 0 ? (long long)g.ntc * NR : (PASS == 1 ? (long long)g.ntc * g.nxu : g.ns);
    const int K = PASS == 0 ? NC : (PASS == 1 ? NR : g.ntc + 1);
    const double* z = g.fac + K;
    for (long long L = blockIdx.x * (long long)blockDim.x + threadIdx.x; L < lines; L += (long long)gridDim.x * blockDim.x) {
        double* tmp = g.tmp + L;
        if (PASS == 0) {
            const int m = (int)(L / NR) + 1, jc = (int)(L % NR);
            const double* cu = g.cU + (long long)(m - 1) * g.nsc;
            const double* ring = g.cring ? g.cring + (long long)(m - 1) * g.ring_len_c : nullptr;
            auto fetch = [&](int ic) -> double {
                if (g.bc == 1) return cu[(long long)jc * g.nxc + ic];
                if (jc > 0 && jc < g.nyc && ic > 0 && ic < g.nxc) return cu[(long long)(jc - 1) * g.nxuc + (ic - 1)];
                if (!ring) return 0.0;
                const int nb = g.nxc + 1;
                if (jc == 0) return ring[ic];
                if (jc == g.nyc) return ring[nb + ic];
                if (ic == 0) return ring[2 * nb + jc - 1];
                return ring[2 * nb + (g.nyc - 1) + jc - 1];
            };
            const double fct = spline_moments_line(K, per, fetch, tmp, lines, g.fac);
            double* out = g.Tx + L * g.nxu;
            for (int iu = 0; iu < g.nxu; ++iu) out[iu] = spline_eval_at(iu + i0, g.cf, K, per, fetch, tmp, lines, fct, z);
        } else if (PASS == 1) {
            const int m = (int)(L / g.nxu) + 1, iu = (int)(L % g.nxu);
            const double* tx = g.Tx + (long long)(m - 1) * NR * g.nxu + iu;
            auto fetch = [&](int jc) -> double { return tx[(long long)jc * g.nxu]; };
            const double fct = spline_moments_line(K, per, fetch, tmp, lines, g.fac);
            double* out = g.Ty + (long long)(m - 1) * g.ns + iu;
            for (int ju = 0; ju < g.nyu; ++ju)
                out[(long long)ju * g.nxu] = spline_eval_at(ju + i0, g.cf, K, per, fetch, tmp, lines, fct, z);
        } else {
            const long long q = L;
            auto fetch = [&](int m) -> double { return m == 0 ? g.u0f[q] : g.Ty[(long long)(m - 1) * g.ns + q]; };
            spline_moments_line(K, false, fetch, tmp, lines, g.fac);
            for (int n = 1; n <= g.nt; ++n)
                __stcs(g.U0 + (long long)(n - 1) * g.ns + q, spline_eval_at(n, g.cf, K, false, fetch, tmp, lines, 0.0, z));
        }
    }
}

}  // namespace pit
