// pit_explicit.cuh — N3: the paper's OWN explicit variant of the decoupled form, on the device.
//
// Theorem 1 / Eq. (8) with the left- and right-hand sides built by the recursions of §5
// (Eq. (10) entrywise):   P^1 = A_1,  P^{m+1} = P^m A_{m+1},  r~^{m+1} = P^m r^{m+1} + r~^m,
// the §7 diagonal preconditioner diag(P^m) applied on the left (DESIGN R11), and every decoupled
// system P^m du^m = r~^m solved by a banded LU WITHOUT pivoting.  Dirichlet grids only: the
// periodic wrap puts entries in the corners of A_n, so P^m is not banded.
//
// Storage: P^m in band form, row i holds offsets d = j - i in [-w, w] at column c = d + w (pitch 2w + 1), all
// window levels side by side ([L][ns][2w+1]); w = min(L nxu, ns - 1) (P^m has half-bandwidth m nxu, Theorem 2
// PAPER.md:269-278, Remark 4 PAPER.md:285).  The products and the right-hand sides are fully parallel over
// entries; the factorisation and the substitutions are sequential in the pivot index k (one CTA per level,
// levels batched over CTAs), as a direct band solver is.  This is the fidelity path that demonstrates the §7
// limit (its cost is O(ns w^2) per level), not the fast path.
#pragma once

namespace pit {

constexpr int BLOCKX = 1024;     // threads of the per-level factorisation / substitution CTAs

__device__ __forceinline__ long long llmin(long long a, long long b) { return a < b ? a : b; }
__device__ __forceinline__ long long llmax(long long a, long long b) { return a > b ? a : b; }

// The five coefficients (C, E, W, N, S) of A_n (Eq. 6) at U for levels n0..n0+L-1, Dirichlet
// columns dropped (they belong to q, Eq. 4): C5[m][5][ns].
__global__ void __launch_bounds__(BLOCK) k_coef5(Prob P, const double* __restrict__ U, const double* __restrict__ ring,
                                                 int n0, double* __restrict__ C5) {
    const int m = blockIdx.y, n = n0 + m;
    const double* Ul = U + (long long)(n - 1) * P.ns;
    const double* ringn = ring ? ring + (long long)(n - 1) * P.ring_len : nullptr;
    double* c = C5 + (long long)m * 5 * P.ns;
    for (long long p = (long long)blockIdx.x * BLOCK + threadIdx.x; p < P.ns; p += (long long)gridDim.x * BLOCK) {
        const Nbr nb = neighbours(P, p);
        const Vals v = stencil_values(P, Ul, ringn, p, nb);
        const RJ o = residual_jacobian(P, v, nb, 0.0);
        c[p] = o.aC; c[P.ns + p] = o.aE; c[2 * P.ns + p] = o.aW; c[3 * P.ns + p] = o.aN; c[4 * P.ns + p] = o.aS;
    }
}

// A(k, j) of level m from its coefficient rows: row k holds C at j = k, E at k + 1, W at k - 1, N at k + nxu,
// S at k - nxu (summed, so nxu = 1 — where E and W are always dropped — stays correct).
__device__ __forceinline__ double a_entry(const double* __restrict__ c, long long ns, int nxu, long long k, long long j) {
    if (k < 0 || k >= ns) return 0.0;
    const long long d = j - k;
    double v = 0.0;
    if (d == 0) v += c[k];
    if (d == 1) v += c[ns + k];
    if (d == -1) v += c[2 * ns + k];
    if (d == nxu) v += c[3 * ns + k];
    if (d == -nxu) v += c[4 * ns + k];
    return v;
}

// P^1 = A_1 in band form.
__global__ void __launch_bounds__(BLOCK) k_band_init(long long ns, int nxu, int w, const double* __restrict__ c,
                                                     double* __restrict__ B) {
    const long long BW = 2LL * w + 1, N = ns * BW;
    for (long long q = (long long)blockIdx.x * BLOCK + threadIdx.x; q < N; q += (long long)gridDim.x * BLOCK) {
        const long long i = q / BW, j = i + (q % BW) - w;
        B[q] = (j >= 0 && j < ns) ? a_entry(c, ns, nxu, i, j) : 0.0;
    }
}

// P^m = P^{m-1} A_m (Eq. 10 / PAPER.md:221-230): p^m_ij = sum_k p^{m-1}_ik a^m_kj over the <= 5 rows k of
// column j of A_m (Lemma 1).
__global__ void __launch_bounds__(BLOCK) k_band_mul(long long ns, int nxu, int w, const double* __restrict__ Bp,
                                                    const double* __restrict__ c, double* __restrict__ B) {
    const long long BW = 2LL * w + 1, N = ns * BW;
    for (long long q = (long long)blockIdx.x * BLOCK + threadIdx.x; q < N; q += (long long)gridDim.x * BLOCK) {
        const long long i = q / BW, j = i + (q % BW) - w;
        double s = 0.0;
        if (j >= 0 && j < ns) {
            const long long ks[5] = {j, j - 1, j + 1, j - nxu, j + nxu};
            #pragma unroll
            for (int t = 0; t < 5; ++t) {
                const long long k = ks[t], dk = k - i;
                if (k < 0 || k >= ns || dk < -w || dk > w) continue;
                if (nxu == 1 && t >= 3) continue;          // j -+ nxu duplicates j -+ 1: counted once
                s += Bp[i * BW + dk + w] * a_entry(c, ns, nxu, k, j);
            }
        }
        B[q] = s;
    }
}

// y^m = P^{m-1} r^m for window levels m = 2..L (batched over blockIdx.y = m - 2); y^1 = r^1 is left in place.
__global__ void __launch_bounds__(BLOCK) k_band_rhs(long long ns, int w, const double* __restrict__ B,
                                                    const double* __restrict__ R, double* __restrict__ Y) {
    const int m = blockIdx.y + 2;
    const long long BW = 2LL * w + 1;
    const double* Bm = B + (long long)(m - 2) * ns * BW;      // P^{m-1}
    const double* r = R + (long long)(m - 1) * ns;
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < ns; i += (long long)gridDim.x * BLOCK) {
        const long long j0 = i - w < 0 ? 0 : i - w, j1 = i + w >= ns ? ns - 1 : i + w;
        double s = 0.0;
        for (long long j = j0; j <= j1; ++j) s += Bm[i * BW + (j - i) + w] * r[j];
        Y[(long long)(m - 1) * ns + i] = s;
    }
}

// §7 diagonal preconditioner: row i of P^m and r~^m_i divided by p^m_ii (left scaling, R11).
__global__ void __launch_bounds__(BLOCK) k_band_scale(long long ns, int w, double* __restrict__ B, double* __restrict__ Y) {
    const int m = blockIdx.y;
    const long long BW = 2LL * w + 1;
    double* Bm = B + (long long)m * ns * BW;
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < ns; i += (long long)gridDim.x * BLOCK) {
        const double dinv = 1.0 / Bm[i * BW + w];
        for (int c = 0; c < (int)BW; ++c) Bm[i * BW + c] *= dinv;
        Y[(long long)m * ns + i] *= dinv;
    }
}

// Banded LU without pivoting, in place (Doolittle), then forward and back substitution of the
// level's right-hand side: one CTA per window level m (blockIdx.x), half-bandwidth min(m nxu, w).  The pivot
// row and the multipliers of step k are staged in shared memory ([2][w]); a zero or non-finite pivot sets
// err (no pivoting: breakdown is reported, not repaired).  x overwrites Y.
__global__ void __launch_bounds__(BLOCKX) k_band_lu_solve(long long ns, int nxu, int w, double* __restrict__ B,
                                                          double* __restrict__ Y, unsigned* __restrict__ err) {
    extern __shared__ double sh[];
    double* prow = sh;           // [w] u_{k, k+1..k+wb}
    double* lcol = sh + w;       // [w] l_{k+1..k+wb, k}
    const int m = blockIdx.x + 1;
    const long long BW = 2LL * w + 1;
    double* Bm = B + (long long)(m - 1) * ns * BW;
    double* y = Y + (long long)(m - 1) * ns;
    const long long wb = llmin((long long)m * nxu, (long long)w);
    const int tid = threadIdx.x;
    for (long long k = 0; k < ns; ++k) {
        const long long nr = llmin(wb, ns - 1 - k);            // rows / columns below / right of the pivot
        const double piv = Bm[k * BW + w];
        if (tid == 0 && (piv == 0.0 || !isfinite(piv))) atomicOr(err, 1u);
        for (long long t = tid; t < nr; t += BLOCKX) {
            prow[t] = Bm[k * BW + w + 1 + t];                      // u_{k, k+1+t}
            const long long i = k + 1 + t;
            const double l = Bm[i * BW + (k - i) + w] / piv;
            Bm[i * BW + (k - i) + w] = l;
            lcol[t] = l;
        }
        __syncthreads();
        const long long nn = nr * nr;
        for (long long q = tid; q < nn; q += BLOCKX) {
            const long long a = q / nr, b = q % nr;                // row k+1+a, column k+1+b
            const long long i = k + 1 + a, j = k + 1 + b;
            Bm[i * BW + (j - i) + w] -= lcol[a] * prow[b];
        }
        __syncthreads();
    }
    // forward: L z = y (unit lower), column oriented
    for (long long k = 0; k < ns; ++k) {
        const double yk = y[k];
        const long long nr = llmin(wb, ns - 1 - k);
        for (long long t = tid; t < nr; t += BLOCKX) {
            const long long i = k + 1 + t;
            y[i] -= Bm[i * BW + (k - i) + w] * yk;
        }
        __syncthreads();
    }
    // back: U x = z
    for (long long k = ns - 1; k >= 0; --k) {
        if (tid == 0) y[k] /= Bm[k * BW + w];
        __syncthreads();
        const double xk = y[k];
        const long long i0 = llmax(0LL, k - wb);
        for (long long i = i0 + tid; i < k; i += BLOCKX) y[i] -= Bm[i * BW + (k - i) + w] * xk;
        __syncthreads();
    }
}

}  // namespace pit
