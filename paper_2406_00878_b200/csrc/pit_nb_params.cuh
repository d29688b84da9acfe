// pit_nb_params.cuh — engine 4 (pit_newton_nb.cuh) parameter block and the host-side entry points of its
// translation units (pit_nb_law0.cu / pit_nb_law1.cu), so pit_api.cu does not compile the engine's kernels itself.
#pragma once
#include "pit_internal.cuh"

namespace pit {

constexpr int NB_RX = 8;     // LL ring entries per CTA and group for x publications (a group's consumer lags <= 2)
constexpr int NB_RU = 8;     // LL ring entries per CTA and group for U boundary-row publications (one per level)
constexpr int NB_LAG = 4;    // a group may finish at most NB_LAG levels ahead of the next group (< NB_RU - 1)
constexpr int NB_DMAX = 6;   // Newton iterations in flight (upper bound; per instantiation DM <= NB_DMAX)
constexpr int NB_NP = 7;     // per-CTA partials per Newton iteration: sum r^2, max|r|, sum du^2, max|du|,
                             // sum res^2, max|res| (level-solve residuals), sum b^2 (level right-hand sides)
__host__ __device__ constexpr bool nb_is_max(int j) { return j == 1 || j == 3 || j == 5; }

struct NbParams {
    Prob P;
    const double* u0;           // [ns], 16-byte aligned
    const double* ring;         // [nt][ring_len] or nullptr (homogeneous Dirichlet / periodic)
    double* U;                  // [B][nt][ns] iterate ring (iterate k in buffer k % B), buffer 0 = U_0
    int B, D, G;
    const double* ctl;          // [4] = { omega, sweeps, q, check stride } written on the device by k_nb_ctl
    unsigned long long* llx;    // [G][DM][NB_RX][2 sides][NXU / 2] cells (2 words each)
    unsigned long long* llu;    // [G][DM][NB_RU][2 sides][NXU] cells
    double* hpart;              // [MAXK][G][NB_NP]
    unsigned* arrive;           // [MAXK] CTAs done with iteration k
    unsigned* decided;          // [MAXK] 0 = pending, else 16 + status (2 = continue)
    double* hist;               // [newton_max][4]
    double* linres;             // [newton_max][2] = { ||res||_2 / ||b||_2 over all levels, max |res| }
    int* info;                  // [2]
    double* u_out;              // [nt][ns] or nullptr
    double newton_tol;
    int newton_max, stop_norm;
    long long* stats;           // [8 + MAXK]
    unsigned long long* trace;  // optional [G][NB_TR] cycle accounts (nullptr = off)
    const double* carry_in;     // time slab (N4): du_k of the level before level 1 [ns] (nullptr = 0), first pass
    double* carry_out;          // time slab (N4): du_k of level nt [ns] (nullptr = not written)
};
constexpr int NB_TR = 8;        // trace: prologue, sweeps, sweep waits, epilogue, iteration reductions, pass ends, total

// Implemented in pit_nb_law{0,1}.cu: the engine-4 kernel for (base strip height hb, row length nxu), its dynamic
// shared memory and its warp groups (iterations in flight; want_dm = 2 asks for the 2-group build where one
// exists); nullptr if that shape has no instantiation.
const void* nb_kernel_law0(int hb, int nxu, int want_dm, size_t* smem, int* dm, int* threads);
const void* nb_kernel_law1(int hb, int nxu, int want_dm, size_t* smem, int* dm, int* threads);
// omega and the sweep count on the device (k_nb_q + k_nb_ctl, pit_newton_nb.cuh) on stream st
void nb_setup_launch(const Prob& P, const double* U1, const double* ring, unsigned long long* qbits, double lin_rtol,
                     int sweeps, int check, double* ctl, int grid, cudaStream_t st);

}  // namespace pit
