// pit_ps_params.cuh — engine 5 (pit_newton_ps.cuh) parameter block and the host-side entry point of its translation
// unit (pit_ps_law1.cu), so pit_api.cu does not compile the engine's kernels itself.
#pragma once
#include "pit_nb_params.cuh"

namespace pit {

constexpr int PS_RX = 8;     // LL ring entries per CTA for x publications (a neighbour lags <= 2)
constexpr int PS_TR = 8;     // trace: stage wait, prologue, sweeps, LL waits, epilogue, residual check, iteration end, total

struct PsParams {
    Prob P;
    const double* u0;           // [ns], 16-byte aligned
    const double* ring;         // [nt][ring_len] Dirichlet boundary values per level, or nullptr (homogeneous / periodic)
    double* U;                  // [B][nt][ns] iterate ring (iterate k in buffer k % B), buffer 0 = U_0
    int B, D, Gs;               // ring buffers (>= D + 1), CTA sets (iterations in flight), strips per set
    const double* ctl;          // [4] = { omega, sweeps, q, check stride } (k_nb_ctl)
    unsigned long long* llx;    // [D][Gs][PS_RX][2 sides][NXU / 2] cells (2 words each)
    unsigned* lvl;              // [D][Gs] levels a strip has finished: pass * nt + n (release / acquire)
    double* hpart;              // [MAXK][Gs][NB_NP]
    unsigned* arrive;           // [MAXK]
    unsigned* decided;          // [MAXK] 0 = pending, else 16 + status (2 = continue)
    double* hist;               // [newton_max][4]
    double* linres;             // [newton_max][2]
    int* info;                  // [2]
    double* u_out;              // [nt][ns] or nullptr
    double newton_tol;
    int newton_max, stop_norm;
    long long* stats;           // [8 + MAXK]
    unsigned long long* trace;  // optional [D * Gs][PS_TR]
    // LAW 1 coefficients of A_n = I + tau dF/du (host-computed, so the kernel reads them from the constant bank):
    // a_E = ax u_E - bx, a_W = -ax u_W - bx, a_N = ay u_N - by, a_S = -ay u_S - by, a_C = aC1
    double ax, bx, ay, by, aC1, invC1;
    int u0_bcast;               // 1: U_0 = u^0 at every level and was NOT materialised in ring buffer 0 (iteration 0 reads u0)
    int* hint;                  // device word: Newton iterations of the previous solve on this handle (0 = none)
    int dbg;                    // developer experiments (PIT_PS_DBG; 0 = product path): bit 0 = do not wait for LL cells (wrong results, timing only)
};

// Implemented in pit_ps_law1.cu: the engine-5 kernel for (row length, base strip height), its dynamic shared memory
// and threads; rg = row groups per CTA (2; 1 = the 256-thread experiment); trace = the developer build with cycle accounts (PIT_TRACE); nullptr if that shape has no instantiation.
const void* ps_kernel_law1(int nxu, int he, int rg, bool trace, size_t* smem, int* threads);
// Implemented in pit_ps_law0.cu (pit_newton_ps0.cuh): the general law, Dirichlet or periodic.
const void* ps_kernel_law0(int nxu, int he, int periodic, bool trace, size_t* smem, int* threads);

}  // namespace pit
