// pit_api.cu — host side of libpit: the C ABI declared in include/pit.h.
//
// Validation, device memory ownership, launch configuration (cooperative persistent grid sized to the
// SM count), and the host-buffer convenience path.  No arithmetic of the method runs on the host: every
// step of the hot path is a kernel in pit_kernels.cu.  There is no CPU fallback.
#include "pit.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "pit_kernels.cu"
#include "pit_guess.cuh"
#include "pit_explicit.cuh"
#include "pit_nb_params.cuh"
#include "pit_ps_params.cuh"

using namespace pit;

// NVTX range around each stage the host issues (visible in nsys / ncu --nvtx; no cost without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct pit_handle {
    pit_config cfg;
    Prob P;
    int device = 0, sms = 0, G = 0, D = 1, B = 3, occ = 1;
    int engine = 1;               // 1 = global-state k_newton, 2 = on-chip k_newton_onchip<ppt>
    int ppt = 0, hmax = 0, law = 0;
    size_t smem2 = 0;
    BarState* bs = nullptr;
    unsigned long long* trace = nullptr;   // [7] cycle accounting when PIT_TRACE is set
    double* pf_Y = nullptr;       // (b2) product-form scratch: [2][nt][ns] chain vectors
    double* pf_R = nullptr;       // (b2) host-driven Newton: residuals [nt][ns]
    double* pf_dU = nullptr;      // (b2) host-driven Newton: update [nt][ns]
    double* pf_part = nullptr;    // (b2) partials
    int product_used = 0;         // last solve: 0 level recurrence, 1 (b2) product form, 2 N3 explicit banded form
    double* ex_B = nullptr;       // N3: band storage of P^1..P^L of a window [L][ns][2w+1]
    double* ex_C5 = nullptr;      // N3: coefficients of A_{s0..s0+L-1} [L][5][ns]
    long long ex_capB = 0, ex_capC = 0;
    unsigned* ex_err = nullptr;   // N3: zero / non-finite pivot flag
    double* U = nullptr;          // [B][nt][ns]
    double* slots = nullptr;      // [D][NVEC][ns]
    double* part = nullptr;       // [2][G][NPART]
    double* hpart = nullptr;      // [max(2, D)][G][4]
    double* halo = nullptr;       // engine 3: [G][2][6][512] published strip boundary rows
    GridBar* bar = nullptr;
    double* hist = nullptr;       // [newton_max][4]
    int* info = nullptr;          // [2]
    long long* stats = nullptr;   // [8 + MAXK]: steps, max-per-step inner its, D, G, sum over pairs, -, -, -, per-k sums
    double* d_u0 = nullptr;       // host-path staging
    double* d_bc = nullptr;
    double* d_small = nullptr;    // [2 * 1024] scratch for kernel (a) partials + norms
    long long bytes = 0;
    long long launches = 0;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // k_init, k_newton, guess start/end
    bool timed = false, guess_timed = false;
    // coarse-grid initial guess (guess_cf >= 2): nested handle on the coarsened problem
    pit_handle* coarse = nullptr;
    GuessParams gp;
    double* c_u0 = nullptr;       // [nsc]
    double* c_ring = nullptr;     // [ntc][ring_len_c] (Dirichlet)
    double* c_U = nullptr;        // [ntc][nsc] coarse solution
    double* c_fac = nullptr;      // [2][Kmax] spline factors
    int* c_info = nullptr;        // [2]
    cudaGraphExec_t c_march = nullptr;   // the coarse level march captured once as a CUDA graph (launch overhead)
    long long c_march_launches = 0;
    // engine 4 (neighbour-synchronised RB-SOR Newton solve, pit_newton_nb.cuh)
    bool nb = false;              // the Newton solve runs on engine 4
    int nb_rmax = 0, nb_G = 0, nb_D = 0, nb_dm = 0;   // base strip height, CTAs, iterations in flight, warp groups
    int nb_threads = 0;                               // threads per CTA
    int nb_want = 0;                                  // warp groups asked of the instantiation table (0 = the shape's default)
    bool nb_ctl_ready = false;                        // slab iterations: omega / sweeps fixed at the first call
    size_t nb_smem = 0;
    unsigned long long* nb_llx = nullptr;   // LL cells, x publications
    unsigned long long* nb_llu = nullptr;   // LL cells, U boundary-row publications
    size_t nb_llx_bytes = 0, nb_llu_bytes = 0;
    double* nb_hpart = nullptr;   // [MAXK][G][NB_NP]
    unsigned* nb_sync = nullptr;  // [2][MAXK] arrive counters, decisions
    unsigned long long* nb_qbits = nullptr;
    double* nb_ctl = nullptr;     // [4] omega, sweeps, q
    double* nb_linres = nullptr;  // [MAXK][2]
    // engine 5 (pipeline of CTA sets, strips on chip, pit_newton_ps.cuh)
    bool ps = false;              // the Newton solve runs on engine 5
    int ps_D = 0, ps_Gs = 0, ps_he = 0, ps_threads = 0;   // CTA sets, strips per set, base strip height, threads per CTA
    size_t ps_smem = 0;
    unsigned long long* ps_llx = nullptr;   // [D][Gs][PS_RX][2][nxu / 2] LL cells
    unsigned* ps_lvl = nullptr;             // [D][Gs] level counters
    int ps_rg = 2;                          // row groups per CTA (PIT_PS_DBG bit 2: the one-group experiment)
    // pit_solve (host buffers) streams the probable final iterate to the host while engine 5 still runs
    cudaStream_t ps_cs = nullptr;           // non-blocking copy stream
    cudaEvent_t ps_ev_reset = nullptr;      // the level counters of this solve are cleared
    unsigned* ps_h_lvl = nullptr;           // pinned host copy of the level counters
    int ps_host_kf = 0;                     // Newton iterations of the previous pit_solve on this handle (0 = none)
    int* ps_hint = nullptr;                 // device word: Newton iterations of the previous engine-5 solve (0 = none)
    size_t ps_llx_bytes = 0;
    int last_engine = 0;          // engine of the last Newton solve
    // developer switches (pit.h "Debug environment"), read once at pit_create so a handle never changes path
    struct {
        bool trace = false;       // PIT_TRACE: cycle accounting of the persistent kernels
        bool resjac_v1 = false;   // PIT_RESJAC_V1: kernel (a) without TMA staging
        int resjac_rt = 0, resjac_ns = 0;   // PIT_RESJAC_RT / _NS: kernel (a) tile rows / pipeline stages
        int x0carry = 1;          // PIT_X0=0: engines 2-3 start level solves from 0 instead of the carry
        bool merge = true;        // PIT_MERGE=0: engine 3 without the merged first BiCGSTAB iteration
        bool guess_graph = true;  // PIT_GUESS_GRAPH=0: the coarse-grid march without a CUDA graph
        int ps_dbg = 0;           // PIT_PS_DBG: engine-5 timing experiments (bit 0: no LL waits — wrong results)
    } dbg;
    int c_march_ring = -1;        // the ring presence the coarse-march graph was captured with (-1: none captured)
    // caller-owned workspace (pit_create_with_workspace): every create-time buffer is carved from it
    char* ws = nullptr;
    size_t ws_size = 0, ws_off = 0;
    bool measure = false;         // pit_workspace_bytes: size the buffers, allocate nothing
    char err[512] = {0};
};

static constexpr size_t WS_ALIGN = 256;
static size_t ws_align(size_t b) { return (b + WS_ALIGN - 1) / WS_ALIGN * WS_ALIGN; }

// Frees a buffer unless it lives in the caller's workspace.
static void dfree(pit_handle* h, void* p) {
    if (!p) return;
    if (h->ws && (char*)p >= h->ws && (char*)p < h->ws + h->ws_size) return;
    cudaFree(p);
}

static int set_err(pit_handle* h, int code, const char* fmt, ...) {
    if (h) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(h->err, sizeof(h->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define CUDA_TRY(h, call)                                                                              \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) return set_err((h), PIT_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// (the definitions below inherit C linkage from the extern "C" declarations in pit.h)

void pit_config_init(pit_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->abi_version = PIT_ABI_VERSION;
    c->x1 = 1.0;
    c->y1 = 1.0;
    c->newton_tol = 1e-12;
    c->newton_max = 30;
}

int pit_abi_version(void) { return PIT_ABI_VERSION; }

const char* pit_strerror(int code) {
    switch (code) {
        case PIT_OK: return "converged";
        case PIT_OK_FLOOR: return "converged at the rounding floor";
        case PIT_EINVAL: return "invalid argument";
        case PIT_ENOMEM: return "device allocation failed";
        case PIT_ECUDA: return "CUDA error";
        case PIT_ENOCONV: return "Newton did not converge within newton_max";
        case PIT_EBREAKDOWN: return "Krylov breakdown or non-finite value";
        case PIT_ECOND: return "product-form window rejected by the Section 7 conditioning gate";
        default: return "unknown status";
    }
}

const char* pit_last_error(const pit_handle* h) { return h ? h->err : "null handle"; }

static int validate(const pit_config* c, char* why, size_t n) {
    if (!c) { snprintf(why, n, "cfg is NULL"); return PIT_EINVAL; }
    if (c->abi_version != PIT_ABI_VERSION) { snprintf(why, n, "abi_version %d != %d", c->abi_version, PIT_ABI_VERSION); return PIT_EINVAL; }
    if (c->pde != PIT_HEAT && c->pde != PIT_BURGERS) { snprintf(why, n, "pde %d", c->pde); return PIT_EINVAL; }
    if (c->bc != PIT_DIRICHLET && c->bc != PIT_PERIODIC) { snprintf(why, n, "bc %d", c->bc); return PIT_EINVAL; }
    const int nmin = c->bc == PIT_DIRICHLET ? 2 : 3;
    if (c->nx < nmin || c->ny < nmin) { snprintf(why, n, "nx, ny must be >= %d", nmin); return PIT_EINVAL; }
    if (c->nx > (1 << 20) || c->ny > (1 << 20)) { snprintf(why, n, "nx, ny too large"); return PIT_EINVAL; }
    if (c->nt < 1) { snprintf(why, n, "nt must be >= 1"); return PIT_EINVAL; }
    if (!(c->x1 > c->x0) || !(c->y1 > c->y0)) { snprintf(why, n, "empty domain"); return PIT_EINVAL; }
    if (!(c->dt > 0.0) || !std::isfinite(c->dt)) { snprintf(why, n, "dt must be > 0"); return PIT_EINVAL; }
    if (!(c->m0 >= 0.0) || !(c->m2 >= 0.0)) { snprintf(why, n, "mu = m0 + m2 u^2 needs m0, m2 >= 0 (PAPER.md:50)"); return PIT_EINVAL; }
    if (!(c->newton_tol > 0.0)) { snprintf(why, n, "newton_tol must be > 0"); return PIT_EINVAL; }
    if (c->newton_max < 1 || c->newton_max > MAXK) { snprintf(why, n, "newton_max must be in 1..%d", MAXK); return PIT_EINVAL; }
    if (c->lin_rtol < 0.0 || c->lin_atol < 0.0 || c->lin_max < 0) { snprintf(why, n, "negative solver tolerance"); return PIT_EINVAL; }
    if (c->inverse_mode < 0 || c->inverse_mode > 3) { snprintf(why, n, "inverse_mode %d", c->inverse_mode); return PIT_EINVAL; }
    if (c->inverse_mode == PIT_INV_EXPLICIT && c->bc != PIT_DIRICHLET) {
        snprintf(why, n, "inverse_mode EXPLICIT needs Dirichlet boundaries (the periodic wrap makes P^n non-banded)");
        return PIT_EINVAL;
    }
    if (c->pipeline_depth < 0 || c->pipeline_depth > MAXD) { snprintf(why, n, "pipeline_depth must be in 0..%d", MAXD); return PIT_EINVAL; }
    if (c->window < 0) { snprintf(why, n, "window < 0"); return PIT_EINVAL; }
    if (c->engine < 0 || c->engine > 5) { snprintf(why, n, "engine %d", c->engine); return PIT_EINVAL; }
    if (c->lin_sweeps < 0 || c->lin_sweeps > 400) { snprintf(why, n, "lin_sweeps must be in 0..400"); return PIT_EINVAL; }
    if (c->lin_check < 0) { snprintf(why, n, "lin_check < 0"); return PIT_EINVAL; }
    if (c->stop_norm < 0 || c->stop_norm > 1) { snprintf(why, n, "stop_norm %d", c->stop_norm); return PIT_EINVAL; }
    if (c->guess_cf == 1 || c->guess_cf < 0) { snprintf(why, n, "guess_cf must be 0 or >= 2"); return PIT_EINVAL; }
    if (c->guess_cf >= 2) {
        const int f = c->guess_cf;
        if (c->nx % f || c->ny % f || c->nt % f) { snprintf(why, n, "guess_cf %d must divide nx, ny and nt", f); return PIT_EINVAL; }
        if (c->nx / f < nmin || c->ny / f < nmin) { snprintf(why, n, "coarse grid below %d intervals", nmin); return PIT_EINVAL; }
    }
    return PIT_OK;
}

static void free_all(pit_handle* h) {
    for (auto& e : h->ev) if (e) { cudaEventDestroy(e); e = nullptr; }
    dfree(h, h->U); dfree(h, h->slots); dfree(h, h->part); dfree(h, h->hpart); dfree(h, h->halo); dfree(h, h->bar);
    dfree(h, h->hist); dfree(h, h->info); dfree(h, h->stats); dfree(h, h->d_u0); dfree(h, h->d_bc);
    dfree(h, h->d_small); dfree(h, h->bs); dfree(h, h->trace);
    dfree(h, h->pf_Y); dfree(h, h->pf_R); dfree(h, h->pf_dU); dfree(h, h->pf_part);
    dfree(h, h->ex_B); dfree(h, h->ex_C5); dfree(h, h->ex_err);
    dfree(h, h->nb_llx); dfree(h, h->nb_llu); dfree(h, h->nb_hpart); dfree(h, h->nb_sync); dfree(h, h->nb_qbits);
    dfree(h, h->nb_ctl); dfree(h, h->nb_linres);
    dfree(h, h->ps_llx); dfree(h, h->ps_lvl); dfree(h, h->ps_hint);
    h->ps_llx = nullptr; h->ps_lvl = nullptr; h->ps_hint = nullptr;
    h->nb_llx = h->nb_llu = nullptr; h->nb_hpart = h->nb_ctl = h->nb_linres = nullptr; h->nb_sync = nullptr;
    h->nb_qbits = nullptr;
    h->ex_B = h->ex_C5 = nullptr; h->ex_err = nullptr; h->ex_capB = h->ex_capC = 0;
    if (h->c_march) cudaGraphExecDestroy(h->c_march);
    h->c_march = nullptr;
    dfree(h, h->c_u0); dfree(h, h->c_ring); dfree(h, h->c_U); dfree(h, h->c_fac); dfree(h, h->c_info);
    h->c_u0 = h->c_ring = h->c_U = h->c_fac = nullptr; h->c_info = nullptr;
    if (h->coarse) { pit_destroy(h->coarse); h->coarse = nullptr; }
    h->bs = nullptr; h->trace = nullptr; h->pf_Y = h->pf_R = h->pf_dU = h->pf_part = nullptr;
    h->halo = nullptr;
    h->U = h->slots = h->part = h->hpart = h->hist = h->d_u0 = h->d_bc = h->d_small = nullptr;
    h->bar = nullptr; h->info = nullptr; h->stats = nullptr;
}

// Device buffer of `count` elements: carved from the caller's workspace (pit_create_with_workspace), only sized
// (pit_workspace_bytes), or cudaMalloc'd.  `lazy` buffers (the product forms' scratch, grown on first use) always
// come from cudaMalloc: they are outside the create-time workspace contract (pit.h).
template <class T>
static int dalloc(pit_handle* h, T** p, size_t count, bool lazy = false) {
    const size_t b = std::max<size_t>(count, 1) * sizeof(T);
    if (!lazy && h->measure) {
        *p = nullptr;
        h->bytes += (long long)ws_align(b);
        return PIT_OK;
    }
    if (!lazy && h->ws) {
        const size_t off = ws_align(h->ws_off);
        if (off + b > h->ws_size)
            return set_err(h, PIT_ENOMEM, "workspace of %zu bytes too small (pit_workspace_bytes)", h->ws_size);
        *p = reinterpret_cast<T*>(h->ws + off);
        h->ws_off = off + b;
        h->bytes += (long long)b;
        return PIT_OK;
    }
    cudaError_t e = cudaMalloc((void**)p, b);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(h, PIT_ENOMEM, "cudaMalloc(%zu bytes): %s", b, cudaGetErrorString(e));
    }
    h->bytes += (long long)b;
    return PIT_OK;
}

template <bool TR, int LAW>
static const void* onchip_fn_t(int ppt) {
    switch (ppt) {
        case 1: return (const void*)k_newton_onchip<1, TR, LAW>;
        case 2: return (const void*)k_newton_onchip<2, TR, LAW>;
        case 4: return (const void*)k_newton_onchip<4, TR, LAW>;
        case 8: return (const void*)k_newton_onchip<8, TR, LAW>;
        default: return (const void*)k_newton_onchip<16, TR, LAW>;
    }
}

template <bool TR, int LAW, int NXU>
static const void* col_fn_t(int rmax) {
    return rmax <= 4 ? (const void*)k_newton_col<4, TR, LAW, NXU>
                     : (rmax <= 7 ? (const void*)k_newton_col<7, TR, LAW, NXU> : (const void*)k_newton_col<8, TR, LAW, NXU>);
}

template <int NXU>
static const void* col_fn_n(int rmax, bool trace, int law) {
    if (law == 1) return trace ? col_fn_t<true, 1, NXU>(rmax) : col_fn_t<false, 1, NXU>(rmax);
    return trace ? col_fn_t<true, 0, NXU>(rmax) : col_fn_t<false, 0, NXU>(rmax);
}

static const void* col_fn(int rmax, bool trace, int law, int nxu) {
    return nxu == 512 ? col_fn_n<512>(rmax, trace, law) : col_fn_n<256>(rmax, trace, law);
}

// Engine 4 kernel for (base strip height, law, row length): its own translation units (pit_nb_law*.cu).
static const void* nb_fn(int hb, int law, int nxu, int want_dm, size_t* smem, int* dm, int* threads) {
    return law == 1 ? nb_kernel_law1(hb, nxu, want_dm, smem, dm, threads) : nb_kernel_law0(hb, nxu, want_dm, smem, dm, threads);
}

// LAW 1 = viscous Burgers with constant viscosity (m2 = 0): specialised matvec coefficients.
static const void* onchip_fn(int ppt, bool trace, int law) {
    if (law == 1) return trace ? onchip_fn_t<true, 1>(ppt) : onchip_fn_t<false, 1>(ppt);
    return trace ? onchip_fn_t<true, 0>(ppt) : onchip_fn_t<false, 0>(ppt);
}

static int create_impl(const pit_config* cfg, char* ws, size_t ws_size, bool measure, pit_handle** out);

// Engine 5 kernel for the handle's law, boundary condition and row length at base strip height he.
static const void* ps_fn(const pit_handle* h, int he, size_t* smem, int* threads) {
    return h->law == 1 ? ps_kernel_law1(h->P.nxu, he, h->ps_rg, h->dbg.trace, smem, threads)
                       : ps_kernel_law0(h->P.nxu, he, h->P.bc == PIT_PERIODIC ? 1 : 0, h->dbg.trace, smem, threads);
}

// The c_f-coarsened problem of the initial guess: N_x / c_f, N_y / c_f intervals, N_t / c_f levels
// of step c_f dt, same law, domain and solver settings.  "Solving Eq. (FDS) sequentially": the nested handle is
// a ONE-level problem; build_guess marches it level by level (u^0 of level m = the converged level m-1), so its
// Newton iteration at each level is exactly the sequential method's (same engines, on the device).
static int create_coarse(pit_handle* h) {
    const pit_config& c = h->cfg;
    const int f = c.guess_cf;
    pit_config cc = c;
    cc.nx = c.nx / f; cc.ny = c.ny / f; cc.nt = 1; cc.dt = c.dt * f;
    cc.guess_cf = 0; cc.pipeline_depth = 0; cc.engine = 0; cc.window = 0; cc.stop_norm = 0;
    cc.inverse_mode = PIT_INV_RECURRENCE;
    int rc;
    if (h->measure) {                       // the nested handle's buffers count into this handle's workspace
        pit_handle* m = nullptr;
        if ((rc = create_impl(&cc, nullptr, 0, true, &m)) != PIT_OK) return set_err(h, rc, "coarse-grid handle: %s", pit_strerror(rc));
        h->bytes += m->bytes + (long long)WS_ALIGN;
        h->coarse = m;                      // kept for its problem constants below; freed with h (it owns nothing)
    } else if (h->ws) {                     // nested handle carved from this handle's workspace
        size_t need = 0;
        if ((rc = pit_workspace_bytes(&cc, &need)) != PIT_OK) return set_err(h, rc, "coarse-grid handle: %s", pit_strerror(rc));
        const size_t off = ws_align(h->ws_off);
        if (off + need > h->ws_size) return set_err(h, PIT_ENOMEM, "workspace of %zu bytes too small", h->ws_size);
        if ((rc = create_impl(&cc, h->ws + off, need, false, &h->coarse)) != PIT_OK)
            return set_err(h, rc, "coarse-grid handle: %s", pit_strerror(rc));
        h->ws_off = off + need;
    } else if ((rc = pit_create(&cc, &h->coarse)) != PIT_OK) {
        return set_err(h, rc, "coarse-grid handle: %s", pit_strerror(rc));
    }
    GuessParams& g = h->gp;
    std::memset(&g, 0, sizeof(g));
    const Prob& P = h->P;
    const Prob& Q = h->coarse->P;
    g.cf = f; g.bc = P.bc;
    g.nx = P.nx; g.ny = P.ny; g.nt = P.nt; g.nxu = P.nxu; g.nyu = P.nyu; g.ns = P.ns;
    g.nxc = Q.nx; g.nyc = Q.ny; g.ntc = P.nt / f; g.nxuc = Q.nxu; g.nyuc = Q.nyu; g.nsc = Q.ns; g.ring_len_c = Q.ring_len;
    const int kmax = std::max(std::max(Q.nx, Q.ny) + 1, g.ntc + 1);
    if ((rc = dalloc(h, &h->c_u0, (size_t)Q.ns)) ||
        (rc = dalloc(h, &h->c_ring, (size_t)(P.bc == PIT_DIRICHLET ? (long long)g.ntc * Q.ring_len : 1))) ||
        (rc = dalloc(h, &h->c_U, (size_t)(Q.ns * g.ntc))) ||
        (rc = dalloc(h, &h->c_fac, (size_t)(2 * kmax))) ||
        (rc = dalloc(h, &h->c_info, 2)))
        return rc;
    return PIT_OK;
}

static int create_impl(const pit_config* cfg, char* ws, size_t ws_size, bool measure, pit_handle** out) {
    if (!out) return PIT_EINVAL;
    *out = nullptr;
    char why[256];
    int rc = validate(cfg, why, sizeof(why));
    if (rc != PIT_OK) return rc;
    pit_handle* h = new (std::nothrow) pit_handle();
    if (!h) return PIT_ENOMEM;
    h->ws = ws;
    h->ws_size = ws_size;
    h->measure = measure;
    h->cfg = *cfg;
    {
        auto env_int = [](const char* n, int dflt) { const char* v = getenv(n); return v ? atoi(v) : dflt; };
        h->dbg.trace = getenv("PIT_TRACE") != nullptr;
        h->dbg.resjac_v1 = getenv("PIT_RESJAC_V1") != nullptr;
        h->dbg.resjac_rt = env_int("PIT_RESJAC_RT", 0);
        h->dbg.resjac_ns = env_int("PIT_RESJAC_NS", 0);
        h->dbg.x0carry = env_int("PIT_X0", 1);
        h->dbg.merge = env_int("PIT_MERGE", 1) != 0;
        h->dbg.guess_graph = env_int("PIT_GUESS_GRAPH", 1) != 0;
        h->dbg.ps_dbg = env_int("PIT_PS_DBG", 0);
        h->ps_rg = (h->dbg.ps_dbg & 4) ? 1 : 2;
    }
    pit_config& c = h->cfg;
    if (c.lin_rtol == 0.0) c.lin_rtol = 1e-6;     // inexact-Newton forcing term (R10)
    if (c.lin_atol == 0.0) c.lin_atol = 1e-4 * c.newton_tol;
    if (c.lin_max == 0) c.lin_max = 1000;

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        delete h;
        return PIT_ECUDA;
    }
    if (c.device < 0 || c.device >= ndev) { delete h; return PIT_EINVAL; }
    h->device = c.device;
    cudaDeviceProp prop;
    if (cudaSetDevice(h->device) != cudaSuccess || cudaGetDeviceProperties(&prop, h->device) != cudaSuccess) {
        cudaGetLastError();
        delete h;
        return PIT_ECUDA;
    }
    if (prop.major != 10 || !prop.cooperativeLaunch) {   // built for sm_100a only
        delete h;
        return PIT_ECUDA;
    }
    h->sms = prop.multiProcessorCount;

    Prob& P = h->P;
    P.pde = c.pde; P.bc = c.bc; P.nx = c.nx; P.ny = c.ny;
    P.nxu = c.bc == PIT_DIRICHLET ? c.nx - 1 : c.nx;
    P.nyu = c.bc == PIT_DIRICHLET ? c.ny - 1 : c.ny;
    P.nt = c.nt;
    P.ring_len = 2 * (c.nx + c.ny);
    P.ns = (long long)P.nxu * P.nyu;
    const double hx = (c.x1 - c.x0) / c.nx, hy = (c.y1 - c.y0) / c.ny;
    P.ihx2 = 1.0 / (hx * hx); P.ihy2 = 1.0 / (hy * hy);
    P.i2hx = 1.0 / (2.0 * hx); P.i2hy = 1.0 / (2.0 * hy);
    P.dt = c.dt; P.m0 = c.m0; P.m2 = c.m2;

    // ---- engine selection ----
    // On-chip engine (default): one 512-thread CTA per SM; pipeline depth D = the largest value <= 8
    // (<= newton_max) whose level strips fit the register/shared-memory budget (PPT <= 8 points per
    // thread, <= 200 KB shared).  Otherwise the global-state engine (any size).
    const int Dmax = std::max(1, std::min(c.pipeline_depth > 0 ? c.pipeline_depth : 8, c.newton_max));
    const int law = (c.pde == PIT_BURGERS && c.m2 == 0.0) ? 1 : 0;
    h->law = law;
    // Column-blocked on-chip engine (engine 3): nx = 256 or 512, one 512-thread CTA per SM, a thread owns a
    // column of at most RMAX (4 or 8) strip rows.  Preferred whenever it fits.
    if ((c.engine == 0 || c.engine == 3) && (P.nxu == 256 || P.nxu == 512) && h->sms <= 160) {
        const int Gr = BLOCK3 / P.nxu;
        for (int D = Dmax; D >= 1 && h->engine != 3; --D) {
            const int C = h->sms / D;
            if (C < 1) continue;
            const int hmax = (P.nyu + C - 1) / C;
            const int rows = (hmax + Gr - 1) / Gr;
            const int rmax = rows <= 4 ? 4 : (rows <= 7 ? 7 : (rows <= 8 ? 8 : 0));
            if (!rmax) continue;
            const size_t smem = (size_t)((2 * hmax + 4) * (P.nxu + 4) + (law == 1 ? 4 : 5) * rmax * BLOCK3) * sizeof(double);
            if (smem > 220 * 1024) continue;
            bool ok = true;
            int occ3 = 0;
            for (bool tr : {false, true}) {
                const void* fn = col_fn(rmax, tr, law, P.nxu);
                ok = ok && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
                     cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, fn, BLOCK3, smem) == cudaSuccess && occ3 >= 1;
            }
            if (!ok) { cudaGetLastError(); continue; }
            h->engine = 3; h->D = D; h->ppt = rmax; h->hmax = hmax; h->smem2 = smem; h->G = h->sms; h->occ = 1;
        }
        if (h->engine != 3 && c.engine == 3) { delete h; return PIT_EINVAL; }
    }
    if ((c.engine == 0 || c.engine == 2) && h->engine == 1 && P.nxu <= BLOCK2 && h->sms <= 160) {
        for (int D = Dmax; D >= 1 && h->engine != 2; --D) {
            const int C = h->sms / D;
            if (C < 1) continue;
            const int hmax = (P.nyu + C - 1) / C;
            const long long need = (long long)hmax * P.nxu;
            int ppt = 0;
            for (int cand : {1, 2, 4, 8, 16})
                if (need <= (long long)cand * BLOCK2) { ppt = cand; break; }
            if (!ppt) continue;
            const size_t smem = (size_t)(2 * (hmax + 2) * (P.nxu + 2) + 4 * ppt * BLOCK2) * sizeof(double);
            if (smem > 220 * 1024) continue;
            int occ2 = 0;
            bool ok = true;
            for (bool tr : {false, true}) {
                const void* fn = onchip_fn(ppt, tr, law);
                ok = ok && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
                     cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, fn, BLOCK2, smem) == cudaSuccess && occ2 >= 1;
            }
            if (!ok) {
                cudaGetLastError();
                continue;
            }
            h->engine = 2; h->D = D; h->ppt = ppt; h->hmax = hmax; h->smem2 = smem; h->G = h->sms; h->occ = 1;
        }
        if (h->engine != 2 && c.engine == 2) { delete h; return PIT_EINVAL; }
    }
    if (h->engine == 1) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_newton, BLOCK, 0) != cudaSuccess || occ < 1) {
            cudaGetLastError();
            delete h;
            return PIT_ECUDA;
        }
        h->occ = std::min(occ, 2);
        h->G = h->sms * h->occ;
        // Pipeline depth: keep the slot state (13 vectors per level) within ~96 MB (L2 is 126 MB).
        const long long slot_bytes = (long long)NVEC * P.ns * 8;
        int D = c.pipeline_depth;
        if (D == 0) D = (int)std::min<long long>(8, std::max<long long>(1, (96ll << 20) / std::max<long long>(slot_bytes, 1)));
        h->D = std::max(1, std::min(D, c.newton_max));
    }
    // Engine 4 (the Newton solve): rows of 64..512 unknowns (even), <= 4 rows per CTA, one CTA per SM.
    if ((c.engine == 0 || c.engine == 4) && (c.inverse_mode == PIT_INV_AUTO || c.inverse_mode == PIT_INV_RECURRENCE) &&
        (P.nxu == 64 || P.nxu == 128 || P.nxu == 256 || P.nxu == 512) && (c.bc == PIT_DIRICHLET || P.nyu % 2 == 0)) {
        const int G4 = std::min(h->sms, P.nyu);
        const int hb4 = P.nyu / G4;
        size_t smem4 = 0;
        int occ4 = 0, dm = 1, thr4 = 0;
        // rows of 256 unknowns, one row per CTA: six warp groups by default (a six-iteration solve in one pass of the
        // level wavefront: c3 63.8 -> 50.0 ms), else the shape's default build
        h->nb_want = c.pipeline_depth > 0 ? c.pipeline_depth : ((P.nxu == 256 && hb4 == 1 && c.newton_max >= 6) ? 6 : 0);
        const void* fn = nb_fn(hb4, law, P.nxu, h->nb_want, &smem4, &dm, &thr4);
        const int D4 = std::max(1, std::min(c.pipeline_depth > 0 ? c.pipeline_depth : dm, std::min(dm, c.newton_max)));
        const int rmax = hb4;
        if (fn && smem4 <= 227 * 1024 && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, fn, thr4, smem4) == cudaSuccess && occ4 >= 1) {
            h->nb = true; h->nb_rmax = rmax; h->nb_G = G4; h->nb_D = D4; h->nb_smem = smem4; h->nb_dm = dm;
            h->nb_threads = thr4;
        }
        cudaGetLastError();
    }
    if (c.engine == 4 && !h->nb) { delete h; return PIT_EINVAL; }
    // Engine 5 (the Newton solve): constant-viscosity Burgers on periodic grids, rows of 512 unknowns; D CTA sets of Gs
    // strips with HE or HE + 2 rows each (HE even: every strip starts on an even row).  D = pipeline_depth, or the
    // largest depth <= min(8, newton_max) whose strips fit on chip.
    if ((c.engine == 0 || c.engine == 5) && (c.inverse_mode == PIT_INV_AUTO || c.inverse_mode == PIT_INV_RECURRENCE) &&
        (law == 1 ? c.bc == PIT_PERIODIC : true) && P.nyu % 2 == 0) {
        const int dmax = std::max(1, std::min(c.pipeline_depth > 0 ? c.pipeline_depth : 8, c.newton_max));
        for (int D5 = dmax; D5 >= 1 && !h->ps; --D5) {
            for (int Gs = std::min(h->sms / D5, P.nyu / 2); Gs >= 1 && !h->ps; --Gs) {
                const int he = 2 * (P.nyu / (2 * Gs));
                const int na = (P.nyu - he * Gs) / 2;          // strips with he + 2 rows
                if (he < 2 || na < 0 || na > Gs) continue;
                size_t smem5 = 0;
                int thr5 = 0, occ5 = 0, he_used = he;
                const void* fn = ps_fn(h, he, &smem5, &thr5);
                if (!fn && na == 0 && he >= 4) {      // every strip has he rows = (he - 2) + 2
                    he_used = he - 2;
                    fn = ps_fn(h, he_used, &smem5, &thr5);
                }
                if (!fn || smem5 > 227 * 1024) continue;
                if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem5) != cudaSuccess ||
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ5, fn, thr5, smem5) != cudaSuccess || occ5 < 1) {
                    cudaGetLastError();
                    continue;
                }
                h->ps = true; h->ps_D = D5; h->ps_Gs = Gs; h->ps_he = he_used; h->ps_threads = thr5; h->ps_smem = smem5;
                break;       // the largest Gs of this depth only: fewer strips would only lengthen them
            }
            if (c.pipeline_depth > 0) break;
        }
        cudaGetLastError();
    }
    if (c.engine == 5 && !h->ps) { delete h; return PIT_EINVAL; }
    const int D = h->D;
    h->B = std::max(std::max(std::max(3, D), h->nb ? h->nb_D + 1 : 0), h->ps ? h->ps_D + 1 : 0);

    const long long N = P.ns * P.nt;
    if ((rc = dalloc(h, &h->U, (size_t)(h->B * N))) ||
        (rc = dalloc(h, &h->slots, (size_t)(D * NVEC * P.ns))) ||
        (rc = dalloc(h, &h->part, (size_t)(2 * h->G * NPART))) ||
        (rc = dalloc(h, &h->hpart, (size_t)(std::max(2, D) * h->G * 4))) ||
        (h->engine == 3 && (rc = dalloc(h, &h->halo, (size_t)h->G * HALO_CTA))) ||
        (rc = dalloc(h, &h->bar, 1)) ||
        (rc = dalloc(h, &h->hist, (size_t)(4 * c.newton_max))) ||
        (rc = dalloc(h, &h->info, 2)) ||
        (rc = dalloc(h, &h->stats, 8 + MAXK)) ||
        (rc = dalloc(h, &h->d_u0, (size_t)P.ns)) ||
        (rc = dalloc(h, &h->d_bc, (size_t)(c.bc == PIT_DIRICHLET ? (long long)P.nt * P.ring_len : 1))) ||
        (rc = dalloc(h, &h->d_small, 2 * 1024 + 2)) ||
        (rc = dalloc(h, &h->bs, 1)) ||
        (h->dbg.trace && (rc = dalloc(h, &h->trace, 13 + 13 * GMAX2 + (h->ps ? (size_t)h->ps_D * h->ps_Gs * PS_TR : 0)))) ||
        (h->nb && ((rc = dalloc(h, &h->nb_llx, (size_t)h->nb_G * h->nb_dm * NB_RX * 2 * (P.nxu / 2) * 2)) ||
                   (rc = dalloc(h, &h->nb_llu, (size_t)h->nb_G * h->nb_dm * NB_RU * 2 * P.nxu * 2)))) ||
        (h->ps && ((rc = dalloc(h, &h->ps_llx, (size_t)h->ps_D * h->ps_Gs * PS_RX * 2 * (P.nxu / 2) * 2)) ||
                   (rc = dalloc(h, &h->ps_lvl, (size_t)h->ps_D * h->ps_Gs)) ||
                   (rc = dalloc(h, &h->ps_hint, 1)))) ||
        ((h->nb || h->ps) && ((rc = dalloc(h, &h->nb_hpart, (size_t)MAXK * std::max(h->nb_G, h->ps_Gs) * NB_NP)) ||
                   (rc = dalloc(h, &h->nb_sync, (size_t)2 * MAXK)) ||
                   (rc = dalloc(h, &h->nb_qbits, 1)) ||
                   (rc = dalloc(h, &h->nb_ctl, 4)) ||
                   (rc = dalloc(h, &h->nb_linres, (size_t)2 * MAXK))))) {
        free_all(h);
        delete h;
        return rc;
    }
    h->nb_llx_bytes = (size_t)h->nb_G * h->nb_dm * NB_RX * 2 * (P.nxu / 2) * 2 * sizeof(unsigned long long);
    h->nb_llu_bytes = (size_t)h->nb_G * h->nb_dm * NB_RU * 2 * P.nxu * 2 * sizeof(unsigned long long);
    h->ps_llx_bytes = (size_t)h->ps_D * h->ps_Gs * PS_RX * 2 * (P.nxu / 2) * 2 * sizeof(unsigned long long);
    bool ev_ok = true;
    for (auto& e : h->ev) ev_ok = ev_ok && cudaEventCreate(&e) == cudaSuccess;
    if (!ev_ok || (!measure && (cudaMemset(h->bar, 0, sizeof(GridBar)) != cudaSuccess ||
                                cudaMemset(h->stats, 0, (8 + MAXK) * sizeof(long long)) != cudaSuccess ||
                                (h->ps_hint && cudaMemset(h->ps_hint, 0, sizeof(int)) != cudaSuccess)))) {
        cudaGetLastError();
        free_all(h);
        delete h;
        return PIT_ECUDA;
    }
    if (c.guess_cf >= 2 && (rc = create_coarse(h)) != PIT_OK) {
        free_all(h);
        delete h;
        return rc;
    }
    *out = h;
    return PIT_OK;
}

int pit_create(const pit_config* cfg, pit_handle** out) { return create_impl(cfg, nullptr, 0, false, out); }

int pit_workspace_bytes(const pit_config* cfg, size_t* bytes) {
    if (!bytes) return PIT_EINVAL;
    *bytes = 0;
    pit_handle* h = nullptr;
    const int rc = create_impl(cfg, nullptr, 0, true, &h);
    if (rc != PIT_OK) return rc;
    *bytes = (size_t)h->bytes + WS_ALIGN;
    pit_destroy(h);
    return PIT_OK;
}

int pit_create_with_workspace(const pit_config* cfg, void* dev_ws, size_t bytes, pit_handle** out) {
    if (!out) return PIT_EINVAL;
    *out = nullptr;
    if (!dev_ws || bytes == 0) return PIT_EINVAL;
    char* base = (char*)dev_ws;
    const size_t skew = (WS_ALIGN - (uintptr_t)base % WS_ALIGN) % WS_ALIGN;   // align the arena start
    if (skew >= bytes) return PIT_EINVAL;
    return create_impl(cfg, base + skew, bytes - skew, false, out);
}

void pit_destroy(pit_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->ps_cs) cudaStreamDestroy(h->ps_cs);
    if (h->ps_ev_reset) cudaEventDestroy(h->ps_ev_reset);
    if (h->ps_h_lvl) cudaFreeHost(h->ps_h_lvl);
    free_all(h);
    delete h;
}

int pit_sizes(const pit_handle* h, int64_t* ns, int64_t* device_bytes) {
    if (!h) return PIT_EINVAL;
    if (ns) *ns = h->P.ns;
    if (device_bytes) *device_bytes = h->bytes;
    return PIT_OK;
}

static int grid_for(long long n, int sms) {
    long long g = (n + BLOCK - 1) / BLOCK;
    return (int)std::max<long long>(1, std::min<long long>(g, (long long)sms * 8));
}

// Kernel (a): the TMA-staged k_resjac_bulk when rows are 16-byte multiples and the level bases are 16-byte
// aligned, else k_resjac.  Returns the number of CTAs whose partial norms are in `part` (<= 1024).
static int launch_resjac(pit_handle* h, int grid, cudaStream_t st, const double* U, const double* u0, const double* ring,
                         double* R, double* diag, double* part) {
    const Prob& P = h->P;
    const bool law1 = P.pde == PIT_BURGERS && P.m2 == 0.0;
    const bool aligned = (P.nxu % 2 == 0) && ((uintptr_t)U % 16 == 0) && ((uintptr_t)u0 % 16 == 0) && !h->dbg.resjac_v1;
    if (aligned) {
        const int rowd = P.nxu;
        // two stages filling the shared memory: the per-tile cost (halo rows, barrier round trips) amortised
        // over the largest tile (c5: 13 rows of 512, 2 x 112 KB)
        int NS = 2;
        int RT = std::max(1, std::min(P.nyu, ((224 * 1024) / (NS * rowd * 8) - 2) / 2));
        if (h->dbg.resjac_rt > 0) RT = h->dbg.resjac_rt;
        if (h->dbg.resjac_ns > 0) NS = std::max(2, std::min(MAXSTAGE, h->dbg.resjac_ns));
        const size_t smem = (size_t)NS * (2 * RT + 2) * rowd * sizeof(double);
        if (smem <= 224 * 1024) {
            const long long ntiles = (long long)P.nt * ((P.nyu + RT - 1) / RT);
            const int g = (int)std::max<long long>(1, std::min<long long>(ntiles, std::min(h->sms, 1024)));
            const void* fn = law1 ? (const void*)k_resjac_bulk<1> : (const void*)k_resjac_bulk<0>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (law1) k_resjac_bulk<1><<<g, BLOCKA + 32, smem, st>>>(P, U, u0, ring, R, diag, part, RT, NS);
            else k_resjac_bulk<0><<<g, BLOCKA + 32, smem, st>>>(P, U, u0, ring, R, diag, part, RT, NS);
            return g;
        }
    }
    if (law1)
        k_resjac<1><<<grid, BLOCK, 0, st>>>(P, U, u0, ring, R, diag, part);
    else
        k_resjac<0><<<grid, BLOCK, 0, st>>>(P, U, u0, ring, R, diag, part);
    return grid;
}

static SolveParams base_params(pit_handle* h) {
    SolveParams S;
    std::memset(&S, 0, sizeof(S));
    S.P = h->P;
    S.U = h->U;
    S.B = h->B; S.D = h->D; S.G = h->G;
    S.slotmem = h->slots;
    S.part = h->part;
    S.hpart = h->hpart;
    S.bar = h->bar;
    S.hist = h->hist;
    S.info = h->info;
    S.newton_tol = h->cfg.newton_tol;
    S.lin_rtol = h->cfg.lin_rtol;
    S.lin_atol = h->cfg.lin_atol;
    S.newton_max = h->cfg.newton_max;
    S.lin_max = h->cfg.lin_max;
    S.stats = h->stats;
    S.stop_norm = h->cfg.stop_norm;
    return S;
}

static int launch_newton(pit_handle* h, SolveParams& S, cudaStream_t st) {
    NvtxRange nvtx_("engines1-3 k_newton*");
    void* args[] = {(void*)&S};
    CUDA_TRY(h, cudaEventRecord(h->ev[2], st));
    if (h->engine >= 2) {
        S.hmax = h->hmax;
        S.bs = h->bs;
        S.trace = h->trace;
        S.x0carry = h->dbg.x0carry;   // default: start from du^{n-1}
        S.halo = h->halo;
        {   // merged first BiCGSTAB iteration: engine 3 Newton solves on periodic grids, strips >= 3 rows
            const int Cmax = (h->G + h->D - 1) / h->D;
            S.merge = (h->engine == 3 && S.mode == 0 && h->P.bc == PIT_PERIODIC && S.x0carry &&
                       h->P.nyu / Cmax >= 3 && h->dbg.merge) ? 1 : 0;
        }
        if (h->trace) CUDA_TRY(h, cudaMemsetAsync(h->trace, 0, 13 * sizeof(unsigned long long), st));
        CUDA_TRY(h, cudaMemsetAsync(h->bs, 0, sizeof(BarState), st));
        CUDA_TRY(h, cudaMemsetAsync(h->stats, 0, (8 + MAXK) * sizeof(long long), st));
        // the dynamic shared-memory limit is a per-function attribute shared by every handle of the process
        // (e.g. the nested coarse-grid handle): set it for this launch
        const void* fn = h->engine == 3 ? col_fn(h->ppt, h->trace != nullptr, h->law, h->P.nxu) : onchip_fn(h->ppt, h->trace != nullptr, h->law);
        CUDA_TRY(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem2));
        CUDA_TRY(h, cudaLaunchCooperativeKernel(fn, dim3(h->G), dim3(h->engine == 3 ? BLOCK3 : BLOCK2), args, h->smem2, st));
    } else {
        CUDA_TRY(h, cudaMemsetAsync(h->bar, 0, sizeof(GridBar), st));
        CUDA_TRY(h, cudaLaunchCooperativeKernel((void*)k_newton, dim3(h->G), dim3(BLOCK), args, 0, st));
    }
    CUDA_TRY(h, cudaEventRecord(h->ev[3], st));
    h->launches += 1;
    return PIT_OK;
}

// Engine 4: omega and the sweep count from the Jacobi bound of A_1 at the initial iterate (device), then the
// persistent neighbour-synchronised kernel.  The LL cells and the per-iteration counters are cleared first, so a
// publication number never matches a cell of an earlier solve.
static int launch_nb(pit_handle* h, const double* d_u0, const double* ring, double* d_u_out, double* d_hist, int* d_info,
                     cudaStream_t st, const double* carry_in = nullptr, double* carry_out = nullptr, bool one_iteration = false) {
    NvtxRange nvtx_("engine4 k_newton_nb");
    const Prob& P = h->P;
    CUDA_TRY(h, cudaEventRecord(h->ev[2], st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_llx, 0, h->nb_llx_bytes, st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_llu, 0, h->nb_llu_bytes, st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_sync, 0, sizeof(unsigned) * 2 * MAXK, st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_linres, 0, sizeof(double) * 2 * MAXK, st));
    CUDA_TRY(h, cudaMemsetAsync(h->stats, 0, (8 + MAXK) * sizeof(long long), st));
    // omega and the sweep count from the Jacobi bound of A_1 at the initial iterate; a time slab keeps the values of
    // its first iteration for the later ones (the relaxation then does not change between Newton iterations)
    if (!(one_iteration && h->nb_ctl_ready)) {
        CUDA_TRY(h, cudaMemsetAsync(h->nb_qbits, 0, sizeof(unsigned long long), st));
        nb_setup_launch(P, h->U, ring, h->nb_qbits, h->cfg.lin_rtol, h->cfg.lin_sweeps, h->cfg.lin_check, h->nb_ctl,
                        std::max(1, std::min(grid_for(P.ns, h->sms), 2 * h->sms)), st);
        CUDA_TRY(h, cudaGetLastError());
        h->nb_ctl_ready = one_iteration;
    }
    NbParams S;
    std::memset(&S, 0, sizeof(S));
    S.P = P; S.u0 = d_u0; S.ring = ring; S.U = h->U; S.B = h->B; S.D = one_iteration ? 1 : h->nb_D; S.G = h->nb_G;
    S.ctl = h->nb_ctl; S.llx = h->nb_llx; S.llu = h->nb_llu; S.hpart = h->nb_hpart;
    S.arrive = h->nb_sync; S.decided = h->nb_sync + MAXK;
    S.hist = d_hist ? d_hist : h->hist; S.linres = h->nb_linres; S.info = d_info ? d_info : h->info;
    S.u_out = d_u_out; S.newton_tol = h->cfg.newton_tol; S.newton_max = one_iteration ? 1 : h->cfg.newton_max;
    S.stop_norm = h->cfg.stop_norm;
    S.carry_in = carry_in; S.carry_out = carry_out;
    S.stats = h->stats;
    S.trace = h->trace ? h->trace + 13 : nullptr;
    void* args[] = {(void*)&S};
    size_t smem4 = 0;
    int dm4 = 0, thr4 = 0;
    const void* fn = nb_fn(h->nb_rmax, h->law, P.nxu, h->nb_want, &smem4, &dm4, &thr4);
    CUDA_TRY(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->nb_smem));
    CUDA_TRY(h, cudaLaunchCooperativeKernel(fn, dim3(h->nb_G), dim3(h->nb_threads), args, h->nb_smem, st));
    CUDA_TRY(h, cudaEventRecord(h->ev[3], st));
    h->launches += 9;
    h->last_engine = 4;
    return PIT_OK;
}

// Engine 5: omega and the sweep count as engine 4 (k_nb_q / k_nb_ctl), then the persistent pipeline-of-sets kernel.
static int launch_ps(pit_handle* h, const double* d_u0, const double* ring, double* d_u_out, double* d_hist, int* d_info,
                     cudaStream_t st, bool u0_bcast) {
    NvtxRange nvtx_("engine5 k_newton_ps");
    const Prob& P = h->P;
    CUDA_TRY(h, cudaEventRecord(h->ev[2], st));
    CUDA_TRY(h, cudaMemsetAsync(h->ps_llx, 0, h->ps_llx_bytes, st));
    CUDA_TRY(h, cudaMemsetAsync(h->ps_lvl, 0, sizeof(unsigned) * h->ps_D * h->ps_Gs, st));
    if (h->ps_ev_reset) CUDA_TRY(h, cudaEventRecord(h->ps_ev_reset, st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_sync, 0, sizeof(unsigned) * 2 * MAXK, st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_linres, 0, sizeof(double) * 2 * MAXK, st));
    CUDA_TRY(h, cudaMemsetAsync(h->stats, 0, (8 + MAXK) * sizeof(long long), st));
    CUDA_TRY(h, cudaMemsetAsync(h->nb_qbits, 0, sizeof(unsigned long long), st));
    nb_setup_launch(P, u0_bcast ? d_u0 : h->U, ring, h->nb_qbits, h->cfg.lin_rtol, h->cfg.lin_sweeps, h->cfg.lin_check, h->nb_ctl,
                    std::max(1, std::min(grid_for(P.ns, h->sms), 2 * h->sms)), st);
    CUDA_TRY(h, cudaGetLastError());
    PsParams S;
    std::memset(&S, 0, sizeof(S));
    S.P = P; S.u0 = d_u0; S.ring = ring; S.U = h->U; S.B = h->B; S.D = h->ps_D; S.Gs = h->ps_Gs;
    S.ctl = h->nb_ctl; S.llx = h->ps_llx; S.lvl = h->ps_lvl; S.hpart = h->nb_hpart;
    S.arrive = h->nb_sync; S.decided = h->nb_sync + MAXK;
    S.hist = d_hist ? d_hist : h->hist; S.linres = h->nb_linres; S.info = d_info ? d_info : h->info;
    S.u_out = d_u_out; S.newton_tol = h->cfg.newton_tol; S.newton_max = h->cfg.newton_max;
    S.stop_norm = h->cfg.stop_norm;
    S.stats = h->stats;
    S.trace = h->trace ? h->trace + 13 + 13 * GMAX2 : nullptr;
    S.ax = P.dt * P.i2hx; S.bx = P.dt * P.m0 * P.ihx2; S.ay = P.dt * P.i2hy; S.by = P.dt * P.m0 * P.ihy2;
    S.aC1 = 1.0 + 2.0 * (S.bx + S.by); S.invC1 = 1.0 / S.aC1;
    S.dbg = h->dbg.ps_dbg;
    S.u0_bcast = u0_bcast ? 1 : 0;
    S.hint = h->ps_hint;
    void* args[] = {(void*)&S};
    size_t smem5 = 0;
    int thr5 = 0;
    const void* fn = ps_fn(h, h->ps_he, &smem5, &thr5);
    CUDA_TRY(h, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->ps_smem));
    CUDA_TRY(h, cudaLaunchCooperativeKernel(fn, dim3(h->ps_D * h->ps_Gs), dim3(h->ps_threads), args, h->ps_smem, st));
    CUDA_TRY(h, cudaEventRecord(h->ev[3], st));
    h->launches += 9;
    h->last_engine = 5;
    return PIT_OK;
}

// k_init_iterate bracketed by events (per-kernel device time on the launching stream, for bench.py)
static int launch_init(pit_handle* h, const double* d_u0, const double* d_guess, cudaStream_t st) {
    NvtxRange nvtx_("k_init_iterate");
    const long long N = h->P.ns * h->P.nt;
    CUDA_TRY(h, cudaEventRecord(h->ev[0], st));
    k_init_iterate<<<grid_for(N, h->sms), BLOCK, 0, st>>>(h->P.ns, h->P.nt, d_u0, d_guess, h->U);
    CUDA_TRY(h, cudaGetLastError());
    CUDA_TRY(h, cudaEventRecord(h->ev[1], st));
    h->launches += 1;
    h->timed = true;
    return PIT_OK;
}


// (b2) helpers, defined below pit_level_solve_device
static const double PIT_GATE = 1e6;     // prod ||A_i||_inf bound over a window's longest forward chain
static int ensure_pf_scratch(pit_handle* h);
static int level_anorms(pit_handle* h, const double* d_U, const double* d_bc, int n0, int L, double* out, cudaStream_t st);
static double chain_bound(const double* anorm_from_s0, int L);
static int product_window(pit_handle* h, int s0, int L, const double* d_U, const double* d_bc, const double* d_R,
                          const double* d_carry, double* d_dU, int* d_info, cudaStream_t st);
static int explicit_window(pit_handle* h, int s0, int L, const double* d_U, const double* d_bc, const double* d_R,
                           const double* d_carry, double* d_dU, int* d_info, cudaStream_t st);

// Host-driven all-at-once Newton with the (b2) product-form inverse (inverse_mode PRODUCT_WINDOW): the same
// iteration, initial guess, norms and stop rule as the persistent kernels, but Eq. (6) is inverted window by
// window with Theorem 1 (windows chained by the exact carry).  One host round trip per Newton iteration
// (norms); the default recurrence path has none.
static int solve_product(pit_handle* h, const double* d_u0, const double* d_bc, double* d_u_out, double* d_hist,
                         int* d_info, cudaStream_t st) {
    NvtxRange nvtx_("product form (b2/N3) Newton loop");
    int rc = ensure_pf_scratch(h);
    if (rc != PIT_OK) return rc;
    const Prob& P = h->P;
    const long long ns = P.ns, N = ns * P.nt;
    double* U = h->U;                             // iterate buffer 0 holds U_0 (k_init_iterate)
    const double* ring = P.bc == PIT_DIRICHLET ? d_bc : nullptr;
    const int kmax = h->cfg.newton_max;
    std::vector<double> hist((size_t)4 * kmax, 0.0), an(P.nt);
    int status = PIT_ENOCONV, kdone = 0;
    double prevmax = INFINITY;
    const int gr = std::min(grid_for(N, h->sms), 1024);
    CUDA_TRY(h, cudaEventRecord(h->ev[2], st));      // device time of the host-driven Newton loop (pit_stats)
    for (int k = 0; k < kmax; ++k) {
        const int gpart = launch_resjac(h, gr, st, U, d_u0, ring, h->pf_R, nullptr, h->d_small);
        CUDA_TRY(h, cudaGetLastError());
        k_finish_norms<<<1, BLOCK, 0, st>>>(h->d_small, gpart, N, h->d_small + 2048);
        CUDA_TRY(h, cudaGetLastError());
        double rn[2];
        CUDA_TRY(h, cudaMemcpyAsync(rn, h->d_small + 2048, sizeof(rn), cudaMemcpyDeviceToHost, st));
        for (int s0 = 1; s0 <= P.nt;) {
            int L;
            if (h->cfg.inverse_mode == PIT_INV_EXPLICIT) {     // N3: the paper's explicit form; no gate (it is what
                L = h->cfg.window > 0 ? std::min(h->cfg.window, P.nt - s0 + 1) : P.nt - s0 + 1;   // shows §7's limit)
                rc = explicit_window(h, s0, L, U, d_bc, h->pf_R, s0 == 1 ? nullptr : h->pf_dU + (long long)(s0 - 2) * ns,
                                     h->pf_dU + (long long)(s0 - 1) * ns, d_info, st);
                if (rc != PIT_OK) return rc;
                s0 += L;
                continue;
            }
            if ((rc = level_anorms(h, U, d_bc, s0, P.nt - s0 + 1, an.data(), st)) != PIT_OK) return rc;
            if (h->cfg.window > 0) {
                L = std::min(h->cfg.window, P.nt - s0 + 1);
                if (!(chain_bound(an.data(), L) <= PIT_GATE))
                    return set_err(h, PIT_ECOND, "forced window [%d, %d) fails the Section 7 gate", s0, s0 + L);
            } else {
                L = 1;
                while (s0 + L <= P.nt && chain_bound(an.data(), L + 1) <= PIT_GATE) ++L;
            }
            rc = product_window(h, s0, L, U, d_bc, h->pf_R, s0 == 1 ? nullptr : h->pf_dU + (long long)(s0 - 2) * ns,
                                h->pf_dU + (long long)(s0 - 1) * ns, d_info, st);
            if (rc != PIT_OK) return rc;
            s0 += L;
        }
        const int gu = std::min(grid_for(N, h->sms), 1024);
        k_update<<<gu, BLOCK, 0, st>>>(N, U, h->pf_dU, h->pf_part);
        CUDA_TRY(h, cudaGetLastError());
        std::vector<double> up((size_t)3 * gu);
        CUDA_TRY(h, cudaMemcpyAsync(up.data(), h->pf_part, up.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        double s2 = 0.0, mx = 0.0, bad = 0.0;
        for (int b = 0; b < gu; ++b) { s2 += up[3 * b]; mx = std::max(mx, up[3 * b + 1]); bad = std::max(bad, up[3 * b + 2]); }
        hist[4 * k + 0] = rn[0]; hist[4 * k + 1] = rn[1];
        hist[4 * k + 2] = std::sqrt(s2 / (double)N); hist[4 * k + 3] = mx;
        kdone = k + 1;
        if (bad != 0.0) { status = PIT_EBREAKDOWN; break; }
        const double dn = h->cfg.stop_norm ? hist[4 * k + 2] : mx;
        if (dn <= h->cfg.newton_tol) { status = PIT_OK; break; }
        if (k >= 1 && dn > 0.5 * prevmax && dn <= 1e3 * h->cfg.newton_tol) { status = PIT_OK_FLOOR; break; }
        prevmax = dn;
    }
    CUDA_TRY(h, cudaEventRecord(h->ev[3], st));
    if (d_u_out) CUDA_TRY(h, cudaMemcpyAsync(d_u_out, U, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    if (d_hist) CUDA_TRY(h, cudaMemcpyAsync(d_hist, hist.data(), sizeof(double) * 4 * kmax, cudaMemcpyHostToDevice, st));
    const int info[2] = {kdone, status};
    CUDA_TRY(h, cudaMemcpyAsync(d_info ? d_info : h->info, info, sizeof(info), cudaMemcpyHostToDevice, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    h->product_used = h->cfg.inverse_mode == PIT_INV_EXPLICIT ? 2 : 1;
    return PIT_OK;
}

// AUTO: the paper's literal product form when the Section 7 gate admits the whole horizon as one window
// (BASELINE c1), the recurrence otherwise.
static bool want_product(pit_handle* h, const double* d_bc, cudaStream_t st) {
    (void)d_bc; (void)st;
    return h->cfg.inverse_mode == PIT_INV_PRODUCT_WINDOW || h->cfg.inverse_mode == PIT_INV_EXPLICIT;
}

// The paper's initial iterate (pit_guess.cuh), written into iterate buffer 0.  Iterate
// buffers 1 and 2 are free before the Newton launch and serve as the interpolation scratch (B >= 3).
static int build_guess(pit_handle* h, const double* d_u0, const double* d_bc, cudaStream_t st) {
    NvtxRange nvtx_("coarse-grid guess (N1)");
    GuessParams g = h->gp;
    const Prob& P = h->P;
    const long long N = P.ns * P.nt;
    g.u0f = d_u0;
    g.cring = (P.bc == PIT_DIRICHLET && d_bc) ? h->c_ring : nullptr;
    g.cU = h->c_U;
    g.fac = h->c_fac;
    g.Tx = h->U + N;
    g.Ty = g.Tx + (long long)g.ntc * (g.bc == 1 ? g.nyc : g.nyc + 1) * g.nxu;
    g.tmp = h->U + 2 * N;
    g.U0 = h->U;
    CUDA_TRY(h, cudaEventRecord(h->ev[4], st));
    k_restrict_u0<<<grid_for(g.nsc, h->sms), BLOCK, 0, st>>>(g, h->c_u0);
    CUDA_TRY(h, cudaGetLastError());
    int nl = 1;
    if (g.cring) {
        k_restrict_ring<<<grid_for((long long)g.ntc * g.ring_len_c, h->sms), BLOCK, 0, st>>>(g, d_bc, h->c_ring);
        CUDA_TRY(h, cudaGetLastError());
        ++nl;
    }
    // sequential BDF1 on the coarse grid: ntc one-level solves.  Every pointer of the march is
    // handle-owned, so it is captured once as a CUDA graph and replayed (a level's solve is ~45 us of kernels; the
    // ~8 API calls that launch it cost about as much again); PIT_GUESS_GRAPH=0 or a failed capture march directly.
    auto march = [&](cudaStream_t s, long long& cl) -> int {
        for (int m = 1; m <= g.ntc; ++m) {
            const double* um1 = m == 1 ? h->c_u0 : h->c_U + (long long)(m - 2) * g.nsc;
            const double* rg = g.cring ? h->c_ring + (long long)(m - 1) * g.ring_len_c : nullptr;
            int rc = pit_solve_device(h->coarse, um1, rg, nullptr, h->c_U + (long long)(m - 1) * g.nsc, nullptr, h->c_info, s);
            if (rc != PIT_OK) return set_err(h, rc, "coarse-grid solve, level %d: %s", m, pit_last_error(h->coarse));
            cl += h->coarse->launches;
        }
        return PIT_OK;
    };
    long long cl = 0;
    const bool use_graph = h->dbg.guess_graph;
    // the graph bakes in whether coarse rings are passed: recapture when that changes between calls
    const int ring_now = g.cring ? 1 : 0;
    if (h->c_march && h->c_march_ring != ring_now) {
        cudaGraphExecDestroy(h->c_march);
        h->c_march = nullptr;
    }
    if (use_graph && !h->c_march) {
        cudaStream_t cs = nullptr;
        cudaGraph_t graph = nullptr;
        long long ccl = 0;
        bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            const int rc = march(cs, ccl);
            ok = cudaStreamEndCapture(cs, &graph) == cudaSuccess && rc == PIT_OK && graph &&
                 cudaGraphInstantiate(&h->c_march, graph, 0) == cudaSuccess;
        }
        if (graph) cudaGraphDestroy(graph);
        if (cs) cudaStreamDestroy(cs);
        if (!ok) { if (h->c_march) cudaGraphExecDestroy(h->c_march); h->c_march = nullptr; }
        cudaGetLastError();
        h->c_march_launches = ccl;
        h->c_march_ring = ring_now;
    }
    if (use_graph && h->c_march) {
        CUDA_TRY(h, cudaGraphLaunch(h->c_march, st));
        cl = h->c_march_launches;
    } else {
        int rc = march(st, cl);
        if (rc != PIT_OK) return rc;
    }
    const int NR = g.bc == 1 ? g.nyc : g.nyc + 1, NC = g.bc == 1 ? g.nxc : g.nxc + 1;
    const long long lines[3] = {(long long)g.ntc * NR, (long long)g.ntc * g.nxu, g.ns};
    const int K[3] = {NC, NR, g.ntc + 1};
    for (int pass = 0; pass < 3; ++pass) {
        const int per = pass < 2 && g.bc == 1;
        k_spline_setup<<<1, 1, 0, st>>>(K[pass], per, h->c_fac);
        CUDA_TRY(h, cudaGetLastError());
        const int gr = (int)std::max<long long>(1, std::min<long long>((lines[pass] + 255) / 256, (long long)h->sms * 16));
        if (pass == 0) k_spline<0><<<gr, 256, 0, st>>>(g);
        else if (pass == 1) k_spline<1><<<gr, 256, 0, st>>>(g);
        else k_spline<2><<<gr, 256, 0, st>>>(g);
        CUDA_TRY(h, cudaGetLastError());
        nl += 2;
    }
    CUDA_TRY(h, cudaEventRecord(h->ev[5], st));
    h->launches += nl + cl;
    h->guess_timed = true;
    return PIT_OK;
}

int pit_solve_device(pit_handle* h, const double* d_u0, const double* d_bc, const double* d_guess, double* d_u_out,
                     double* d_hist, int32_t* d_info, void* cuda_stream) {
    NvtxRange nvtx_("pit_solve_device");
    if (!h || !d_u0 || !d_u_out) return set_err(h, PIT_EINVAL, "null argument");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    h->launches = 0;
    h->guess_timed = false;
    int rc;
    // engine 5 reads the broadcast u^0 itself: U_0 = u^0 at every level is not materialised
    const bool ps_bcast = h->ps && !d_guess && !h->coarse && !want_product(h, d_bc, st);
    if (!d_guess && h->coarse) {
        if ((rc = build_guess(h, d_u0, d_bc, st)) != PIT_OK) return rc;
        CUDA_TRY(h, cudaEventRecord(h->ev[0], st));       // U_0 is already in place: no init kernel
        CUDA_TRY(h, cudaEventRecord(h->ev[1], st));
        h->timed = true;
    } else if (ps_bcast) {
        CUDA_TRY(h, cudaEventRecord(h->ev[0], st));
        CUDA_TRY(h, cudaEventRecord(h->ev[1], st));
        h->timed = true;
    } else if ((rc = launch_init(h, d_u0, d_guess, st)) != PIT_OK) {
        return rc;
    }
    if (d_hist) CUDA_TRY(h, cudaMemsetAsync(d_hist, 0, sizeof(double) * 4 * h->cfg.newton_max, st));
    h->product_used = 0;
    if (want_product(h, d_bc, st)) return solve_product(h, d_u0, d_bc, d_u_out, d_hist, (int*)d_info, st);
    if (((uintptr_t)d_u0 % 16) != 0) {         // engine 3 stages u^0 rows in 16-byte pieces
        CUDA_TRY(h, cudaMemcpyAsync(h->d_u0, d_u0, sizeof(double) * h->P.ns, cudaMemcpyDeviceToDevice, st));
        d_u0 = h->d_u0;
    }
    if (h->ps) return launch_ps(h, d_u0, h->P.bc == PIT_DIRICHLET ? d_bc : nullptr, d_u_out, d_hist, (int*)d_info, st, ps_bcast);
    if (h->nb) return launch_nb(h, d_u0, h->P.bc == PIT_DIRICHLET ? d_bc : nullptr, d_u_out, d_hist, (int*)d_info, st);
    SolveParams S = base_params(h);
    S.u0 = d_u0;
    S.ring = h->P.bc == PIT_DIRICHLET ? d_bc : nullptr;
    S.u_out = d_u_out;
    S.hist = d_hist ? d_hist : h->hist;
    S.info = d_info ? (int*)d_info : h->info;
    S.mode = 0;
    h->last_engine = h->engine;
    return launch_newton(h, S, st);
}

// N4: one all-at-once Newton iteration over this handle's levels as a time slab of a longer horizon (engine 4).
int pit_slab_iterate_device(pit_handle* h, const double* d_uprev, const double* d_carry_in, const double* d_bc,
                            const double* d_U_k, double* d_U_k1, double* d_carry_out, double* d_hist, int32_t* d_info,
                            void* cuda_stream) {
    NvtxRange nvtx_("pit_slab_iterate_device (N4)");
    if (!h || !d_uprev || !d_U_k || !d_U_k1 || !d_hist) return set_err(h, PIT_EINVAL, "null argument");
    if (!h->nb) return set_err(h, PIT_EINVAL, "time-slab iterations need engine 4 (pit_config.engine)");
    if (((uintptr_t)d_uprev | (uintptr_t)d_U_k | (uintptr_t)d_U_k1 | (uintptr_t)d_carry_in | (uintptr_t)d_carry_out) % 16)
        return set_err(h, PIT_EINVAL, "device buffers must be 16-byte aligned");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    h->launches = 0;
    int rc = launch_init(h, d_uprev, d_U_k, st);
    if (rc != PIT_OK) return rc;
    return launch_nb(h, d_uprev, h->P.bc == PIT_DIRICHLET ? d_bc : nullptr, d_U_k1, d_hist, (int*)d_info, st, d_carry_in,
                     d_carry_out, true);
}

int pit_initial_guess_device(pit_handle* h, const double* d_u0, const double* d_bc, double* d_U0, void* cuda_stream) {
    if (!h || !d_u0 || !d_U0) return set_err(h, PIT_EINVAL, "null argument");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    h->launches = 0;
    int rc;
    if (h->coarse) {
        if ((rc = build_guess(h, d_u0, d_bc, st)) != PIT_OK) return rc;
    } else if ((rc = launch_init(h, d_u0, nullptr, st)) != PIT_OK) {
        return rc;
    }
    CUDA_TRY(h, cudaMemcpyAsync(d_U0, h->U, sizeof(double) * h->P.ns * h->P.nt, cudaMemcpyDeviceToDevice, st));
    return PIT_OK;
}

int pit_solve(pit_handle* h, const double* u0, const double* bc, const double* guess, double* u_out, double* hist,
              int32_t* n_iter) {
    NvtxRange nvtx_("pit_solve");
    if (!h || !u0 || !u_out) return set_err(h, PIT_EINVAL, "null argument");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const Prob& P = h->P;
    const long long N = P.ns * P.nt;
    CUDA_TRY(h, cudaMemcpy(h->d_u0, u0, sizeof(double) * P.ns, cudaMemcpyHostToDevice));
    const bool has_bc = P.bc == PIT_DIRICHLET && bc;
    if (has_bc) CUDA_TRY(h, cudaMemcpy(h->d_bc, bc, sizeof(double) * P.nt * P.ring_len, cudaMemcpyHostToDevice));
    // the guess is staged straight into iterate buffer 0 (k_init_iterate then copies it in place); without a guess
    // a guess_cf handle builds the paper's coarse-grid guess there, as pit_solve_device does
    if (guess) CUDA_TRY(h, cudaMemcpy(h->U, guess, sizeof(double) * N, cudaMemcpyHostToDevice));
    h->launches = 0;
    h->guess_timed = false;
    int rc;
    const bool ps_bcast = h->ps && !guess && !h->coarse && !want_product(h, has_bc ? h->d_bc : nullptr, 0);
    if (!guess && h->coarse) {
        if ((rc = build_guess(h, h->d_u0, has_bc ? h->d_bc : nullptr, 0)) != PIT_OK) return rc;
        CUDA_TRY(h, cudaEventRecord(h->ev[0], 0));
        CUDA_TRY(h, cudaEventRecord(h->ev[1], 0));
        h->timed = true;
    } else if (ps_bcast) {
        CUDA_TRY(h, cudaEventRecord(h->ev[0], 0));
        CUDA_TRY(h, cudaEventRecord(h->ev[1], 0));
        h->timed = true;
    } else if ((rc = launch_init(h, h->d_u0, guess ? h->U : nullptr, 0)) != PIT_OK) {
        return rc;
    }
    CUDA_TRY(h, cudaMemset(h->hist, 0, sizeof(double) * 4 * h->cfg.newton_max));
    h->product_used = 0;
    const bool prod = want_product(h, has_bc ? h->d_bc : nullptr, 0);
    bool stream_copy = false;
    if (prod) {
        rc = solve_product(h, h->d_u0, has_bc ? h->d_bc : nullptr, nullptr, h->hist, h->info, 0);
    } else if (h->ps) {
        if (!h->ps_cs) {        // (first host-path solve on this handle) the streaming copy's stream, event and pinned counters
            if (cudaStreamCreateWithFlags(&h->ps_cs, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&h->ps_ev_reset, cudaEventDisableTiming) != cudaSuccess ||
                cudaHostAlloc((void**)&h->ps_h_lvl, sizeof(unsigned) * h->ps_D * h->ps_Gs, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                if (h->ps_cs) cudaStreamDestroy(h->ps_cs);
                if (h->ps_ev_reset) cudaEventDestroy(h->ps_ev_reset);
                h->ps_cs = nullptr; h->ps_ev_reset = nullptr; h->ps_h_lvl = nullptr;      // fall back to the copy after the solve
            }
        }
        rc = launch_ps(h, h->d_u0, has_bc ? h->d_bc : nullptr, nullptr, h->hist, h->info, 0, ps_bcast);
        stream_copy = rc == PIT_OK && h->ps_cs && h->ps_host_kf > 0;
    } else if (h->nb) {
        rc = launch_nb(h, h->d_u0, has_bc ? h->d_bc : nullptr, nullptr, h->hist, h->info, 0);
    } else {
        SolveParams S = base_params(h);
        S.u0 = h->d_u0;
        S.ring = has_bc ? h->d_bc : nullptr;
        S.u_out = nullptr;       // the host copy is taken straight from the final iterate buffer
        S.mode = 0;
        h->last_engine = h->engine;
        rc = launch_newton(h, S, 0);
    }
    if (rc != PIT_OK) return rc;
    // Engine 5 writes iterate K level by level (set (K-1) % D, one level counter per strip, published behind a fence):
    // with K guessed from the previous solve on this handle, the levels every strip has published are copied to the
    // host WHILE the kernel runs (the copy stream reads the counters, then the rows, in stream order); if the solve
    // ends in another iteration the copy is simply redone.  No kernel takes part in this.
    int copied = 0;
    const int Kg = h->ps_host_kf;
    if (stream_copy) {
        const int D5 = h->ps_D, Gs = h->ps_Gs, pset = (Kg - 1) % D5;
        const long long pbase = (long long)((Kg - 1) / D5) * P.nt;
        const double* Us = h->U + (long long)(Kg % h->B) * N;
        const int chunk = std::max(1, (P.nt + 31) / 32);
        CUDA_TRY(h, cudaStreamWaitEvent(h->ps_cs, h->ps_ev_reset, 0));
        for (;;) {
            const bool fin = cudaStreamQuery(0) == cudaSuccess;      // the kernel (and everything before it) has finished
            CUDA_TRY(h, cudaMemcpyAsync(h->ps_h_lvl, h->ps_lvl, sizeof(unsigned) * D5 * Gs, cudaMemcpyDeviceToHost, h->ps_cs));
            CUDA_TRY(h, cudaStreamSynchronize(h->ps_cs));
            unsigned mn = 0xffffffffu;
            for (int q = 0; q < Gs; ++q) mn = std::min(mn, h->ps_h_lvl[(size_t)pset * Gs + q]);
            const long long done = std::max(0ll, std::min<long long>((long long)mn - pbase, P.nt));
            while (copied < P.nt && (copied + chunk <= done || done == P.nt)) {
                const int L = std::min(chunk, P.nt - copied);
                CUDA_TRY(h, cudaMemcpyAsync(u_out + (long long)copied * P.ns, Us + (long long)copied * P.ns,
                                            sizeof(double) * L * P.ns, cudaMemcpyDeviceToHost, h->ps_cs));
                copied += L;
            }
            if (fin) break;
        }
        cudaGetLastError();      // (cudaStreamQuery's cudaErrorNotReady)
    }
    int info[2];
    CUDA_TRY(h, cudaMemcpy(info, h->info, sizeof(info), cudaMemcpyDeviceToHost));
    const int kf = info[0];
    const double* Uf = prod ? h->U : h->U + (long long)(kf % h->B) * N;
    if (stream_copy) {
        CUDA_TRY(h, cudaStreamSynchronize(h->ps_cs));
        if (kf != Kg) copied = 0;                                   // the guess was wrong: the rows copied so far are another iterate's
    }
    if (copied < P.nt)
        CUDA_TRY(h, cudaMemcpy(u_out + (long long)copied * P.ns, Uf + (long long)copied * P.ns,
                               sizeof(double) * (P.nt - copied) * P.ns, cudaMemcpyDeviceToHost));
    if (h->ps && !prod) h->ps_host_kf = kf;
    if (hist) CUDA_TRY(h, cudaMemcpy(hist, h->hist, sizeof(double) * 4 * h->cfg.newton_max, cudaMemcpyDeviceToHost));
    if (n_iter) *n_iter = kf;
    return info[1];
}

int pit_residual_device(pit_handle* h, const double* d_U, const double* d_u0, const double* d_bc, double* d_R,
                        double* d_diag, double* d_norms, void* cuda_stream) {
    NvtxRange nvtx_("pit_residual_device (kernel a)");
    if (!h || !d_U || !d_u0 || !d_R) return set_err(h, PIT_EINVAL, "null argument");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const long long N = h->P.ns * h->P.nt;
    const int grid = std::min(grid_for(N, h->sms), 1024);
    const int gpart = launch_resjac(h, grid, st, d_U, d_u0, h->P.bc == PIT_DIRICHLET ? d_bc : nullptr, d_R, d_diag, h->d_small);
    CUDA_TRY(h, cudaGetLastError());
    if (d_norms) {
        k_finish_norms<<<1, BLOCK, 0, st>>>(h->d_small, gpart, N, d_norms);
        CUDA_TRY(h, cudaGetLastError());
    }
    return PIT_OK;
}

// Batch of independent level solves A_{lev[a]} x_a = b_a (A at the iterate d_U [nt][ns]); chunks of <= D.
static int level_solves(pit_handle* h, int nb, const int* lev, const double* const* b, double* const* x, const double* d_U,
                        const double* d_bc, int* d_info, cudaStream_t st) {
    if (h->engine == 3 && ((uintptr_t)d_U % 16) != 0)     // engine 3 stages u rows in 16-byte pieces
        return set_err(h, PIT_EINVAL, "d_U must be 16-byte aligned");
    for (int a0 = 0; a0 < nb; a0 += h->D) {
        SolveParams S = base_params(h);
        S.U = const_cast<double*>(d_U);
        S.u0 = d_U;
        S.ring = h->P.bc == PIT_DIRICHLET ? d_bc : nullptr;
        S.mode = 1;
        S.nb = std::min(h->D, nb - a0);
        for (int j = 0; j < S.nb; ++j) {
            S.blev[j] = lev[a0 + j];
            S.bptr[j] = b[a0 + j];
            S.xptr[j] = x[a0 + j];
        }
        S.info = d_info ? d_info : h->info;
        S.x0carry = 0;
        int rc = launch_newton(h, S, st);
        if (rc != PIT_OK) return rc;
    }
    return PIT_OK;
}

int pit_level_solve_device(pit_handle* h, int32_t level, const double* d_U, const double* d_bc, const double* d_b,
                           double* d_x, int32_t* d_info, void* cuda_stream) {
    if (!h || !d_U || !d_b || !d_x) return set_err(h, PIT_EINVAL, "null argument");
    if (level < 1 || level > h->P.nt) return set_err(h, PIT_EINVAL, "level %d out of 1..%d", level, h->P.nt);
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int lev[1] = {level};
    const double* b[1] = {d_b};
    double* x[1] = {d_x};
    return level_solves(h, 1, lev, b, x, d_U, d_bc, (int*)d_info, (cudaStream_t)cuda_stream);
}

// ---- (b2): the literal Theorem 1 product form inside a Section 7 window ------------------------------

static int ensure_pf_scratch(pit_handle* h) {
    if (h->pf_Y) return PIT_OK;
    const long long ns = h->P.ns, N = ns * h->P.nt;
    int rc;
    if ((rc = dalloc(h, &h->pf_Y, (size_t)(2 * N), true)) || (rc = dalloc(h, &h->pf_R, (size_t)N, true)) ||
        (rc = dalloc(h, &h->pf_dU, (size_t)N, true)) || (rc = dalloc(h, &h->pf_part, (size_t)(4096 + 8), true)))
        return rc;
    return PIT_OK;
}

// ||A_n||_inf for levels n0..n0+L-1 at d_U -> host array (synchronizes the stream).
static int level_anorms(pit_handle* h, const double* d_U, const double* d_bc, int n0, int L, double* out, cudaStream_t st) {
    const int gx = std::max(1, std::min(64, (int)((h->P.ns + BLOCK - 1) / BLOCK)));
    for (int c0 = 0; c0 < L; c0 += 32) {
        const int Lc = std::min(32, L - c0);
        k_anorm<<<dim3(gx, Lc), BLOCK, 0, st>>>(h->P, d_U, h->P.bc == PIT_DIRICHLET ? d_bc : nullptr, n0 + c0, h->pf_part);
        CUDA_TRY(h, cudaGetLastError());
        std::vector<double> tmp((size_t)gx * Lc);
        CUDA_TRY(h, cudaMemcpyAsync(tmp.data(), h->pf_part, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(h, cudaStreamSynchronize(st));
        for (int j = 0; j < Lc; ++j) {
            double m = 0.0;
            for (int b = 0; b < gx; ++b) m = std::max(m, tmp[(size_t)j * gx + b]);
            out[c0 + j] = m;
        }
    }
    return PIT_OK;
}

// Longest chain of a window [s0, s0+L): P^{L-1} r^L applies A_{s0} .. A_{s0+L-2}.
static double chain_bound(const double* anorm_from_s0, int L) {
    double p = 1.0;
    for (int i = 0; i + 1 < L; ++i) p *= anorm_from_s0[i];
    return p;
}

// du^{s0..s0+L-1} of Eq. (6) by Theorem 1: y^m = A_1..A_{m-1} r^m (batched stencil chain), r~^m = sum_{j<=m} y^j
// (level scan), then P^m du^m = r~^m solved as A_m^{-1} .. A_1^{-1} r~^m (nested multi-right-hand-side
// level solves: at nested step q every m >= q solves with the same A_q).  Window-local A_m = A_{s0+m-1}.
static int product_window(pit_handle* h, int s0, int L, const double* d_U, const double* d_bc, const double* d_R,
                          const double* d_carry, double* d_dU, int* d_info, cudaStream_t st) {
    const long long ns = h->P.ns;
    double* Y = h->pf_Y;                       // [L][ns] chain / scan / nested-solve vectors
    double* T = h->pf_Y + (long long)h->P.nt * ns;   // [L][ns] ping-pong partner of the chain
    CUDA_TRY(h, cudaMemcpyAsync(Y, d_R + (long long)(s0 - 1) * ns, sizeof(double) * L * ns, cudaMemcpyDeviceToDevice, st));
    if (d_carry) {   // first row of the window: A_{s0} du^{s0} = r^{s0} + du^{s0-1}
        k_update<<<grid_for(ns, h->sms), BLOCK, 0, st>>>(ns, Y, d_carry, h->pf_part);   // Y[0] += carry
        CUDA_TRY(h, cudaGetLastError());
    }
    const int gx = grid_for(ns, h->sms);
    for (int j = 1; j <= L - 1; ++j) {         // chain step j: vector m (m - 1 >= j) applies A_{m-j}
        std::vector<int> ms;
        for (int m = j + 1; m <= L; ++m) ms.push_back(m);
        for (size_t c0 = 0; c0 < ms.size(); c0 += MAXD) {
            MatvecJobs J;
            J.n = (int)std::min<size_t>(MAXD, ms.size() - c0);
            for (int t = 0; t < J.n; ++t) {
                const int m = ms[c0 + t];
                J.lev[t] = s0 + (m - j) - 1;
                J.x[t] = Y + (long long)(m - 1) * ns;
                J.y[t] = T + (long long)(m - 1) * ns;
            }
            k_matvec_batch<<<dim3(std::min(gx, 256), J.n), BLOCK, 0, st>>>(h->P, d_U, h->P.bc == PIT_DIRICHLET ? d_bc : nullptr, J);
            CUDA_TRY(h, cudaGetLastError());
        }
        // move the chained vectors back into Y
        CUDA_TRY(h, cudaMemcpyAsync(Y + (long long)j * ns, T + (long long)j * ns, sizeof(double) * (L - j) * ns,
                                    cudaMemcpyDeviceToDevice, st));
    }
    k_level_prefix<<<gx, BLOCK, 0, st>>>(ns, L, Y);
    CUDA_TRY(h, cudaGetLastError());
    for (int q = 1; q <= L; ++q) {             // nested step q: every m >= q solves A_q z = z
        std::vector<int> lev;
        std::vector<const double*> b;
        std::vector<double*> x;
        for (int m = q; m <= L; ++m) {
            lev.push_back(s0 + q - 1);
            b.push_back(Y + (long long)(m - 1) * ns);
            x.push_back(Y + (long long)(m - 1) * ns);
        }
        int rc = level_solves(h, (int)lev.size(), lev.data(), b.data(), x.data(), d_U, d_bc, d_info, st);
        if (rc != PIT_OK) return rc;
    }
    CUDA_TRY(h, cudaMemcpyAsync(d_dU, Y, sizeof(double) * L * ns, cudaMemcpyDeviceToDevice, st));
    return PIT_OK;
}

int pit_product_window_device(pit_handle* h, int32_t s0, int32_t L, const double* d_U, const double* d_u0,
                              const double* d_bc, const double* d_R, const double* d_carry, double* d_dU,
                              int32_t* d_info, void* cuda_stream) {
    (void)d_u0;
    if (!h || !d_U || !d_R || !d_dU) return set_err(h, PIT_EINVAL, "null argument");
    if (s0 < 1 || L < 1 || s0 + L - 1 > h->P.nt) return set_err(h, PIT_EINVAL, "window [%d, %d) out of 1..%d", s0, s0 + L, h->P.nt);
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    int rc = ensure_pf_scratch(h);
    if (rc != PIT_OK) return rc;
    std::vector<double> an(L);
    if ((rc = level_anorms(h, d_U, d_bc, s0, L, an.data(), st)) != PIT_OK) return rc;
    const double bound = chain_bound(an.data(), L);
    if (!(bound <= PIT_GATE))
        return set_err(h, PIT_ECOND, "window [%d, %d): prod ||A_i||_inf = %.3e > %.0e (Section 7 gate)", s0, s0 + L, bound, PIT_GATE);
    return product_window(h, s0, L, d_U, d_bc, d_R, d_carry, d_dU, (int*)d_info, st);
}

int pit_stats(pit_handle* h, int64_t* out, int32_t n) {
    if (!h || !out || n < 1) return PIT_EINVAL;
    long long s[8 + MAXK];
    CUDA_TRY(h, cudaSetDevice(h->device));
    CUDA_TRY(h, cudaMemcpy(s, h->stats, sizeof(s), cudaMemcpyDeviceToHost));
    float t_init = 0.f, t_newton = 0.f;
    if (h->timed) {
        CUDA_TRY(h, cudaEventSynchronize(h->ev[3]));
        CUDA_TRY(h, cudaEventElapsedTime(&t_init, h->ev[0], h->ev[1]));
        CUDA_TRY(h, cudaEventElapsedTime(&t_newton, h->ev[2], h->ev[3]));
    }
    unsigned long long tr[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (h->trace) CUDA_TRY(h, cudaMemcpy(tr, h->trace, sizeof(tr), cudaMemcpyDeviceToHost));
    const bool nbps = h->last_engine == 4 || h->last_engine == 5;      // these kernels report their own depth and grid
    const long long v[17] = {s[0], s[1], nbps ? s[2] : h->D, nbps ? s[3] : h->G, h->launches, (long long)(t_newton * 1e6), (long long)(t_init * 1e6),
                             h->last_engine ? h->last_engine : h->engine, (long long)tr[0], (long long)tr[1], (long long)tr[2], (long long)tr[3],
                             (long long)tr[4], (long long)tr[5], (long long)tr[6], (long long)h->product_used, s[4]};
    for (int i = 0; i < n && i < 17; ++i) out[i] = v[i];
    for (int i = 17; i < n && i < 17 + MAXK; ++i) out[i] = s[8 + (i - 17)];
    for (int i = 17 + MAXK; i < n && i < 17 + MAXK + 6; ++i) out[i] = (long long)tr[7 + (i - 17 - MAXK)];
    if (n > 17 + MAXK + 6) {
        float t_guess = 0.f;
        if (h->guess_timed) CUDA_TRY(h, cudaEventElapsedTime(&t_guess, h->ev[4], h->ev[5]));
        out[17 + MAXK + 6] = (long long)(t_guess * 1e6);
    }
    if (n > 17 + MAXK + 7) out[17 + MAXK + 7] = s[5];   // grid barriers of the last solve (engine 3; 0 otherwise)
    // trace builds: per-CTA cycle accounts [G][13] after the fixed fields (engine 3 only; tools/skew_run.py)
    const int base = 17 + MAXK + 8;
    if (h->trace && h->engine == 3 && n >= base + 13 * h->G) {
        std::vector<unsigned long long> pc((size_t)13 * h->G);
        CUDA_TRY(h, cudaMemcpy(pc.data(), h->trace + 13, pc.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < pc.size(); ++i) out[base + i] = (long long)pc[i];
    }
    return PIT_OK;
}

int pit_engine_info(pit_handle* h, double* out, int32_t n) {
    if (!h || !out || n < 1) return PIT_EINVAL;
    CUDA_TRY(h, cudaSetDevice(h->device));
    std::vector<double> v((size_t)4 + 2 * MAXK + 2 * NB_TR, 0.0);
    v[0] = h->last_engine ? h->last_engine : h->engine;
    if (h->last_engine == 4 || h->last_engine == 5) {
        double ctl[3];
        CUDA_TRY(h, cudaMemcpy(ctl, h->nb_ctl, sizeof(ctl), cudaMemcpyDeviceToHost));
        v[1] = ctl[0]; v[2] = ctl[1]; v[3] = ctl[2];
        CUDA_TRY(h, cudaMemcpy(v.data() + 4, h->nb_linres, sizeof(double) * 2 * MAXK, cudaMemcpyDeviceToHost));
        if (h->trace) {   // cycle accounts: mean and max over CTAs (PIT_TRACE builds of the handle)
            static_assert(PS_TR == NB_TR, "one trace layout");
            const int ng = h->last_engine == 5 ? h->ps_D * h->ps_Gs : h->nb_G;
            std::vector<unsigned long long> tr((size_t)ng * NB_TR);
            CUDA_TRY(h, cudaMemcpy(tr.data(), h->trace + 13 + (h->last_engine == 5 ? 13 * GMAX2 : 0), tr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            for (int i = 0; i < NB_TR; ++i) {
                double sum = 0, mx = 0;
                for (int g = 0; g < ng; ++g) { sum += (double)tr[(size_t)g * NB_TR + i]; mx = std::max(mx, (double)tr[(size_t)g * NB_TR + i]); }
                v[4 + 2 * MAXK + i] = sum / ng;
                v[4 + 2 * MAXK + NB_TR + i] = mx;
            }
        }
    }
    for (int i = 0; i < n && i < (int)v.size(); ++i) out[i] = v[i];
    return PIT_OK;
}

// ---- N3: the paper's explicit banded form (pit_explicit.cuh) --------------------------------------------

__global__ void k_err_to_info(const unsigned* err, int* info) {
    info[0] = 0;
    info[1] = *err ? PIT_EBREAKDOWN : PIT_OK;
}

// du^{s0..s0+L-1} of Eq. (6) by the explicit decoupled form: A_m coefficients, P^1 = A_1 and P^m = P^{m-1} A_m
// in band storage (Eq. 10), y^m = P^{m-1} r^m and the level scan r~^m = sum_{j<=m} y^j, the
// §7 diagonal scaling, then one banded LU without pivoting + substitution per level.  r^1 includes the carry.
static int explicit_window(pit_handle* h, int s0, int L, const double* d_U, const double* d_bc, const double* d_R,
                           const double* d_carry, double* d_dU, int* d_info, cudaStream_t st) {
    const Prob& P = h->P;
    const long long ns = P.ns;
    if (P.bc != PIT_DIRICHLET) return set_err(h, PIT_EINVAL, "explicit form needs Dirichlet boundaries");
    const long long w = std::min<long long>((long long)L * P.nxu, ns - 1), BW = 2 * w + 1;
    const long long needB = (long long)L * ns * BW, needC = (long long)L * 5 * ns;
    if ((double)needB * 8.0 > 16e9)
        return set_err(h, PIT_EINVAL, "explicit form: band storage of %d levels x %lld x %lld needs %.1f GB (> 16 GB)", L,
                       ns, BW, (double)needB * 8e-9);
    const size_t smem = (size_t)std::max<long long>(1, 2 * w) * sizeof(double);
    if (smem > 200 * 1024) return set_err(h, PIT_EINVAL, "explicit form: half-bandwidth %lld too large", w);
    int rc = ensure_pf_scratch(h);
    if (rc != PIT_OK) return rc;
    if (needB > h->ex_capB) {
        dfree(h, h->ex_B); h->ex_B = nullptr; h->ex_capB = 0;
        if ((rc = dalloc(h, &h->ex_B, (size_t)needB, true))) return rc;
        h->ex_capB = needB;
    }
    if (needC > h->ex_capC) {
        dfree(h, h->ex_C5); h->ex_C5 = nullptr; h->ex_capC = 0;
        if ((rc = dalloc(h, &h->ex_C5, (size_t)needC, true))) return rc;
        h->ex_capC = needC;
    }
    if (!h->ex_err) CUDA_TRY(h, cudaMalloc((void**)&h->ex_err, sizeof(unsigned)));
    const int gx = std::max(1, std::min(grid_for(ns, h->sms), 256));
    k_coef5<<<dim3(gx, L), BLOCK, 0, st>>>(P, d_U, d_bc, s0, h->ex_C5);
    CUDA_TRY(h, cudaGetLastError());
    const int gb = std::max(1, std::min(grid_for(ns * BW, h->sms), 16 * h->sms));
    k_band_init<<<gb, BLOCK, 0, st>>>(ns, P.nxu, (int)w, h->ex_C5, h->ex_B);
    CUDA_TRY(h, cudaGetLastError());
    for (int m = 2; m <= L; ++m) {
        k_band_mul<<<gb, BLOCK, 0, st>>>(ns, P.nxu, (int)w, h->ex_B + (long long)(m - 2) * ns * BW,
                                         h->ex_C5 + (long long)(m - 1) * 5 * ns, h->ex_B + (long long)(m - 1) * ns * BW);
        CUDA_TRY(h, cudaGetLastError());
    }
    const double* Rw = d_R + (long long)(s0 - 1) * ns;
    CUDA_TRY(h, cudaMemcpyAsync(d_dU, Rw, sizeof(double) * ns, cudaMemcpyDeviceToDevice, st));
    if (d_carry) {   // first row of the window: A_{s0} du^{s0} = r^{s0} + du^{s0-1}
        k_update<<<grid_for(ns, h->sms), BLOCK, 0, st>>>(ns, d_dU, d_carry, h->pf_part);
        CUDA_TRY(h, cudaGetLastError());
    }
    if (L > 1) {
        k_band_rhs<<<dim3(gx, L - 1), BLOCK, 0, st>>>(ns, (int)w, h->ex_B, Rw, d_dU);
        CUDA_TRY(h, cudaGetLastError());
    }
    k_level_prefix<<<gx, BLOCK, 0, st>>>(ns, L, d_dU);
    CUDA_TRY(h, cudaGetLastError());
    k_band_scale<<<dim3(gx, L), BLOCK, 0, st>>>(ns, (int)w, h->ex_B, d_dU);
    CUDA_TRY(h, cudaGetLastError());
    CUDA_TRY(h, cudaMemsetAsync(h->ex_err, 0, sizeof(unsigned), st));
    CUDA_TRY(h, cudaFuncSetAttribute(k_band_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_band_lu_solve<<<L, BLOCKX, smem, st>>>(ns, P.nxu, (int)w, h->ex_B, d_dU, h->ex_err);
    CUDA_TRY(h, cudaGetLastError());
    if (d_info) {
        k_err_to_info<<<1, 1, 0, st>>>(h->ex_err, d_info);
        CUDA_TRY(h, cudaGetLastError());
    }
    h->launches += 7 + (L - 1) + (d_carry ? 1 : 0) + (d_info ? 1 : 0);
    return PIT_OK;
}

int pit_explicit_window_device(pit_handle* h, int32_t s0, int32_t L, const double* d_U, const double* d_u0,
                               const double* d_bc, const double* d_R, const double* d_carry, double* d_dU,
                               int32_t* d_info, void* cuda_stream) {
    (void)d_u0;
    if (!h || !d_U || !d_R || !d_dU) return set_err(h, PIT_EINVAL, "null argument");
    if (s0 < 1 || L < 1 || s0 + L - 1 > h->P.nt) return set_err(h, PIT_EINVAL, "window [%d, %d) out of 1..%d", s0, s0 + L, h->P.nt);
    CUDA_TRY(h, cudaSetDevice(h->device));
    return explicit_window(h, s0, L, d_U, d_bc, d_R, d_carry, d_dU, (int*)d_info, (cudaStream_t)cuda_stream);
}
