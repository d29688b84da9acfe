// pit_ps_law1.cu — engine-5 instantiations (LAW 1: viscous Burgers, constant viscosity; periodic grids), compiled as
// their own translation unit.
#include "pit_newton_ps.cuh"

namespace pit {

template <int NXU, int HE, int RG>
static const void* ps_inst(bool trace, size_t* smem, int* threads) {
    *smem = PsEngine<NXU, HE, RG, false>::SMEM;
    *threads = PsEngine<NXU, HE, RG, false>::NTH;
    return trace ? (const void*)k_newton_ps<NXU, HE, RG, true> : (const void*)k_newton_ps<NXU, HE, RG, false>;
}

// Instantiated shapes: (row length, base strip height HE); a set's strips have HE or HE + 2 rows.
const void* ps_kernel_law1(int nxu, int he, int rg, bool trace, size_t* smem, int* threads) {
    if (nxu == 512 && he == 20 && rg == 1) return ps_inst<512, 20, 1>(trace, smem, threads);   // (experiment: one row group, 256 threads)
    if (rg != 2) return nullptr;
    if (nxu == 512 && he == 20) return ps_inst<512, 20, 2>(trace, smem, threads);     // BASELINE c5: 6 sets of 24 strips
    if (nxu == 256 && he == 14) return ps_inst<256, 14, 2>(trace, smem, threads);     // BASELINE c4: 8 sets of 18 strips
    if (nxu == 64 && he == 2) return ps_inst<64, 2, 2>(trace, smem, threads);         // BASELINE c2: 8 sets of 18 strips of 4 / 2 rows
    return nullptr;
}

}  // namespace pit
