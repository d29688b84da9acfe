// pit_ps_law0.cu — engine-5 instantiations for the general law (pit_newton_ps0.cuh), compiled as their own translation unit.
#include "pit_newton_ps0.cuh"

namespace pit {

template <int NXU, int HE, bool PER>
static const void* ps0_inst(bool trace, size_t* smem, int* threads) {
    *smem = PsEngine0<NXU, HE, PER, false>::SMEM;
    *threads = PsEngine0<NXU, HE, PER, false>::NTH;
    return trace ? (const void*)k_newton_ps0<NXU, HE, PER, true> : (const void*)k_newton_ps0<NXU, HE, PER, false>;
}

// Instantiated shapes: (row length, base strip height HE, periodic); a set's strips have HE or HE + 2 rows.
const void* ps_kernel_law0(int nxu, int he, int periodic, bool trace, size_t* smem, int* threads) {
    if (nxu == 256 && he == 10) return periodic ? ps0_inst<256, 10, true>(trace, smem, threads) : ps0_inst<256, 10, false>(trace, smem, threads);   // BASELINE c3: 6 sets of 24 strips
    return nullptr;
}

}  // namespace pit
