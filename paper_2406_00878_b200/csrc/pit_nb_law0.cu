// pit_nb_law0.cu — engine-4 instantiations for LAW 0 (general mu(u) = m0 + m2 u^2: the heat law and Burgers with m2 > 0), compiled as their own translation unit.
#include "pit_newton_nb.cuh"

namespace pit {

template <int HB, int NXU, int DM, int CPT>
static const void* nb_inst(size_t* smem, int* dm, int* threads) {
    *smem = NbEngine<HB, 0, NXU, DM, CPT>::SMEM;
    *dm = DM;
    *threads = DM * (NXU / CPT);
    return (const void*)k_newton_nb<HB, 0, NXU, DM, CPT>;
}

// Instantiated shapes: (row length, base strip height HB) -> warp groups DM (Newton iterations in flight) and columns
// per thread CPT = 2.  Rows of 512: 2 groups (768 threads at 3 groups cap registers at 80 and spill in the sweeps;
// 4 columns per thread was slower everywhere); want_dm = 3 asks for the 3-group build.
const void* nb_kernel_law0(int hb, int nxu, int want_dm, size_t* smem, int* dm, int* threads) {
    switch (nxu) {
        case 64: return hb == 1 ? nb_inst<1, 64, 4, 2>(smem, dm, threads) : nullptr;
        case 128: return hb == 1 ? nb_inst<1, 128, 4, 2>(smem, dm, threads) : nullptr;
        case 256:
            if (want_dm == 6)      // six groups of 128 threads: the six iterations of a c3-like solve in one pass
                return hb == 1 ? nb_inst<1, 256, 6, 2>(smem, dm, threads) : nullptr;
            return hb == 1 ? nb_inst<1, 256, 4, 2>(smem, dm, threads)
                           : (hb == 2 ? nb_inst<2, 256, 4, 2>(smem, dm, threads) : nullptr);
        case 512:
            if (want_dm == 3)
                return hb == 1 ? nb_inst<1, 512, 3, 2>(smem, dm, threads)
                               : (hb == 2 ? nb_inst<2, 512, 3, 2>(smem, dm, threads) : (hb == 3 ? nb_inst<3, 512, 3, 2>(smem, dm, threads) : nullptr));
            return hb == 1 ? nb_inst<1, 512, 2, 2>(smem, dm, threads)
                           : (hb == 2 ? nb_inst<2, 512, 2, 2>(smem, dm, threads) : (hb == 3 ? nb_inst<3, 512, 2, 2>(smem, dm, threads) : nullptr));
        default: return nullptr;
    }
}

}  // namespace pit
