// pit_nb_law1.cu — engine-4 instantiations for LAW 1 (viscous Burgers, constant viscosity), compiled as their own translation unit.
#include "pit_newton_nb.cuh"

namespace pit {

template <int HB, int NXU, int DM>
static const void* nb_inst(size_t* smem, int* dm) {
    *smem = NbEngine<HB, 1, NXU, DM>::SMEM;
    *dm = DM;
    return (const void*)k_newton_nb<HB, 1, NXU, DM>;
}

// warp groups: DM * NXU / 2 <= 1024 threads; rows of 512: 2 groups by default, 3 on request (pipeline_depth 3)
const void* nb_kernel_law1(int hb, int nxu, int want_dm, size_t* smem, int* dm) {
    switch (nxu) {
        case 64: return hb == 1 ? nb_inst<1, 64, 4>(smem, dm) : nullptr;
        case 128: return hb == 1 ? nb_inst<1, 128, 4>(smem, dm) : nullptr;
        case 256: return hb == 1 ? nb_inst<1, 256, 4>(smem, dm) : (hb == 2 ? nb_inst<2, 256, 4>(smem, dm) : nullptr);
        case 512:
            if (want_dm != 3)   // default: 2 groups (128 registers; the 3-group build spills)
                return hb == 1 ? nb_inst<1, 512, 2>(smem, dm) : (hb == 2 ? nb_inst<2, 512, 2>(smem, dm) : (hb == 3 ? nb_inst<3, 512, 2>(smem, dm) : nullptr));
            return hb == 1 ? nb_inst<1, 512, 3>(smem, dm) : (hb == 2 ? nb_inst<2, 512, 3>(smem, dm) : (hb == 3 ? nb_inst<3, 512, 3>(smem, dm) : nullptr));
        default: return nullptr;
    }
}

void nb_setup_launch(const Prob& P, const double* U1, const double* ring, unsigned long long* qbits, double lin_rtol,
                     int sweeps, int check, double* ctl, int grid, cudaStream_t st) {
    k_nb_q<<<grid, BLOCK, 0, st>>>(P, U1, ring, qbits);
    k_nb_ctl<<<1, 1, 0, st>>>(qbits, lin_rtol, sweeps, check, ctl);
}

}  // namespace pit
