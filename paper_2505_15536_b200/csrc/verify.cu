// verify.cu - parity-test instantiations of the K3 / K6 kernels (VER = true):
// the same template source as the production kernels in engine.cu, plus a
// store of every evaluated candidate's cost into the context's verify sink
// (gp_diag_verify_begin / _end).  A separate translation unit so that the
// doubled instantiation set compiles in parallel with engine.cu.
#include "k3_argmin.cuh"
#include "k3_sweep_rec.cuh"
#include "verify.h"

SwFn pick_sweep_verify(int mode, int nb, int k) {
    static const SwFn table[3][4] = {
        {k3_sweep<0, 1, 0, true>, k3_sweep<0, 2, 0, true>, k3_sweep<0, 3, 0, true>, k3_sweep<0, 4, 0, true>},
        {k3_sweep<1, 1, 0, true>, k3_sweep<1, 2, 0, true>, k3_sweep<1, 3, 0, true>, k3_sweep<1, 4, 0, true>},
        {k3_sweep<2, 1, 0, true>, k3_sweep<2, 2, 0, true>, k3_sweep<2, 3, 0, true>, k3_sweep<2, 4, 0, true>}};
    static const SwFn fixed[4][4] = {
        {k3_sweep<2, 1, 3, true>, k3_sweep<2, 1, 4, true>, k3_sweep<2, 1, 5, true>, k3_sweep<2, 1, 6, true>},
        {k3_sweep<2, 2, 3, true>, k3_sweep<2, 2, 4, true>, k3_sweep<2, 2, 5, true>, k3_sweep<2, 2, 6, true>},
        {k3_sweep<2, 3, 3, true>, k3_sweep<2, 3, 4, true>, k3_sweep<2, 3, 5, true>, k3_sweep<2, 3, 6, true>},
        {k3_sweep<2, 4, 3, true>, k3_sweep<2, 4, 4, true>, k3_sweep<2, 4, 5, true>, k3_sweep<2, 4, 6, true>}};
    return (mode == 2 && k >= 3 && k <= 6) ? fixed[nb - 1][k - 3] : table[mode][nb - 1];
}

K3Fn pick_argmin_verify(int mode, int nb) {
    static const K3Fn table[3][4] = {
        {k3_argmin<0, 1, true>, k3_argmin<0, 2, true>, k3_argmin<0, 3, true>, k3_argmin<0, 4, true>},
        {k3_argmin<1, 1, true>, k3_argmin<1, 2, true>, k3_argmin<1, 3, true>, k3_argmin<1, 4, true>},
        {k3_argmin<2, 1, true>, k3_argmin<2, 2, true>, k3_argmin<2, 3, true>, k3_argmin<2, 4, true>}};
    return table[mode][nb - 1];
}

SwFn pick_sweep_rec_verify(int nb, int k) {
    static const SwFn table[4][4] = {
        {k3_sweep_rec<1, 3, true>, k3_sweep_rec<1, 4, true>, k3_sweep_rec<1, 5, true>, k3_sweep_rec<1, 6, true>},
        {k3_sweep_rec<2, 3, true>, k3_sweep_rec<2, 4, true>, k3_sweep_rec<2, 5, true>, k3_sweep_rec<2, 6, true>},
        {k3_sweep_rec<3, 3, true>, k3_sweep_rec<3, 4, true>, k3_sweep_rec<3, 5, true>, k3_sweep_rec<3, 6, true>},
        {k3_sweep_rec<4, 3, true>, k3_sweep_rec<4, 4, true>, k3_sweep_rec<4, 5, true>, k3_sweep_rec<4, 6, true>}};
    return table[nb - 1][k - 3];
}

unsigned int verify_tu_checks() {
#if defined(GP_CHECKS)
    unsigned int v = 0, z = 0;
    if (cudaMemcpyFromSymbol(&v, g_chk_line, sizeof(v)) != cudaSuccess) return 0xFFFFFFFEu;
    cudaMemcpyToSymbol(g_chk_line, &z, sizeof(z));
    return v;
#else
    return 0;
#endif
}
